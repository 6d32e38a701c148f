"""Thin Python binding over libcx.so (include/cx.h). Argument marshalling only:
every step of the hot path runs in the CUDA kernels behind the C ABI. torch
supplies device memory and the current stream; nothing here computes.

There is no CPU fallback: if libcx.so cannot be loaded (or built) the import
of the binding raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import torch

from . import _build

# --- enums mirrored from include/cx.h --------------------------------------
SEQUENCE, TREE, DAG = 0, 1, 2
TREERNN, TREEFC, TREELSTM, TREEGRU, MVRNN, DAGRNN, SIMPLETREEGRU = range(7)
F32, BF16 = 0, 1
OK, E_ARG, E_CHILD_RANGE, E_CHILD_LAYOUT, E_KIND, E_CYCLE, E_ARITY, E_WORD_RANGE, \
    E_UNSUPPORTED, E_WORKSPACE, E_CUDA = range(11)

CELL_IDS = {"treernn": TREERNN, "treefc": TREEFC, "treelstm": TREELSTM,
            "treegru": TREEGRU, "mvrnn": MVRNN, "dagrnn": DAGRNN,
            "simpletreegru": SIMPLETREEGRU}
N_WEIGHTS = {TREERNN: 0, TREEFC: 2, TREELSTM: 5, TREEGRU: 7, MVRNN: 4, DAGRNN: 3,
             SIMPLETREEGRU: 7}
HEADER_FIELDS = ("status", "bad_node", "num_nodes", "num_levels", "num_leaves", "first_leaf",
                 "max_level_size", "num_roots")


class CxError(RuntimeError):
    def __init__(self, code, where, bad_node=-1):
        self.code, self.bad_node = code, bad_node
        super().__init__(f"{where}: {status_str(code)} (code {code}, node {bad_node})")


class _Lin(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in (
        "header", "perm", "inv", "children", "height", "level_begin", "level_size", "roots",
        "structure")] + [
        ("n", ctypes.c_int32), ("max_children", ctypes.c_int32), ("kind", ctypes.c_int32)]


class _Model(ctypes.Structure):
    _fields_ = [("cell", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("dtype", ctypes.c_int32)]


class _Weights(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p * 8)]


_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load (building first if stale) the in-tree libcx.so. Raises if absent."""
    global _lib
    with _lib_lock:
        if _lib is None:
            path = os.environ.get("CX_LIB")  # measurement variants (tools/build_variant.sh)
            if not path:
                path = _build.LIB
                if _build.stale():
                    path = _build.build()
            L = ctypes.CDLL(path)
            P, I, S = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
            L.cx_linearize_workspace_bytes.argtypes = [I, I]
            L.cx_linearize_workspace_bytes.restype = S
            L.cx_linearize.argtypes = [P, I, I, I, P, S, ctypes.POINTER(_Lin), P]
            L.cx_linearize.restype = ctypes.c_int
            L.cx_forward_workspace_bytes.argtypes = [ctypes.POINTER(_Model), I]
            L.cx_forward_workspace_bytes.restype = S
            L.cx_forward.argtypes = [ctypes.POINTER(_Model), ctypes.POINTER(_Weights), P, P,
                                     ctypes.POINTER(_Lin), P, P, P, P, S, P]
            L.cx_forward.restype = ctypes.c_int
            L.cx_linearize_forward_workspace_bytes.argtypes = [ctypes.POINTER(_Model), I, I]
            L.cx_linearize_forward_workspace_bytes.restype = S
            L.cx_linearize_forward.argtypes = [P, I, I, I, ctypes.POINTER(_Model),
                                               ctypes.POINTER(_Weights), P, P, ctypes.POINTER(_Lin),
                                               P, P, P, P, S, P]
            L.cx_linearize_forward.restype = ctypes.c_int
            L.cx_status_sync.argtypes = [ctypes.POINTER(_Lin), ctypes.POINTER(I), P]
            L.cx_status_sync.restype = ctypes.c_int
            L.cx_status_str.argtypes = [ctypes.c_int]
            L.cx_status_str.restype = ctypes.c_char_p
            L.cx_forward_launch_info.argtypes = [ctypes.POINTER(_Model), ctypes.POINTER(I),
                                                 ctypes.POINTER(I), ctypes.POINTER(I)]
            L.cx_forward_launch_info.restype = ctypes.c_int
            _lib = L
    return _lib


def status_str(code: int) -> str:
    return lib().cx_status_str(int(code)).decode()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class _WorkspaceCache:
    """Zero-filled workspaces, grown on demand, one per (device, stream, role).
    The kernels leave their synchronisation words zero, so a call with the same
    shape as the buffer's previous call needs no memset; the words' offsets
    depend on the shape (cx.h), so a buffer is zero-filled again, on the call's
    stream, whenever the shape key changes. Keyed by stream too: two streams
    never share grid-barrier words. A grown buffer never frees its predecessor:
    CUDA graphs captured earlier may still point at it (they stay valid for the
    life of the process). Pass an explicit `workspace=` to control the memory
    instead."""

    def __init__(self):
        self._bufs = {}
        self._shape = {}
        self._retired = []
        self._lock = threading.Lock()

    def get(self, device, role, nbytes, stream=None, shape=None):
        dev = torch.device(device)
        st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        key = (str(dev), int(st or 0), role)
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                if buf is not None:
                    self._retired.append(buf)
                buf = torch.zeros(max(nbytes, 1 << 12), dtype=torch.uint8, device=dev)
                self._bufs[key] = buf
            elif self._shape.get(key) != shape:
                # another shape: its synchronisation words sit elsewhere
                if stream is None:
                    buf.zero_()
                else:
                    with torch.cuda.stream(torch.cuda.ExternalStream(int(stream), device=dev)):
                        buf.zero_()
            self._shape[key] = shape
            return buf


_ws = _WorkspaceCache()


def _plan_env():
    """The debug / measurement variables that change which kernel (and so which
    workspace layout) a call uses; part of the workspace shape key."""
    return tuple(os.environ.get(k) for k in ("CX_FORWARD_PATH", "CX_FUSED", "CX_TC_F32_MIN_N", "CX_TC_HOIST",
                                             "CX_GRU_REFACTOR", "CX_UNROLL", "CX_PUSH"))


@dataclass
class Linearization:
    """Device tensors written by cx_linearize plus the C struct pointing at them."""
    header: torch.Tensor      # int32[10] (cx_lin_header, 40 bytes)
    perm: torch.Tensor
    inv: torch.Tensor
    children: torch.Tensor    # int32 [maxc, n]
    height: torch.Tensor
    level_begin: torch.Tensor
    level_size: torch.Tensor
    roots: torch.Tensor
    structure: torch.Tensor   # int32 [n]: index in roots of the owning root
    n: int
    max_children: int
    kind: int
    c: _Lin = None

    def header_dict(self):
        """Synchronising read of the header fields (host)."""
        h = self.header.cpu().tolist()
        return dict(zip(HEADER_FIELDS, h[:8]))


def alloc_linearization(n: int, max_children: int, kind: int, device) -> Linearization:
    """Allocate the output buffers of cx_linearize once (reusable via out=)."""
    size = max(n, 1)
    mk = lambda *s: torch.empty(*s, dtype=torch.int32, device=device)
    lin = Linearization(header=torch.zeros(10, dtype=torch.int32, device=device), perm=mk(size),
                        inv=mk(size), children=mk(max_children, size), height=mk(size),
                        level_begin=mk(size), level_size=mk(size), roots=mk(size),
                        structure=mk(size), n=n,
                        max_children=max_children, kind=kind)
    c = _Lin()
    for f in ("header", "perm", "inv", "children", "height", "level_begin", "level_size", "roots",
              "structure"):
        setattr(c, f, getattr(lin, f).data_ptr())
    lin.c = c
    lin.children = lin.children[:, :n]
    return lin


def linearize(children: torch.Tensor, kind: int, stream=None, workspace=None,
              out: Linearization = None) -> Linearization:
    """cx_linearize on an int32 [max_children, n] CUDA tensor of input ids.
    `out` (from alloc_linearization or a previous call) is reused without
    allocating, which also makes the call CUDA-graph capturable."""
    if children.dim() != 2 or children.dtype != torch.int32 or not children.is_cuda:
        raise ValueError("children must be an int32 CUDA tensor [max_children, n]")
    if not children.is_contiguous():
        children = children.contiguous()
    maxc, n = children.shape
    if out is None:
        out = alloc_linearization(n, maxc, kind, children.device)
    elif (out.n, out.max_children) != (n, maxc):
        raise ValueError("out was allocated for a different (n, max_children)")
    out.kind = kind
    L = lib()
    need = L.cx_linearize_workspace_bytes(n, maxc)
    ws = workspace if workspace is not None else _ws.get(children.device, "lin", need, None if stream is None else stream.cuda_stream,
                                                         shape=(n, maxc))
    st = L.cx_linearize(_ptr(children), n, maxc, kind, _ptr(ws), ws.numel(), ctypes.byref(out.c),
                        _stream(stream))
    if st != OK:
        raise CxError(st, "cx_linearize")
    return out


def check(lin: Linearization, stream=None):
    """cx_status_sync: synchronise and raise CxError if a data error was latched."""
    bad = ctypes.c_int32(-1)
    st = lib().cx_status_sync(ctypes.byref(lin.c), ctypes.byref(bad), _stream(stream))
    if st != OK:
        raise CxError(st, "device", bad.value)


def status(lin: Linearization, stream=None):
    bad = ctypes.c_int32(-1)
    st = lib().cx_status_sync(ctypes.byref(lin.c), ctypes.byref(bad), _stream(stream))
    return st, bad.value


def _model(cell, hidden, vocab, dtype):
    return _Model(cell=cell, hidden=hidden, vocab=vocab, dtype=dtype)


def launch_info(cell, hidden, vocab=1, dtype=F32):
    m = _model(cell, hidden, vocab, dtype)
    a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    st = lib().cx_forward_launch_info(ctypes.byref(m), ctypes.byref(a), ctypes.byref(b),
                                      ctypes.byref(c))
    if st != OK:
        raise CxError(st, "cx_forward_launch_info")
    return dict(ctas=a.value, threads=b.value, smem=c.value)


def _outputs(cell, hidden, n, dev, want_aux, num_roots, h_out, aux_out, root_out):
    if h_out is None:
        h_out = torch.empty(max(n, 1), hidden, dtype=torch.float32, device=dev)[:n]
    if want_aux and aux_out is None:
        if cell == TREELSTM:
            aux_out = torch.empty(n, hidden, dtype=torch.float32, device=dev)
        elif cell == MVRNN:
            aux_out = torch.empty(n, hidden, hidden, dtype=torch.float32, device=dev)
    if num_roots is not None and root_out is None:
        root_out = torch.empty(num_roots, hidden, dtype=torch.float32, device=dev)
    return h_out, aux_out, root_out


def _weights(cell, weights):
    ws_list = list(weights)
    if len(ws_list) != N_WEIGHTS[cell]:
        raise ValueError(f"cell {cell} takes {N_WEIGHTS[cell]} weight tensors")
    for t in ws_list:
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("weights must be contiguous fp32 CUDA tensors")
    w = _Weights()
    for i, t in enumerate(ws_list):
        w.p[i] = t.data_ptr()
    return w


def linearize_forward_launch_info(cell, hidden, n, max_children, vocab=1, dtype=F32):
    """The launch cx_linearize_forward makes for n nodes: fused flag and kernel shape."""
    L = lib()
    P = ctypes.POINTER(ctypes.c_int32)
    L.cx_linearize_forward_launch_info.argtypes = [ctypes.POINTER(_Model), ctypes.c_int32,
                                                   ctypes.c_int32, P, P, P, P, P]
    L.cx_linearize_forward_launch_info.restype = ctypes.c_int
    m = _model(cell, hidden, vocab, dtype)
    v = [ctypes.c_int32() for _ in range(5)]
    st = L.cx_linearize_forward_launch_info(ctypes.byref(m), n, max_children,
                                            *[ctypes.byref(x) for x in v])
    if st != OK:
        raise CxError(st, "cx_linearize_forward_launch_info")
    return dict(fused=bool(v[0].value), ctas=v[1].value, threads=v[2].value, smem=v[3].value,
                cluster=v[4].value)


def diag_sync_cycles(kind: int, levels: int, device=None) -> int:
    """SM cycles per level of a synchronisation / dependent-arithmetic step
    (cx_diag_sync_cycles: 0 push hand-off, 1 cluster barrier, 2 grid barrier,
    3 one level's dependent arithmetic). Synchronises the device."""
    L = lib()
    L.cx_diag_sync_cycles.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]
    L.cx_diag_sync_cycles.restype = ctypes.c_int
    dev = device or torch.device("cuda", torch.cuda.current_device())
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.zeros(32, dtype=torch.int32, device=dev)
    st = L.cx_diag_sync_cycles(kind, levels, ctypes.c_void_p(out.data_ptr()),
                               ctypes.c_void_p(ws.data_ptr()),
                               ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    if st != OK:
        raise CxError(st, "cx_diag_sync_cycles")
    torch.cuda.synchronize(dev)
    return int(out[0].item())


FAMILIES = {1: "smem", 2: "rw", 3: "cluster", 4: "big", 5: "mvrnn", 6: "tc", 7: "single",
            8: "tc32"}


def forward_family(cell, hidden, n, max_children, vocab=1, dtype=F32):
    """Name of the kernel family cx_forward runs for this shape (honours
    CX_FORWARD_PATH), or None."""
    L = lib()
    L.cx_debug_forward_family.argtypes = [ctypes.POINTER(_Model), ctypes.c_int32, ctypes.c_int32]
    L.cx_debug_forward_family.restype = ctypes.c_int32
    m = _model(cell, hidden, vocab, dtype)
    return FAMILIES.get(L.cx_debug_forward_family(ctypes.byref(m), n, max_children))


def fused_applies(cell, hidden, n, max_children, vocab=1, dtype=F32) -> bool:
    """Whether cx_linearize_forward runs as ONE launch for this shape (reporting)."""
    L = lib()
    L.cx_debug_fused_applies.argtypes = [ctypes.POINTER(_Model), ctypes.c_int32, ctypes.c_int32]
    L.cx_debug_fused_applies.restype = ctypes.c_int32
    m = _model(cell, hidden, vocab, dtype)
    return bool(L.cx_debug_fused_applies(ctypes.byref(m), n, max_children))


def linearize_forward(children: torch.Tensor, kind: int, cell: int, hidden: int, weights,
                      emb: torch.Tensor, word_ids: torch.Tensor, dtype: int = F32,
                      out: Linearization = None, want_aux: bool = False, num_roots=None,
                      h_out=None, aux_out=None, root_out=None, stream=None, workspace=None):
    """cx_linearize_forward: linearize + forward, one launch where the batch
    allows it. Returns (lin, h_out, aux or None, roots or None)."""
    if children.dim() != 2 or children.dtype != torch.int32 or not children.is_cuda:
        raise ValueError("children must be an int32 CUDA tensor [max_children, n]")
    if not children.is_contiguous():
        children = children.contiguous()
    maxc, n = children.shape
    dev = emb.device
    if out is None:
        out = alloc_linearization(n, maxc, kind, children.device)
    elif (out.n, out.max_children) != (n, maxc):
        raise ValueError("out was allocated for a different (n, max_children)")
    out.kind = kind
    w = _weights(cell, weights)
    h_out, aux_out, root_out = _outputs(cell, hidden, n, dev, want_aux, num_roots, h_out,
                                        aux_out, root_out)
    m = _model(cell, hidden, emb.shape[0], dtype)
    L = lib()
    need = L.cx_linearize_forward_workspace_bytes(ctypes.byref(m), n, maxc)
    ws = workspace if workspace is not None else _ws.get(dev, "linfwd", need, None if stream is None else stream.cuda_stream,
                                                         shape=(n, maxc, cell, hidden, emb.shape[0], dtype, _plan_env()))
    st = L.cx_linearize_forward(_ptr(children), n, maxc, kind, ctypes.byref(m), ctypes.byref(w),
                                _ptr(emb), _ptr(word_ids), ctypes.byref(out.c), _ptr(h_out),
                                _ptr(aux_out), _ptr(root_out), _ptr(ws), ws.numel(),
                                _stream(stream))
    if st != OK:
        raise CxError(st, "cx_linearize_forward")
    return out, h_out, aux_out, root_out


class LinearizeForwardPlan:
    """A prepared cx_linearize_forward call for repeated batches of one shape
    (serving): outputs, workspace and the marshalled C arguments are built
    once; each call() is a single C call on the same device buffers. The
    caller refreshes `children` / `word_ids` in place (e.g. an async H2D copy
    on `stream`) before calling. Same results as linearize_forward()."""

    def __init__(self, children: torch.Tensor, kind: int, cell: int, hidden: int, weights,
                 emb: torch.Tensor, word_ids: torch.Tensor, dtype: int = F32,
                 want_aux: bool = False, num_roots=None, stream=None):
        if children.dim() != 2 or children.dtype != torch.int32 or not children.is_cuda \
                or not children.is_contiguous():
            raise ValueError("children must be a contiguous int32 CUDA tensor [max_children, n]")
        maxc, n = children.shape
        dev = emb.device
        self.children, self.word_ids, self.emb = children, word_ids, emb
        self.weights = list(weights)  # keep the tensors alive
        self.lin = alloc_linearization(n, maxc, kind, children.device)
        self.lin.kind = kind
        self.h_out, self.aux_out, self.root_out = _outputs(cell, hidden, n, dev, want_aux,
                                                           num_roots, None, None, None)
        self._w = _weights(cell, self.weights)
        self._m = _model(cell, hidden, emb.shape[0], dtype)
        L = lib()
        need = L.cx_linearize_forward_workspace_bytes(ctypes.byref(self._m), n, maxc)
        self.workspace = torch.zeros(max(need, 1), dtype=torch.uint8, device=dev)
        self._fn = L.cx_linearize_forward
        self._args = (_ptr(children), n, maxc, kind, ctypes.byref(self._m), ctypes.byref(self._w),
                      _ptr(emb), _ptr(word_ids), ctypes.byref(self.lin.c), _ptr(self.h_out),
                      _ptr(self.aux_out), _ptr(self.root_out), _ptr(self.workspace),
                      self.workspace.numel(), _stream(stream))

    def __call__(self):
        st = self._fn(*self._args)
        if st != OK:
            raise CxError(st, "cx_linearize_forward")
        return self.h_out, self.aux_out, self.root_out


def forward(cell: int, hidden: int, weights, emb: torch.Tensor, word_ids: torch.Tensor,
            lin: Linearization, dtype: int = F32, want_aux: bool = False, num_roots=None,
            h_out=None, aux_out=None, root_out=None, stream=None, workspace=None):
    """cx_forward. Returns (h_out [n, H], aux or None, roots or None)."""
    dev = emb.device
    n = lin.n
    vocab = emb.shape[0]
    w = _weights(cell, weights)
    h_out, aux_out, root_out = _outputs(cell, hidden, n, dev, want_aux, num_roots, h_out,
                                        aux_out, root_out)
    m = _model(cell, hidden, vocab, dtype)
    L = lib()
    need = L.cx_forward_workspace_bytes(ctypes.byref(m), n)
    ws = workspace if workspace is not None else _ws.get(dev, "fwd", need, None if stream is None else stream.cuda_stream,
                                                         shape=(n, lin.max_children, cell, hidden, vocab, dtype, _plan_env()))
    st = L.cx_forward(ctypes.byref(m), ctypes.byref(w), _ptr(emb), _ptr(word_ids),
                      ctypes.byref(lin.c), _ptr(h_out), _ptr(aux_out), _ptr(root_out), _ptr(ws),
                      ws.numel(), _stream(stream))
    if st != OK:
        raise CxError(st, "cx_forward")
    return h_out, aux_out, root_out
