"""CPU oracle for the Cortex hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
`--impl reference` legs may import this package. The product
(paper_2011_01383_b200/) never imports it, and it never imports the product.

The arithmetic lives in oracle.c (plain C99, fp64); this module only marshals
numpy arrays through ctypes. See oracle.h for the citations.

Parity status per function (every pin is a -m "not gpu" test):
  linearize        pinned: worked examples S:228/S:247 (tests/golden/worked_examples.json),
                   closed forms (perfect trees, grids, chains), brute force over all
                   labellings (N <= 6), invariants on fuzz cases
  forward, all 7 cells (TreeRNN, TreeFC, TreeLSTM, TreeGRU, SimpleTreeGRU, MV-RNN,
  DAG-RNN)         pinned by brute force: tests/golden/brute_force.json, written by
                   tools/gen_goldens.py in 50-digit mpmath from hand-typed inputs at
                   H = 1-2 on <= 7-node structures (asymmetric, non-identity matrices,
                   so the MV-RNN pairing [B a; A b] and the TreeGRU per-child reset gate
                   are distinguished from their alternatives)
  plus             S:471 worked example and the tanh(2t) closed form (TreeRNN); identity
                   reduction TreeFC == TreeRNN and MV-RNN == TreeFC; torch LSTMCell /
                   GRUCell / RNNCell on chains; W = U = 0 TreeLSTM closed form
The mutation check (tests/test_oracle_mutations.py) rebuilds oracle.c with each of 14
plausible bugs (-DCX_ORACLE_MUTATION=k) and asserts that some pin fails for every k.
Absolute agreement with Cortex's own trained models is unpinnable (the paper prints no
hidden-state values).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
# CX_ORACLE_MUTATION=k (mutation check only) builds a separate, deliberately broken library
_MUTATION = int(os.environ.get("CX_ORACLE_MUTATION", "0") or 0)
_LIB_PATH = os.path.join(_DIR, "liboracle.so" if not _MUTATION else f"liboracle_mut{_MUTATION}.so")
_SRC = [os.path.join(_DIR, "oracle.c"), os.path.join(_DIR, "oracle.h")]
_lock = threading.Lock()
_lib = None

OK, E_ARG, E_CHILD_RANGE, E_CHILD_LAYOUT, E_KIND, E_CYCLE, E_ARITY, E_WORD_RANGE = range(8)


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc -O2 (no -ffast-math, no SIMD intrinsics)."""
    stale = force or not os.path.exists(_LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB_PATH) for s in _SRC)
    if stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-Wall",
                               f"-DCX_ORACLE_MUTATION={_MUTATION}", "-o", tmp, _SRC[0], "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class LinHeader(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in (
        "status", "bad_node", "num_nodes", "num_levels", "num_leaves", "first_leaf",
        "max_level_size", "num_roots")]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            P = ctypes.c_void_p
            I = ctypes.c_int32
            lib.oracle_linearize.argtypes = [P, I, I, I, ctypes.POINTER(LinHeader)] + [P] * 8
            lib.oracle_linearize.restype = ctypes.c_int
            lib.oracle_forward.argtypes = [I, I, I, P, P, P, P, I, I, P, P, ctypes.POINTER(I)]
            lib.oracle_forward.restype = ctypes.c_int
            lib.oracle_forward_subset.argtypes = [I, I, I, P, P, P, P, I, I, P, I, P, P,
                                                  ctypes.POINTER(I)]
            lib.oracle_forward_subset.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def linearize(children, kind: int) -> dict:
    """Returns dict with header fields and arrays perm, inv, children, height,
    level_begin, level_size (trimmed to num_levels), roots (trimmed) and
    structure (per new id: index in roots of the owning root)."""
    lib = _load()
    ch = np.ascontiguousarray(children, dtype=np.int32)
    maxc, n = ch.shape
    size = max(n, 1)
    perm = np.zeros(size, np.int32)
    inv = np.zeros(size, np.int32)
    chn = np.zeros((maxc, size), np.int32)
    hgt = np.zeros(size, np.int32)
    lb = np.zeros(size, np.int32)
    ls = np.zeros(size, np.int32)
    roots = np.zeros(size, np.int32)
    struct = np.zeros(size, np.int32)
    hdr = LinHeader()
    lib.oracle_linearize(_ptr(ch), n, maxc, kind, ctypes.byref(hdr), _ptr(perm), _ptr(inv),
                         _ptr(chn), _ptr(hgt), _ptr(lb), _ptr(ls), _ptr(roots), _ptr(struct))
    out = {f: getattr(hdr, f) for f, _ in LinHeader._fields_}
    L, R = hdr.num_levels, hdr.num_roots
    out.update(perm=perm[:n], inv=inv[:n], children=chn[:, :n], height=hgt[:n],
               level_begin=lb[:L], level_size=ls[:L], roots=roots[:R], structure=struct[:n])
    return out


def forward(cell: int, hidden: int, vocab: int, weights, emb, words, children,
            want_aux: bool = False, targets=None):
    """Naive recursive forward in double. weights: list of float32 arrays in
    cx_weights order (or (name, array) pairs). Returns (status, bad_node,
    h[N,H] float64, aux or None). With `targets`, only nodes reachable from
    them are evaluated (other rows are NaN)."""
    lib = _load()
    ws = [np.ascontiguousarray(w[1] if isinstance(w, tuple) else w, dtype=np.float32)
          for w in weights]
    arr = (ctypes.c_void_p * max(len(ws), 1))(*[w.ctypes.data for w in ws])
    ch = np.ascontiguousarray(children, dtype=np.int32)
    maxc, n = ch.shape
    emb = np.ascontiguousarray(emb, dtype=np.float32)
    words = np.ascontiguousarray(words, dtype=np.int32)
    h = np.full((max(n, 1), hidden), np.nan)
    aux = None
    if want_aux:
        if cell == 2:
            aux = np.full((max(n, 1), hidden), np.nan)
        elif cell == 4:
            aux = np.full((max(n, 1), hidden, hidden), np.nan)
    bad = ctypes.c_int32(-1)
    if targets is None:
        st = lib.oracle_forward(cell, hidden, vocab, arr, _ptr(emb), _ptr(words), _ptr(ch), n,
                                maxc, _ptr(h), _ptr(aux), ctypes.byref(bad))
    else:
        t = np.ascontiguousarray(targets, dtype=np.int32)
        st = lib.oracle_forward_subset(cell, hidden, vocab, arr, _ptr(emb), _ptr(words),
                                       _ptr(ch), n, maxc, _ptr(t), len(t), _ptr(h), _ptr(aux),
                                       ctypes.byref(bad))
    return st, bad.value, h[:n], (aux[:n] if aux is not None else None)
