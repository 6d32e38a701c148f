"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every symbol include/cx.h declares, and rejects bad arguments synchronously
(before any CUDA call, so these run without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cxmod():
    import paper_2011_01383_b200 as cx
    cx.lib()
    return cx


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cx_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(cxmod):
    names = declared_functions()
    assert len(names) == 16
    L = cxmod.lib()
    for name in names:
        assert hasattr(L, name), name


def test_every_exported_symbol_is_declared(cxmod):
    import subprocess
    from paper_2011_01383_b200 import _build
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True,
                         text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines()
                       if ln.split() and ln.split()[-1].startswith("cx_")})
    assert exported == declared_functions()


def test_built_for_sm100a(cxmod):
    import subprocess
    from paper_2011_01383_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(cxmod):
    assert cxmod.status_str(0) == "ok"
    assert "cycle" in cxmod.status_str(5)


def _lin_struct(cx, n=4, maxc=2, null_header=False):
    c = cx._cx._Lin()
    for i, f in enumerate(("header", "perm", "inv", "children", "height", "level_begin",
                           "level_size", "roots", "structure")):
        setattr(c, f, 0 if (null_header and f == "header") else 0x1000 + 64 * i)
    return c


def test_linearize_argument_errors(cxmod):
    L = cxmod.lib()
    c = _lin_struct(cxmod)
    ws = ctypes.c_void_p(0x100000)
    big = 1 << 30
    dummy = ctypes.c_void_p(0x2000)
    # sequence needs max_children == 1
    assert L.cx_linearize(dummy, 4, 2, cxmod.SEQUENCE, ws, big, ctypes.byref(c), None) == 1
    # bad kind, n < 0, max_children < 1, null output
    assert L.cx_linearize(dummy, 4, 2, 7, ws, big, ctypes.byref(c), None) == 1
    assert L.cx_linearize(dummy, -1, 2, cxmod.TREE, ws, big, ctypes.byref(c), None) == 1
    assert L.cx_linearize(dummy, 4, 0, cxmod.TREE, ws, big, ctypes.byref(c), None) == 1
    assert L.cx_linearize(dummy, 4, 2, cxmod.TREE, ws, big, None, None) == 1
    assert L.cx_linearize(None, 4, 2, cxmod.TREE, ws, big, ctypes.byref(c), None) == 1
    c2 = _lin_struct(cxmod, null_header=True)
    assert L.cx_linearize(dummy, 4, 2, cxmod.TREE, ws, big, ctypes.byref(c2), None) == 1
    # workspace too small
    need = L.cx_linearize_workspace_bytes(4, 2)
    assert need > 0
    assert L.cx_linearize(dummy, 4, 2, cxmod.TREE, ws, need - 1, ctypes.byref(c), None) == 9


def test_forward_argument_errors(cxmod):
    L = cxmod.lib()
    _cx = cxmod._cx
    c = _lin_struct(cxmod)
    c.n, c.max_children, c.kind = 4, 2, cxmod.TREE
    w = _cx._Weights()
    for i in range(8):
        w.p[i] = 0x3000 + 64 * i
    d = ctypes.c_void_p(0x4000)
    ws = ctypes.c_void_p(0x100000)
    m = _cx._Model(cell=cxmod.TREELSTM, hidden=256, vocab=10, dtype=cxmod.F32)
    need = L.cx_forward_workspace_bytes(ctypes.byref(m), 4)
    # bad cell / dtype enums
    bad = _cx._Model(cell=9, hidden=256, vocab=10, dtype=0)
    assert L.cx_forward(ctypes.byref(bad), ctypes.byref(w), d, d, ctypes.byref(c), d, None, None,
                        ws, need, None) == 1
    bad = _cx._Model(cell=2, hidden=256, vocab=10, dtype=5)
    assert L.cx_forward(ctypes.byref(bad), ctypes.byref(w), d, d, ctypes.byref(c), d, None, None,
                        ws, need, None) == 1
    # missing weight pointer
    w2 = _cx._Weights()
    assert L.cx_forward(ctypes.byref(m), ctypes.byref(w2), d, d, ctypes.byref(c), d, None, None,
                        ws, need, None) == 1
    # null h_out
    assert L.cx_forward(ctypes.byref(m), ctypes.byref(w), d, d, ctypes.byref(c), None, None, None,
                        ws, need, None) == 1
    # small workspace
    assert L.cx_forward(ctypes.byref(m), ctypes.byref(w), d, d, ctypes.byref(c), d, None, None,
                        ws, need - 1, None) == 9


def test_binding_refuses_cpu_tensors(cxmod):
    import torch
    with pytest.raises(ValueError):
        cxmod.linearize(torch.zeros((2, 3), dtype=torch.int32), cxmod.TREE)
