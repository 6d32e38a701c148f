"""TreeGRU and SimpleTreeGRU (SimpleTreeGRU = footnote
P:1638-1640, reading Q24) under both schedules of the register-weight kernel:
the original (phase A: U_z h~ and U_r h_k; phase B: U_h s) and the recursive
refactoring of §3.1 (m_k = sigma(U_r h_k + b_r) h_k moved into the
child's step). Every case against the fp64 oracle at the fp32 tolerance."""
import numpy as np
import pytest

import synth
from gpu_helpers import TOL_F32, normwise_rel_err, run_both, weights_dev

pytestmark = pytest.mark.gpu
T = synth


@pytest.fixture(params=["original", "refactored"])
def schedule(request, monkeypatch):
    monkeypatch.setenv("CX_GRU_REFACTOR", "1" if request.param == "refactored" else "0")
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    return request.param


def _parity(cell, H, V, ch, kind, seed, wcell=None):
    words = synth.word_ids(ch, V, seed)
    emb = synth.embedding(V, H, seed)
    ws_np, ws_dev = weights_dev(cell if wcell is None else wcell, H, V)
    import oracle
    R = oracle.linearize(ch, kind)["num_roots"]
    lin, (st, bad), h, _, roots, (rst, rbad), rh, _ = run_both(
        cell, H, V, ch, kind, words, emb, ws_np, ws_dev, num_roots=R)
    assert (st, bad) == (rst, rbad) == (0, -1)
    e = normwise_rel_err(h.cpu().numpy(), rh)
    assert e <= TOL_F32, f"max normwise rel err {e:.3e}"
    return h.cpu().numpy()


@pytest.mark.parametrize("cell", [T.TREEGRU, T.SIMPLETREEGRU])
@pytest.mark.parametrize("H", [64, 256, 512])
def test_small_forests(cell, H, schedule):
    ch, _ = synth.sst_shaped_forest(7, 5, leaves=13)
    _parity(cell, H, 97, ch, T.TREE, seed=5)


@pytest.mark.parametrize("cell", [T.TREEGRU, T.SIMPLETREEGRU])
def test_general_arity_and_chains(cell, schedule):
    ch = synth.random_forest(150, 4, 11)
    _parity(cell, 64, 50, ch, T.TREE, seed=2)
    ch, _ = synth.chains(5, 40)
    _parity(cell, 64, 30, ch, T.SEQUENCE, seed=4)


@pytest.mark.parametrize("name", ["cfg3_treegru_b1", "cfg3_treegru_b10", "f4_gru_seq100_b10"])
@pytest.mark.parametrize("cell", [T.TREEGRU, T.SIMPLETREEGRU])
def test_configs(name, cell, schedule):
    w = synth.workload(name)
    _parity(cell, w["hidden"], w["vocab"], w["children"], w["kind"], seed=w["seed"])


def test_schedules_agree(monkeypatch):
    """Both schedules compute the same cell: results within rounding."""
    w = synth.workload("cfg3_treegru_b10")
    out = {}
    for sched in ("0", "1"):
        monkeypatch.setenv("CX_GRU_REFACTOR", sched)
        out[sched] = _parity(T.TREEGRU, w["hidden"], w["vocab"], w["children"], w["kind"],
                             seed=w["seed"])
    d = np.abs(out["0"] - out["1"]).max()
    assert d < 1e-4, d


def test_simple_differs_from_treegru():
    """SimpleTreeGRU drops z * h~ at internal nodes: leaves agree, internal nodes differ."""
    w = synth.workload("cfg3_treegru_b1")
    H, V, ch = 64, w["vocab"], w["children"]
    a = _parity(T.TREEGRU, H, V, ch, w["kind"], seed=w["seed"])
    b = _parity(T.SIMPLETREEGRU, H, V, ch, w["kind"], seed=w["seed"], wcell=T.TREEGRU)
    leaf = ch[0] < 0
    assert np.array_equal(a[leaf], b[leaf])
    assert np.abs(a[~leaf] - b[~leaf]).max() > 1e-3
