"""cx_forward with dtype = CX_F32 on the split-fp32 tensor-core kernel
(forward_tc.cu, SP = 2: every operand split into bf16 hi + lo, products
A_hi B_hi + A_hi B_lo + A_lo B_hi with fp32 accumulation in TMEM) vs the fp64
oracle at the fp32 tolerance: max per-node normwise relative error <= 1e-4
(BASELINE.json north_star). Forced with CX_FORWARD_PATH=tc at every size
(inputs spanning several 128-node tiles per CTA with ragged tails, both
input-row modes, sequences, child-sum arity 1..2, the BASELINE.json configs
the kernel covers); the automatic dispatch (large batches, per-cell thresholds) at the
full batch-4096 configs, sampled; a TreeLSTM DAG linearization stays on FMA."""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import dev_f32, dev_i32, normwise_rel_err, weights_dev

pytestmark = pytest.mark.gpu
T = synth
TOL_F32 = 1e-4


@pytest.fixture(scope="module")
def cx():
    import paper_2011_01383_b200 as m
    return m


@pytest.fixture
def forced(monkeypatch):
    monkeypatch.setenv("CX_FORWARD_PATH", "tc")


def _run(cx, cell, H, V, ch, kind, words, emb, want_aux=False, num_roots=None):
    _, wd = weights_dev(cell, H, V)
    lin = cx.linearize(dev_i32(ch), kind)
    h, aux, roots = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(words), lin, dtype=cx.F32,
                               want_aux=want_aux, num_roots=num_roots)
    return lin, h, aux, roots


def _parity(cx, cell, H, V, ch, kind, seed=0, want_aux=True):
    assert cx.forward_family(cell, H, ch.shape[1], ch.shape[0], V) == "tc32"
    words = synth.word_ids(ch, V, seed, all_nodes=(cell == T.DAGRNN))
    emb = synth.embedding(V, H, seed)
    ref_lin = oracle.linearize(ch, kind)
    R = ref_lin["num_roots"]
    lin, h, aux, roots = _run(cx, cell, H, V, ch, kind, words, emb, want_aux, R)
    assert cx.status(lin) == (0, -1)
    ws_np, _ = weights_dev(cell, H, V)
    rst, _, rh, raux = oracle.forward(cell, H, V, ws_np, emb, words, ch, want_aux=want_aux)
    assert rst == 0
    e = normwise_rel_err(h.cpu().numpy(), rh)
    assert e <= TOL_F32, f"h max normwise rel err {e:.3e}"
    if want_aux and raux is not None and aux is not None:
        ea = normwise_rel_err(aux.cpu().numpy(), raux)
        assert ea <= TOL_F32, f"aux err {ea:.3e}"
    root_ids = ref_lin["perm"][ref_lin["roots"]]
    assert np.array_equal(roots.cpu().numpy(), h.cpu().numpy()[root_ids])
    return e


@pytest.mark.parametrize("H", [128, 256])
@pytest.mark.parametrize("V", [97, 50000])  # table mode (hoisted leaves) / node-order mode
def test_treelstm_multitile(cx, forced, H, V):
    ch, _ = synth.sst_shaped_forest(300 if H == 128 else 120, 3)
    _parity(cx, T.TREELSTM, H, V, ch, T.TREE, seed=3)


@pytest.mark.parametrize("H", [128, 256])
@pytest.mark.parametrize("V", [97, 50000])
def test_dagrnn_multitile(cx, forced, H, V):
    ch, _ = synth.grid_dags(40, 9, 11)
    _parity(cx, T.DAGRNN, H, V, ch, T.DAG, seed=4)


@pytest.mark.parametrize("H", [256, 512])
def test_treefc_perfect(cx, forced, H):
    ch, _ = synth.perfect_forest(12, 7)
    _parity(cx, T.TREEFC, H, 20000, ch, T.TREE, seed=1)


def test_treefc_sst_ragged(cx, forced):
    ch, _ = synth.sst_shaped_forest(150, 6, leaves=17)
    _parity(cx, T.TREEFC, 256, 333, ch, T.TREE, seed=6)


@pytest.mark.parametrize("cell", [T.TREELSTM, T.DAGRNN])
def test_sequences(cx, forced, cell):
    ch, _ = synth.chains(300, 37)
    _parity(cx, cell, 128, 64, ch, T.SEQUENCE, seed=8)


@pytest.mark.parametrize("cell", [T.TREELSTM, T.DAGRNN])
def test_child_sum_arity_1_and_2(cx, forced, cell):
    if cell == T.DAGRNN:
        ch, kind = synth.random_dag(3000, 2, 11, p_edge=0.6), T.DAG
    else:
        ch, kind = synth.random_forest(4000, 2, 11), T.TREE
    _parity(cx, cell, 128, 500, ch, kind, seed=2)


@pytest.mark.parametrize("name", ["cfg2_treelstm_b10", "cfg2_treelstm_b1", "cfg3_treefc_b1",
                                  "cfg3_treefc_b10", "cfg5_dagrnn_b1", "cfg5_dagrnn_b10",
                                  "f4_lstm_seq100_b10"])
def test_baseline_configs(cx, forced, name):
    w = synth.workload(name)
    _parity(cx, w["cell"], w["hidden"], w["vocab"], w["children"], w["kind"], seed=w["seed"])


def test_treefc_b10_automatic(cx, monkeypatch):
    """TreeFC batch 10 (2,550 nodes) takes the split-fp32 kernel by default."""
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    w = synth.workload("cfg3_treefc_b10")
    _parity(cx, w["cell"], w["hidden"], w["vocab"], w["children"], w["kind"], seed=w["seed"])


def test_treelstm_dag_stays_on_fma(cx, monkeypatch):
    """A TreeLSTM over a DAG linearization (a child shared by two parents) is
    not run on the tensor-core kernel (it hands each h to ONE parent slot): the
    automatic dispatch keeps it on an FMA kernel, with fp32 parity."""
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    ch = synth.random_dag(3000, 2, 5, p_edge=0.6)
    H, V = 128, 500
    words = synth.word_ids(ch, V, 5)
    emb = synth.embedding(V, H, 5)
    lin, h, _, _ = _run(cx, T.TREELSTM, H, V, ch, T.DAG, words, emb)
    assert cx.status(lin) == (0, -1)
    ws_np, _ = weights_dev(T.TREELSTM, H, V)
    rst, _, rh, _ = oracle.forward(T.TREELSTM, H, V, ws_np, emb, words, ch)
    assert rst == 0
    assert normwise_rel_err(h.cpu().numpy(), rh) <= TOL_F32


@pytest.mark.parametrize("name", ["cfg5_treelstm_b4096", "cfg5_dagrnn_b4096"])
def test_batch4096_sampled(cx, name, monkeypatch):
    """The bench launch (full batch, fp32, automatic dispatch) checked on 64
    sampled structures."""
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    w = synth.workload(name)
    ch, cell, H, V = w["children"], w["cell"], w["hidden"], w["vocab"]
    assert cx.forward_family(cell, H, ch.shape[1], ch.shape[0], V) == "tc32"
    words, emb = w["words"], synth.embedding(V, H, w["seed"])
    lin, h, _, roots = _run(cx, cell, H, V, ch, w["kind"], words, emb, num_roots=w["batch"])
    assert cx.status(lin) == (0, -1)
    off = w["offsets"]
    picks = np.sort(np.random.default_rng(2).choice(w["batch"], 64, replace=False))
    targets = off[picks] if w["kind"] == T.TREE else off[picks + 1] - 1
    ws_np, _ = weights_dev(cell, H, V)
    rst, _, rh, _ = oracle.forward(cell, H, V, ws_np, emb, words, ch, targets=targets)
    assert rst == 0
    rows = np.concatenate([np.arange(off[g], off[g + 1]) for g in picks])
    e = normwise_rel_err(h.cpu().numpy(), rh, rows=rows)
    assert e <= TOL_F32, e
    assert np.array_equal(roots.cpu().numpy()[picks], h.cpu().numpy()[targets])


def test_errors(cx, forced):
    """Latched data errors on the split-fp32 kernel: the lowest (code, node)
    wins, as on every other path (word range in table mode -- hoisted leaves /
    hoisted DAG projection -- and in node-order mode; TreeFC arity)."""
    H, V = 128, 5
    emb = np.ones((50, H), np.float32)
    ch = np.array([[1, -1, -1], [2, -1, -1]], np.int32)
    for Vx in (V, 50):
        lin, _, _, _ = _run(cx, T.TREELSTM, H, Vx, ch, T.TREE, np.array([-1, 70, 0]), emb[:Vx])
        assert cx.status(lin) == (7, 1)
        lin, _, _, _ = _run(cx, T.DAGRNN, H, Vx, ch, T.DAG, np.array([90, 0, 0]), emb[:Vx])
        assert cx.status(lin) == (7, 0)
    ch = np.array([[1, 2, -1], [-1, -1, -1]], np.int32)
    lin, _, _, _ = _run(cx, T.TREEFC, 256, V, ch, T.TREE, np.array([-1, -1, 0]),
                        np.ones((V, 256), np.float32))
    assert cx.status(lin) == (6, 0)


def test_single_nodes(cx, forced):
    """One-node structures only: every node is a leaf and a root (no level
    beyond 0; hoisted tables in table mode)."""
    ch = np.full((2, 300), -1, np.int32)
    _parity(cx, T.TREELSTM, 128, 50, ch, T.TREE, seed=1)
    _parity(cx, T.DAGRNN, 128, 50, ch, T.DAG, seed=1)
    _parity(cx, T.TREEFC, 256, 50, ch, T.TREE, seed=1)


def test_dag_slots_reused_workspace(cx, forced):
    """DAG-RNN on parent-slot operands: a second call of the same shape whose
    DAG has fewer edges reuses the workspace (no re-zeroing for an unchanged
    shape); the slot rows of now-absent children must read as zeros. Also a
    DAG with a third parent for some node (the cp.async gather fallback)."""
    ch, _ = synth.grid_dags(40, 9, 11)
    _parity(cx, T.DAGRNN, 128, 97, ch, T.DAG, seed=4)
    ch2 = ch.copy()
    rng = np.random.default_rng(5)
    two = np.where(ch2[1] >= 0)[0]
    ch2[1, rng.choice(two, len(two) // 3, replace=False)] = -1  # drop some second children
    _parity(cx, T.DAGRNN, 128, 97, ch2, T.DAG, seed=4)
    ch3 = ch.copy()
    ch3[1, 50] = ch3[0, 1]  # ... gives node ch[0, 1] extra parents (in-degree 3)
    if ch3[1, 50] != ch3[0, 50] and ch3[1, 50] >= 0 and ch[0, 50] >= 0:
        _parity(cx, T.DAGRNN, 128, 97, ch3, T.DAG, seed=4)
