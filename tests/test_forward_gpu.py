"""cx_forward (CUDA, fp32) vs the fp64 oracle: max per-node normwise relative
error <= 1e-4 (BASELINE.json north_star), on small multi-tile/ragged inputs
and at every BASELINE.json configuration (sampled at batch 4096)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import (TOL_F32, dev_f32, dev_i32, normwise_rel_err, run_both, weights_dev)

pytestmark = pytest.mark.gpu
T = synth


@pytest.fixture(scope="module")
def cx():
    import paper_2011_01383_b200 as m
    return m


@pytest.fixture(params=["auto", "rw", "smem", "cluster", "big"])
def path(request, monkeypatch):
    """Run a test through each forward kernel family (CX_FORWARD_PATH is read
    by libcx on every cx_forward call)."""
    if request.param == "auto":
        monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    else:
        monkeypatch.setenv("CX_FORWARD_PATH", request.param)
    return request.param


def _parity(cell, hidden, vocab, children, kind, seed=0, want_aux=False, all_words=None,
            check_roots=True):
    import os
    import paper_2011_01383_b200 as cx
    forced = os.environ.get("CX_FORWARD_PATH")
    if forced:
        # the forced family must be the one that runs (fwd_plan falls back to
        # another family for shapes the forced one does not instantiate): skip
        # such cases instead of testing a different kernel under this ID; the
        # automatic path is covered by the "auto" parameter
        fam = cx.forward_family(cell, hidden, children.shape[1], children.shape[0], vocab)
        if fam != forced:
            pytest.skip(f"forced {forced} does not instantiate this shape (runs {fam})")
    words = synth.word_ids(children, vocab, seed, all_nodes=(cell == T.DAGRNN))
    emb = synth.embedding(vocab, hidden, seed)
    ws_np, ws_dev = weights_dev(cell, hidden, vocab)
    ref_lin = oracle.linearize(children, kind)
    R = ref_lin["num_roots"]
    lin, (st, bad), h, aux, roots, (rst, rbad), rh, raux = run_both(
        cell, hidden, vocab, children, kind, words, emb, ws_np, ws_dev, want_aux=want_aux,
        num_roots=R if check_roots else None)
    assert (st, bad) == (rst, rbad) == (0, -1)
    e = normwise_rel_err(h.cpu().numpy(), rh)
    assert e <= TOL_F32, f"h max normwise rel err {e:.3e}"
    if want_aux and raux is not None:
        ea = normwise_rel_err(aux.cpu().numpy(), raux)
        assert ea <= TOL_F32, f"aux err {ea:.3e}"
    if check_roots:
        # packed roots == h rows of the in-degree-0 nodes in ascending input id
        root_ids = ref_lin["perm"][ref_lin["roots"]]
        assert np.array_equal(roots.cpu().numpy(), h.cpu().numpy()[root_ids])
    return e


SMALL = [  # (cell, H) at sizes that still span several tiles and node groups
    (T.TREERNN, 8), (T.TREERNN, 64), (T.TREEFC, 64), (T.TREELSTM, 64), (T.TREEGRU, 64),
    (T.MVRNN, 16), (T.MVRNN, 64), (T.DAGRNN, 64), (T.TREELSTM, 32), (T.TREEGRU, 96),
    (T.TREELSTM, 128), (T.TREEGRU, 512), (T.TREEFC, 512), (T.DAGRNN, 512), (T.TREELSTM, 512),
]


@pytest.mark.parametrize("cell,H", SMALL)
def test_small_forests(cx, cell, H, path):
    V = 97
    if cell == T.DAGRNN:
        ch, _ = synth.grid_dags(3, 5, 7)
        kind = T.DAG
    else:
        ch, _ = synth.sst_shaped_forest(7, 5, leaves=13)
        kind = T.TREE
    _parity(cell, H, V, ch, kind, seed=5, want_aux=True)


@pytest.mark.parametrize("cell", [T.TREELSTM, T.TREEGRU, T.DAGRNN])
def test_child_sum_general_arity(cx, cell, path):
    """Child-sum cells on nodes with 0..4 children (random DAG / forest)."""
    H, V = 64, 50
    if cell == T.DAGRNN:
        ch, kind = synth.random_dag(120, 4, 11, p_edge=0.6), T.DAG
    else:
        ch, kind = synth.random_forest(150, 4, 11), T.TREE
    _parity(cell, H, V, ch, kind, seed=2, want_aux=True)


@pytest.mark.parametrize("cell", [T.TREELSTM, T.TREEGRU, T.DAGRNN])
def test_sequences(cx, cell):
    H, V = 64, 30
    ch, _ = synth.chains(5, 40)
    _parity(cell, H, V, ch, T.SEQUENCE, seed=4, want_aux=True)


@pytest.mark.parametrize("name", ["cfg1_treernn", "cfg2_treelstm_b10", "cfg2_treelstm_b1",
                                  "cfg3_treegru_b1", "cfg3_treegru_b10", "cfg3_treefc_b1",
                                  "cfg3_treefc_b10", "cfg4_mvrnn_b10", "cfg5_dagrnn_b1",
                                  "cfg5_dagrnn_b10", "f4_lstm_seq100_b1", "f4_lstm_seq100_b10",
                                  "f4_gru_seq100_b1", "f4_gru_seq100_b10"])
def test_baseline_configs(cx, name, path):
    w = synth.workload(name)
    _parity(w["cell"], w["hidden"], w["vocab"], w["children"], w["kind"], seed=w["seed"],
            want_aux=True)


@pytest.mark.parametrize("name", ["cfg5_treelstm_b4096", "cfg5_dagrnn_b4096"])
@pytest.mark.parametrize("fpath", ["auto", "smem", "big"])
def test_batch4096_sampled(cx, name, fpath, monkeypatch):
    """Full-size launch (the bench configuration); oracle on 64 sampled
    structures (their roots and everything below them)."""
    if fpath == "auto":
        monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    else:
        monkeypatch.setenv("CX_FORWARD_PATH", fpath)
    w = synth.workload(name)
    ch, cell, H, V = w["children"], w["cell"], w["hidden"], w["vocab"]
    # automatic: the split-fp32 tensor-core kernel (test_forward_tc32_gpu.py)
    assert cx.forward_family(cell, H, ch.shape[1], ch.shape[0], V) == ("tc32" if fpath == "auto"
                                                                       else fpath)
    words, emb = w["words"], synth.embedding(V, H, w["seed"])
    ws_np, ws_dev = weights_dev(cell, H, V)
    lin = cx.linearize(dev_i32(ch), w["kind"])
    h, _, roots = cx.forward(cell, H, ws_dev, dev_f32(emb), dev_i32(words), lin,
                             num_roots=w["batch"])
    assert cx.status(lin) == (0, -1)
    off = w["offsets"]
    rng = np.random.default_rng(0)
    picks = np.sort(rng.choice(w["batch"], 64, replace=False))
    # the root of structure g: tree root = first node (pre-order); grid = last cell
    targets = off[picks] if w["kind"] == T.TREE else off[picks + 1] - 1
    rst, _, rh, _ = oracle.forward(cell, H, V, ws_np, emb, words, ch, targets=targets)
    assert rst == 0
    rows = np.concatenate([np.arange(off[g], off[g + 1]) for g in picks])
    e = normwise_rel_err(h.cpu().numpy(), rh, rows=rows)
    assert e <= TOL_F32, e
    # packed roots: structure g's root row
    hr = h.cpu().numpy()
    rt = roots.cpu().numpy()
    assert np.array_equal(rt[picks], hr[targets])


def test_permutation_and_batch_invariance(cx, path):
    """Relabelling permutes outputs identically; a tree alone == the tree in a
    forest (bitwise: per-node arithmetic does not depend on level size)."""
    H, V = 64, 40
    cell = T.TREELSTM
    ch, off = synth.sst_shaped_forest(9, 7, leaves=11)
    words = synth.word_ids(ch, V, 7)
    emb = synth.embedding(V, H, 7)
    _, wd = weights_dev(cell, H, V)
    lin = cx.linearize(dev_i32(ch), T.TREE)
    h = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(words), lin)[0].cpu().numpy()
    ch2, w2, pi = synth.shuffle_ids(ch, words, 7)
    lin2 = cx.linearize(dev_i32(ch2), T.TREE)
    h2 = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(w2), lin2)[0].cpu().numpy()
    assert np.array_equal(h2[pi], h)
    # tree 3 alone
    a, b = off[3], off[4]
    sub = ch[:, a:b].copy()
    sub[sub >= 0] -= a
    lin3 = cx.linearize(dev_i32(sub), T.TREE)
    h3 = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(words[a:b]), lin3)[0].cpu().numpy()
    assert np.array_equal(h3, h[a:b])


def test_forward_errors(cx):
    H, V = 32, 5
    emb = dev_f32(np.ones((V, H), np.float32))
    # binary cell, internal node with one child -> ARITY at the node (input id)
    ch = np.array([[1, 2, -1], [-1, -1, -1]], np.int32)
    lin = cx.linearize(dev_i32(ch), T.TREE)
    cx.forward(T.TREERNN, H, [], emb, dev_i32([-1, -1, 0]), lin)
    assert cx.status(lin) == (6, 0)
    # word id out of range at leaf 1
    ch = np.array([[1, -1, -1], [2, -1, -1]], np.int32)
    lin = cx.linearize(dev_i32(ch), T.TREE)
    _, wd = weights_dev(T.TREELSTM, H, V)
    cx.forward(T.TREELSTM, H, wd, emb, dev_i32([-1, 7, 0]), lin)
    assert cx.status(lin) == (7, 1)
    # a linearization error is kept; forward does not run
    ch = np.array([[1, 2, 1]], np.int32)
    lin = cx.linearize(dev_i32(ch), T.DAG)
    h, _, _ = cx.forward(T.DAGRNN, H, weights_dev(T.DAGRNN, H, V)[1], emb, dev_i32([0, 0, 0]), lin)
    assert cx.status(lin) == (5, 0)
    # unsupported H
    ch = np.array([[1, -1, -1], [2, -1, -1]], np.int32)
    lin = cx.linearize(dev_i32(ch), T.TREE)
    with pytest.raises(cx.CxError):
        cx.forward(T.TREELSTM, 48, weights_dev(T.TREELSTM, 48, V)[1],
                   dev_f32(np.ones((V, 48), np.float32)), dev_i32([-1, 0, 0]), lin)


def test_all_leaves_and_single_node(cx):
    H, V = 64, 10
    for cell in (T.TREELSTM, T.TREERNN, T.DAGRNN, T.MVRNN):
        Hc = 64
        ch = np.full((2, 5), -1, np.int32)  # five single-node trees
        _parity(cell, Hc, V, ch, T.TREE if cell != T.DAGRNN else T.DAG, seed=1, want_aux=True)


@pytest.mark.parametrize("name,family", [("cfg1_treernn", "smem"), ("cfg2_treelstm_b10", "cluster"),
                                         ("cfg3_treegru_b10", "rw"), ("cfg3_treefc_b10", "tc32"),
                                         ("cfg4_mvrnn_b10", "mvrnn"), ("cfg5_dagrnn_b10", "cluster"),
                                         ("cfg5_treelstm_b4096", "tc32"), ("cfg5_dagrnn_b4096", "tc32")])
def test_automatic_family(cx, name, family, monkeypatch):
    """The automatic plan (cx_forward, fp32) runs the documented kernel family
    for every BASELINE configuration."""
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    w = synth.workload(name)
    ch = w["children"]
    assert cx.forward_family(w["cell"], w["hidden"], ch.shape[1], ch.shape[0], w["vocab"]) == family
