"""Pins for the oracle's forward pass (SURVEY.md §8(c) "Forward")."""
import json
import math
import os

import mpmath
import numpy as np
import pytest

import oracle
import synth
import torch_cells

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
T = synth


def _run(cell, H, V, ws, emb, words, ch, aux=False):
    st, bad, h, a = oracle.forward(cell, H, V, ws, emb, words, ch, want_aux=aux)
    assert st == 0, (st, bad)
    return (h, a) if aux else h


def _small_trees(seed, batch=3, leaves=5):
    ch, _ = synth.sst_shaped_forest(batch, seed, leaves)
    return ch


def test_treernn_worked_example():
    g = GOLD["treernn_three_node"]
    ch = np.array([[1, -1, -1], [2, -1, -1]], np.int32)
    h = _run(T.TREERNN, 2, 2, [], np.array(g["emb"], np.float32), np.array(g["words"]), ch)
    assert np.allclose(h[0], g["root"], atol=g["tol"])
    assert h[1].tolist() == [1.0, 2.0] and h[2].tolist() == [3.0, 4.0]
    # and against 30-digit tanh
    assert abs(h[0][0] - float(mpmath.tanh(4))) < 1e-15
    assert abs(h[0][1] - float(mpmath.tanh(6))) < 1e-15


def test_treernn_uniform_leaves_closed_form():
    """All leaves share one word: height-k nodes hold t_k = tanh(2 t_{k-1})."""
    w = synth.workload("cfg1_treernn")
    emb = synth.embedding(100, 8, 0)
    words = np.where(w["words"] >= 0, 7, -1).astype(np.int32)
    h = _run(T.TREERNN, 8, 100, [], emb, words, w["children"])
    lin = oracle.linearize(w["children"], T.TREE)
    t = [emb[7].astype(np.float64)]
    for k in range(1, 4):
        t.append(np.array([math.tanh(2 * x) for x in t[-1]]))
    hin = lin["height"][lin["inv"]]
    for v in range(15):
        assert np.array_equal(h[v], t[hin[v]])


def test_cfg1_anchor():
    w = synth.workload("cfg1_treernn")
    h = _run(T.TREERNN, 8, 100, [], synth.embedding(100, 8, 0), w["words"], w["children"])
    anchor = [0.181175638, 0.764987337, 0.319241104, -0.516140177,
              -0.316455034, -0.415677225, -0.372489589, 0.058719904]
    assert np.allclose(h[0], anchor, atol=5e-10)


def test_treefc_identity_reduces_to_treernn():
    H, V = 6, 30
    ch = _small_trees(3, batch=4, leaves=7)
    emb = synth.embedding(V, H, 3)
    words = synth.word_ids(ch, V, 3)
    W = np.hstack([np.eye(H), np.eye(H)]).astype(np.float32)
    hfc = _run(T.TREEFC, H, V, [W, np.zeros(H, np.float32)], emb, words, ch)
    hrnn = _run(T.TREERNN, H, V, [], emb, words, ch)
    assert np.array_equal(hfc, hrnn)  # bitwise


def test_treefc_left_projection_library():
    """W = [P 0]: h_root = tanh(P h_left + b) with numpy matmul (catches a
    transposed W or swapped children)."""
    H, V = 5, 10
    rng = np.random.default_rng(0)
    P = rng.uniform(-1, 1, (H, H)).astype(np.float32)
    b = rng.uniform(-1, 1, H).astype(np.float32)
    W = np.hstack([P, np.zeros((H, H), np.float32)])
    ch = np.array([[1, -1, -1], [2, -1, -1]], np.int32)
    emb = rng.uniform(-1, 1, (V, H)).astype(np.float32)
    words = np.array([-1, 3, 8], np.int32)
    h = _run(T.TREEFC, H, V, [W, b], emb, words, ch)
    ref = np.tanh(P.astype(np.float64) @ emb[3].astype(np.float64) + b)
    assert np.allclose(h[0], ref, rtol=0, atol=1e-14)


def test_mvrnn_identity_reduces_to_treefc():
    H, V = 4, 12
    ch = _small_trees(5, batch=3, leaves=6)
    ws = dict(synth.weights(T.MVRNN, H, V, seed=7))
    emb = synth.embedding(V, H, 5)
    words = synth.word_ids(ch, V, 5)
    Mw = np.broadcast_to(np.eye(H, dtype=np.float32), (V, H, H)).copy()
    WM = np.hstack([0.5 * np.eye(H), 0.5 * np.eye(H)]).astype(np.float32)
    h_mv, A = _run(T.MVRNN, H, V, [Mw, ws["W"], ws["beta"], WM], emb, words, ch, aux=True)
    h_fc = _run(T.TREEFC, H, V, [ws["W"], ws["beta"]], emb, words, ch)
    assert np.array_equal(h_mv, h_fc)
    assert np.array_equal(A, np.broadcast_to(np.eye(H), A.shape))


def test_mvrnn_matrix_path_library():
    """Per-node matrices != I: compare with numpy matmul composition, plus
    W_M = [I 0] keeps the leftmost leaf's matrix exactly."""
    H, V = 5, 20
    ch = _small_trees(11, batch=2, leaves=6)
    ws = synth.weights(T.MVRNN, H, V, seed=3)
    emb = synth.embedding(V, H, 11)
    words = synth.word_ids(ch, V, 11)
    arrs = [w for _, w in ws]
    h, A = _run(T.MVRNN, H, V, arrs, emb, words, ch, aux=True)
    ra, rA = torch_cells.mvrnn(arrs, emb, words, ch)
    assert np.allclose(h, ra, rtol=0, atol=1e-13)
    assert np.allclose(A, rA, rtol=0, atol=1e-13)
    WM = np.hstack([np.eye(H), np.zeros((H, H))]).astype(np.float32)
    h2, A2 = _run(T.MVRNN, H, V, [arrs[0], arrs[1], arrs[2], WM], emb, words, ch, aux=True)
    # root 0's leftmost leaf: follow children[0]
    v = 0
    while ch[0, v] != -1:
        v = ch[0, v]
    assert np.array_equal(A2[0], arrs[0][words[v]].astype(np.float64))


def test_treelstm_chain_is_lstmcell():
    """On chains (kind=sequence) TreeLSTM == torch.nn.LSTMCell."""
    H, V = 8, 50
    ch, _ = synth.chains(2, 12)
    ws = [w for _, w in synth.weights(T.TREELSTM, H, V)]
    emb = synth.embedding(V, H, 1)
    words = synth.word_ids(ch, V, 1)
    h, c = _run(T.TREELSTM, H, V, ws, emb, words, ch, aux=True)
    rh, rc = torch_cells.treelstm(ws, emb, words, ch)
    assert np.allclose(h, rh, rtol=0, atol=1e-14) and np.allclose(c, rc, rtol=0, atol=1e-14)


def test_treelstm_trees_lstmcell_composition():
    H, V = 6, 40
    ch = _small_trees(2, batch=3, leaves=9)
    ws = [w for _, w in synth.weights(T.TREELSTM, H, V)]
    emb = synth.embedding(V, H, 2)
    words = synth.word_ids(ch, V, 2)
    h, c = _run(T.TREELSTM, H, V, ws, emb, words, ch, aux=True)
    rh, rc = torch_cells.treelstm(ws, emb, words, ch)
    assert np.allclose(h, rh, rtol=0, atol=1e-13) and np.allclose(c, rc, rtol=0, atol=1e-13)


def test_treelstm_zero_weights_closed_form():
    """W = U = 0 on a perfect tree: c_k = alpha sum_{j<=k} (2 beta)^j,
    h_k = sigma(b_o) tanh(c_k), alpha = s(b_i) tanh(b_u), beta = s(b_f)."""
    H, V = 3, 5
    ch, _ = synth.perfect_forest(1, 4)
    z = np.zeros((3 * H, H), np.float32)
    b_iou = np.array([0.3, -0.2, 0.1, 0.5, -0.4, 0.25, -0.6, 0.7, 0.05], np.float32)
    b_f = np.array([0.2, -0.1, 0.4], np.float32)
    ws = [z, z, b_iou, np.zeros((H, H), np.float32), b_f]
    emb = synth.embedding(V, H, 0)
    words = synth.word_ids(ch, V, 0)
    h, c = _run(T.TREELSTM, H, V, ws, emb, words, ch, aux=True)
    s = lambda x: 1.0 / (1.0 + math.exp(-x))
    lin = oracle.linearize(ch, T.TREE)
    hin = lin["height"][lin["inv"]]
    for v in range(ch.shape[1]):
        k = hin[v]
        for i in range(H):
            alpha = s(float(b_iou[i])) * math.tanh(float(b_iou[2 * H + i]))
            beta = s(float(b_f[i]))
            ck = alpha * sum((2 * beta) ** j for j in range(k + 1))
            assert abs(c[v, i] - ck) < 1e-13
            assert abs(h[v, i] - s(float(b_iou[H + i])) * math.tanh(ck)) < 1e-13


def test_treegru_chain_is_grucell():
    """Chain with U_r = 0, b_r = 100 (r == 1): TreeGRU == torch.nn.GRUCell."""
    H, V = 8, 50
    ch, _ = synth.chains(2, 10)
    ws = [w for _, w in synth.weights(T.TREEGRU, H, V)]
    ws[2] = np.zeros((H, H), np.float32)
    ws[5] = np.full(H, 100.0, np.float32)
    emb = synth.embedding(V, H, 4)
    words = synth.word_ids(ch, V, 4)
    h = _run(T.TREEGRU, H, V, ws, emb, words, ch)
    import torch
    cell = torch.nn.GRUCell(H, H, dtype=torch.float64)
    W_zh, U_z, _, U_h, b_z, _, b_h = [torch.tensor(w, dtype=torch.float64) for w in ws]
    zz = torch.zeros(H, H, dtype=torch.float64)
    with torch.no_grad():
        cell.weight_ih.copy_(torch.cat([zz, W_zh[:H], W_zh[H:]]))
        cell.weight_hh.copy_(torch.cat([zz, U_z, U_h]))
        cell.bias_ih.copy_(torch.cat([torch.full((H,), 100.0, dtype=torch.float64), b_z, b_h]))
        cell.bias_hh.zero_()
        for b in range(2):
            base = b * 10
            hs = torch.zeros(1, H, dtype=torch.float64)
            for t in range(9, -1, -1):  # leaf is the last node of the chain
                x = torch.tensor(emb[words[base + t]], dtype=torch.float64)[None] if t == 9 \
                    else torch.zeros(1, H, dtype=torch.float64)
                hs = cell(x, hs)
                assert np.allclose(h[base + t], hs[0].numpy(), rtol=0, atol=1e-14)


def test_treegru_trees_grucell_composition():
    H, V = 6, 40
    ch = _small_trees(9, batch=3, leaves=8)
    ws = [w for _, w in synth.weights(T.TREEGRU, H, V)]
    emb = synth.embedding(V, H, 9)
    words = synth.word_ids(ch, V, 9)
    h = _run(T.TREEGRU, H, V, ws, emb, words, ch)
    assert np.allclose(h, torch_cells.treegru(ws, emb, words, ch), rtol=0, atol=1e-13)


def test_dagrnn_chain_is_rnncell_and_grid_composition():
    H, V = 8, 30
    for rows, cols in ((1, 9), (4, 5)):
        ch, _ = synth.grid_dags(2, rows, cols)
        ws = [w for _, w in synth.weights(T.DAGRNN, H, V)]
        emb = synth.embedding(V, H, 6)
        words = synth.word_ids(ch, V, 6, all_nodes=True)
        h = _run(T.DAGRNN, H, V, ws, emb, words, ch)
        assert np.allclose(h, torch_cells.dagrnn(ws, emb, words, ch), rtol=0, atol=1e-13)


@pytest.mark.parametrize("cell", range(6))
def test_all_zero_is_zero(cell):
    H, V = 4, 6
    ch = _small_trees(1, batch=2, leaves=5) if cell != T.DAGRNN else synth.grid_dags(1, 3, 3)[0]
    ws = [np.zeros_like(w) for _, w in synth.weights(cell, H, V)]
    emb = np.zeros((V, H), np.float32)
    words = synth.word_ids(ch, V, 0, all_nodes=True)
    h = _run(cell, H, V, ws, emb, words, ch)
    assert (h == 0).all()


def test_shared_dag_child_computed_once():
    """both parents read the same state of a shared child."""
    H, V = 4, 9
    ch = np.array([[1, 3, 3, -1], [2, -1, -1, -1]], np.int32)  # 1 and 2 share child 3
    ws = [w for _, w in synth.weights(T.DAGRNN, H, V)]
    emb = synth.embedding(V, H, 0)
    words = np.array([1, 2, 2, 5], np.int32)
    h = _run(T.DAGRNN, H, V, ws, emb, words, ch)
    assert np.array_equal(h[1], h[2])


def test_forward_errors():
    H, V = 2, 3
    emb = np.ones((V, H), np.float32)
    # binary cell, a node with one child -> ARITY at that node
    ch = np.array([[1, 2, -1], [-1, -1, -1]], np.int32)
    st, bad, _, _ = oracle.forward(T.TREERNN, H, V, [], emb, np.array([-1, -1, 0]), ch)
    assert (st, bad) == (oracle.E_ARITY, 0)
    # word out of range at a leaf
    ch = np.array([[1, -1, -1], [2, -1, -1]], np.int32)
    st, bad, _, _ = oracle.forward(T.TREERNN, H, V, [], emb, np.array([-1, 7, 0]), ch)
    assert (st, bad) == (oracle.E_WORD_RANGE, 1)
    # internal word ids are ignored by tree cells, required by DAG-RNN
    ws = [w for _, w in synth.weights(T.DAGRNN, H, V)]
    st, bad, _, _ = oracle.forward(T.DAGRNN, H, V, ws, emb, np.array([-1, 1, 0]), ch)
    assert (st, bad) == (oracle.E_WORD_RANGE, 0)
    # ARITY (6) ranks below WORD_RANGE (7)
    ch = np.array([[1, 2, -1, -1], [3, -1, -1, -1]], np.int32)
    st, bad, _, _ = oracle.forward(T.TREERNN, H, V, [], emb, np.array([-1, -1, 9, 0]), ch)
    assert (st, bad) == (oracle.E_ARITY, 1)
