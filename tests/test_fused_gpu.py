"""cx_linearize_forward (linearizer fused into the forward
launch) vs the two separate calls and vs the oracle.

The fused kernel runs the same single-CTA linearizer and the same cluster
forward code, so its outputs must equal the two-call path bit for bit (every
cx_linearization array, the header, h / aux / roots), and the oracle within
the fp32 tolerance. Also: error latching (linearization errors win, forward
word errors are merged by the last CTA), workspace reuse after an error, the
two-launch fallback (batches / cells the fused kernel does not take) and CUDA
graph capture."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import (TOL_F32, assert_lin_equal, dev_f32, dev_i32, lin_to_numpy,
                         normwise_rel_err, weights_dev)

pytestmark = pytest.mark.gpu
T = synth


@pytest.fixture(scope="module")
def cx():
    import paper_2011_01383_b200 as m
    return m


def _case(cell, H, V, children, kind, seed, all_nodes=None):
    words = synth.word_ids(children, V, seed, all_nodes=(cell == T.DAGRNN) if all_nodes is None
                           else all_nodes)
    emb = synth.embedding(V, H, seed)
    ws_np, ws_dev = weights_dev(cell, H, V)
    return words, emb, ws_np, ws_dev


def _fused_vs_separate(cx, cell, H, V, children, kind, seed=0, monkeypatch=None, bitwise=True):
    words, emb, ws_np, ws_dev = _case(cell, H, V, children, kind, seed)
    ref_lin = oracle.linearize(children, kind)
    R = ref_lin["num_roots"]
    chd, wdd, embd = dev_i32(children), dev_i32(words), dev_f32(emb)
    lin_f, h_f, aux_f, r_f = cx.linearize_forward(chd, kind, cell, H, ws_dev, embd, wdd,
                                                  want_aux=True, num_roots=R)
    st_f = cx.status(lin_f)
    lin_s = cx.linearize(chd, kind)
    h_s, aux_s, r_s = cx.forward(cell, H, ws_dev, embd, wdd, lin_s, want_aux=True, num_roots=R)
    assert cx.status(lin_s) == st_f == (0, -1)
    # linearization: bit-exact vs the oracle and vs the separate kernel
    assert_lin_equal(lin_to_numpy(lin_f), ref_lin)
    assert_lin_equal(lin_to_numpy(lin_f), lin_to_numpy(lin_s))
    # forward: bit-exact vs the two-call path (same kernel family), within
    # tolerance of the oracle
    if bitwise:
        assert torch.equal(h_f, h_s)
    if aux_s is not None and bitwise:
        assert torch.equal(aux_f, aux_s)
    if bitwise:
        assert torch.equal(r_f, r_s)
    rst, rbad, rh, raux = oracle.forward(cell, H, V, ws_np, emb, words, children, want_aux=True)
    assert (rst, rbad) == (0, -1)
    e = normwise_rel_err(h_f.cpu().numpy(), rh)
    assert e <= TOL_F32, e
    if raux is not None and aux_f is not None:
        assert normwise_rel_err(aux_f.cpu().numpy(), raux) <= TOL_F32
    root_ids = ref_lin["perm"][ref_lin["roots"]]
    assert np.array_equal(r_f.cpu().numpy(), h_f.cpu().numpy()[root_ids])
    return e


@pytest.mark.parametrize("name", ["cfg2_treelstm_b10", "cfg2_treelstm_b1", "cfg5_dagrnn_b1",
                                  "cfg5_dagrnn_b10", "f4_lstm_seq100_b1"])
def test_baseline_configs_fused(cx, name):
    w = synth.workload(name)
    _fused_vs_separate(cx, w["cell"], w["hidden"], w["vocab"], w["children"], w["kind"],
                       seed=w["seed"])


@pytest.mark.parametrize("cell,H", [(T.TREELSTM, 64), (T.TREELSTM, 128), (T.TREELSTM, 256),
                                    (T.DAGRNN, 64), (T.DAGRNN, 256)])
def test_small_forests_fused(cx, cell, H):
    V = 50
    if cell == T.DAGRNN:
        ch, _ = synth.grid_dags(3, 5, 7)
        kind = T.DAG
    else:
        ch, _ = synth.sst_shaped_forest(12, 3, leaves=9)
        kind = T.TREE
    _fused_vs_separate(cx, cell, H, V, ch, kind, seed=3)


@pytest.mark.parametrize("maxc", [1, 3, 4])
def test_arity_fused(cx, maxc):
    """Random shuffled forests with up to `maxc` children, ragged sizes."""
    rng = np.random.default_rng(maxc)
    for trial in range(3):
        n = int(rng.integers(1, 300))
        ch = synth.random_forest(n, maxc, 100 * maxc + trial)
        ch, _, _ = synth.shuffle_ids(ch, None, trial)
        _fused_vs_separate(cx, T.TREELSTM, 64, 40, ch, T.TREE, seed=trial)


def test_shared_dag_one_cluster(cx):
    """DAG whose structures share nodes: the fused kernel falls back to one
    cluster for everything; roots still go to their own root_out rows."""
    # two roots (0, 1) sharing child 2; 2 -> 3, 4 leaves; 5 a separate leaf root
    ch = np.array([[2, 2, 3, -1, -1, -1], [-1, 4, 4, -1, -1, -1]], np.int32)
    _fused_vs_separate(cx, T.DAGRNN, 64, 10, ch, T.DAG, seed=1)


def test_single_nodes_and_all_leaves(cx):
    ch = np.full((2, 7), -1, np.int32)
    _fused_vs_separate(cx, T.TREELSTM, 64, 10, ch, T.TREE, seed=2)
    _fused_vs_separate(cx, T.DAGRNN, 64, 10, ch, T.DAG, seed=2)
    ch1 = np.full((2, 1), -1, np.int32)
    _fused_vs_separate(cx, T.TREELSTM, 256, 10, ch1, T.TREE, seed=2)


def test_fused_errors_and_reuse(cx):
    H, V = 64, 5
    emb = dev_f32(np.ones((V, H), np.float32))
    _, wd = weights_dev(T.TREELSTM, H, V)
    _, wdag = weights_dev(T.DAGRNN, H, V)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device="cuda")
    # word id out of range at leaves 1 and 2: the lowest node is latched
    ch = np.array([[1, -1, -1], [2, -1, -1]], np.int32)
    lin, _, _, _ = cx.linearize_forward(dev_i32(ch), T.TREE, T.TREELSTM, H, wd, emb,
                                        dev_i32([-1, 9, 7]), workspace=ws)
    assert cx.status(lin) == (7, 1)
    # the same workspace, a clean call: the header and the error word are reset
    lin, h, _, _ = cx.linearize_forward(dev_i32(ch), T.TREE, T.TREELSTM, H, wd, emb,
                                        dev_i32([-1, 1, 2]), workspace=ws)
    assert cx.status(lin) == (0, -1)
    assert lin.header_dict()["num_levels"] == 2
    # cycle: the linearization error wins, the forward part does not run
    ch = np.array([[1, 2, 1]], np.int32)
    lin, _, _, _ = cx.linearize_forward(dev_i32(ch), T.DAG, T.DAGRNN, H, wdag, emb,
                                        dev_i32([0, 9, 0]), workspace=ws)
    assert cx.status(lin) == (5, 0)
    # layout / kind errors, same as cx_linearize
    for chx, kind in ((np.array([[-1, -1, -1], [2, -1, -1]], np.int32), T.TREE),
                      (np.array([[2, 2, -1], [-1, -1, -1]], np.int32), T.TREE),
                      (np.array([[5, -1, -1]], np.int32), T.SEQUENCE)):
        lin, _, _, _ = cx.linearize_forward(dev_i32(chx), kind, T.TREELSTM, H, wd, emb,
                                            dev_i32([0, 0, 0]), workspace=ws)
        ref = oracle.linearize(chx, kind)
        assert cx.status(lin) == (ref["status"], ref["bad_node"])
    # and clean again
    lin, _, _, _ = cx.linearize_forward(dev_i32(ch * 0 - 1), T.DAG, T.DAGRNN, H, wdag, emb,
                                        dev_i32([0, 1, 2]), workspace=ws)
    assert cx.status(lin) == (0, -1)


@pytest.mark.parametrize("case", ["big_batch", "treegru", "bf16", "forced_off"])
def test_two_launch_fallback(cx, case, monkeypatch):
    """Where the fused kernel does not apply, cx_linearize_forward launches the
    two kernels; results equal the two separate calls."""
    dtype = cx.F32
    if case == "big_batch":
        ch, off = synth.sst_shaped_forest(40, 5, leaves=20)  # n > the fused limit
        cell, H, V, kind = T.TREELSTM, 256, 200, T.TREE
    elif case == "treegru":
        ch, off = synth.sst_shaped_forest(6, 5, leaves=9)
        cell, H, V, kind = T.TREEGRU, 64, 30, T.TREE
    elif case == "bf16":
        ch, off = synth.sst_shaped_forest(6, 5, leaves=9)
        cell, H, V, kind, dtype = T.TREELSTM, 256, 30, T.TREE, cx.BF16
    else:
        monkeypatch.setenv("CX_FUSED", "0")
        ch, off = synth.sst_shaped_forest(6, 5, leaves=9)
        cell, H, V, kind = T.TREELSTM, 64, 30, T.TREE
    words, emb, ws_np, ws_dev = _case(cell, H, V, ch, kind, 5)
    chd, wdd, embd = dev_i32(ch), dev_i32(words), dev_f32(emb)
    R = len(off) - 1
    lin_f, h_f, _, r_f = cx.linearize_forward(chd, kind, cell, H, ws_dev, embd, wdd, dtype=dtype,
                                              num_roots=R)
    lin_s = cx.linearize(chd, kind)
    h_s, _, r_s = cx.forward(cell, H, ws_dev, embd, wdd, lin_s, dtype=dtype, num_roots=R)
    assert cx.status(lin_f) == cx.status(lin_s) == (0, -1)
    assert_lin_equal(lin_to_numpy(lin_f), lin_to_numpy(lin_s))
    assert torch.equal(h_f, h_s)
    assert torch.equal(r_f, r_s)


def test_graph_capture(cx):
    """The fused call is capturable and replays to identical results."""
    w = synth.workload("cfg2_treelstm_b10")
    cell, H, V = w["cell"], w["hidden"], w["vocab"]
    words, emb, ws_np, ws_dev = _case(cell, H, V, w["children"], w["kind"], w["seed"])
    chd, wdd, embd = dev_i32(w["children"]), dev_i32(words), dev_f32(emb)
    lin, h, _, r = cx.linearize_forward(chd, w["kind"], cell, H, ws_dev, embd, wdd,
                                        num_roots=w["batch"])
    h0, r0 = h.clone(), r.clone()
    h.zero_()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        cx.linearize_forward(chd, w["kind"], cell, H, ws_dev, embd, wdd, out=lin, h_out=h,
                             root_out=r, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            cx.linearize_forward(chd, w["kind"], cell, H, ws_dev, embd, wdd, out=lin, h_out=h,
                                 root_out=r, stream=s)
    h.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(h, h0) and torch.equal(r, r0)
    assert cx.status(lin) == (0, -1)


@pytest.mark.parametrize("seed", range(12))
def test_fused_fuzz(cx, seed):
    """Random shuffled forests / DAGs / chains up to the fused size limit:
    linearization bit-exact vs the oracle, forward bit-exact vs the two calls."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 700))
    maxc = int(rng.integers(1, 5))
    shape = seed % 3
    if shape == 0:
        ch = synth.random_forest(n, maxc, seed)
        kind, cell = T.TREE, T.TREELSTM
    elif shape == 1:
        ch = synth.random_dag(min(n, 300), maxc, seed)
        kind, cell = T.DAG, T.DAGRNN
    else:
        ch, _ = synth.chains(1 + seed % 4, 1 + n // (1 + seed % 4))
        kind, cell = T.SEQUENCE, T.TREELSTM
    ch, _, _ = synth.shuffle_ids(ch, None, seed)
    H = (64, 128, 256)[seed % 3]
    words, emb, ws_np, ws_dev = _case(cell, H, 37, ch, kind, seed)
    chd, wdd, embd = dev_i32(ch), dev_i32(words), dev_f32(emb)
    ref = oracle.linearize(ch, kind)
    R = ref["num_roots"]
    lin_f, h_f, _, r_f = cx.linearize_forward(chd, kind, cell, H, ws_dev, embd, wdd, num_roots=R)
    assert cx.status(lin_f) == (0, -1)
    assert_lin_equal(lin_to_numpy(lin_f), ref)
    lin_s = cx.linearize(chd, kind)
    h_s, _, r_s = cx.forward(cell, H, ws_dev, embd, wdd, lin_s, num_roots=R)
    assert torch.equal(h_f, h_s) and torch.equal(r_f, r_s)


def test_plan_matches_call(cx):
    """LinearizeForwardPlan (prepared call) == linearize_forward, also after the
    input buffers are refreshed in place."""
    w = synth.workload("cfg2_treelstm_b10")
    cell, H, V = w["cell"], w["hidden"], w["vocab"]
    words, emb, ws_np, ws_dev = _case(cell, H, V, w["children"], w["kind"], w["seed"])
    chd, wdd, embd = dev_i32(w["children"]), dev_i32(words), dev_f32(emb)
    plan = cx.LinearizeForwardPlan(chd, w["kind"], cell, H, ws_dev, embd, wdd,
                                   num_roots=w["batch"])
    h, _, r = plan()
    lin2, h2, _, r2 = cx.linearize_forward(chd, w["kind"], cell, H, ws_dev, embd, wdd,
                                           num_roots=w["batch"])
    assert cx.status(plan.lin) == (0, -1)
    assert torch.equal(h, h2) and torch.equal(r, r2)
    words2 = synth.word_ids(w["children"], V, 99)
    wdd.copy_(dev_i32(words2))
    h, _, _ = plan()
    h3 = cx.linearize_forward(chd, w["kind"], cell, H, ws_dev, embd, dev_i32(words2))[1]
    assert torch.equal(h, h3) and not torch.equal(h3, h2)


# ---- single-CTA-per-structure one-launch path -------------
def _random_binary_dag(n, seed):
    """Every internal node has exactly 2 distinct children with smaller ids
    (shared children allowed): a TreeRNN-valid DAG."""
    rng = np.random.default_rng(seed)
    ch = -np.ones((2, n), np.int32)
    for v in range(n):
        if v >= 6 and rng.random() < 0.7:
            a, b = rng.choice(v, 2, replace=False)
            ch[0, v], ch[1, v] = a, b
    return ch


@pytest.mark.parametrize("unroll", ["1", "2"])
@pytest.mark.parametrize("name", ["cfg1_treernn", "tiny_treernn_forest", "tiny_treefc",
                                  "tiny_treernn_dag"])
def test_single_cta_path(cx, name, unroll, monkeypatch):
    """TreeRNN (unrolled by CX_UNROLL) and tiny TreeFC through the fused
    single-CTA kernel: one launch, linearization bit-exact, h vs the oracle
    and identical to the two separate calls."""
    monkeypatch.setenv("CX_UNROLL", unroll)
    if name == "cfg1_treernn":
        w = synth.workload(name)
        cell, H, V, ch, kind, seed = w["cell"], w["hidden"], w["vocab"], w["children"], w["kind"], w["seed"]
    elif name == "tiny_treernn_forest":
        ch, _ = synth.sst_shaped_forest(13, 3, leaves=9)
        cell, H, V, kind, seed = synth.TREERNN, 64, 50, synth.TREE, 3
    elif name == "tiny_treefc":
        ch, _ = synth.perfect_forest(4, 4)
        cell, H, V, kind, seed = synth.TREEFC, 64, 50, synth.TREE, 3
    else:
        ch = _random_binary_dag(60, 7)
        cell, H, V, kind, seed = synth.TREERNN, 16, 30, synth.DAG, 2
    assert cx.fused_applies(cell, H, ch.shape[1], ch.shape[0], V)
    info = cx.linearize_forward_launch_info(cell, H, ch.shape[1], ch.shape[0], V)
    assert info["fused"] and info["cluster"] == 1
    # TreeRNN: the same arithmetic as the separate kernel (bitwise); TreeFC's
    # dot products run in a different order than the register-weight kernel's
    _fused_vs_separate(cx, cell, H, V, ch, kind, seed=seed, bitwise=cell == T.TREERNN)
