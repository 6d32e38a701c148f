"""cx_linearize (CUDA) vs oracle.linearize: bit-exact on every output."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cx():
    import paper_2011_01383_b200 as m
    return m


def _check(cx, ch, kind):
    from gpu_helpers import assert_lin_equal, dev_i32, lin_to_numpy
    lin = cx.linearize(dev_i32(ch), kind)
    dev = lin_to_numpy(lin)
    ref = oracle.linearize(ch, kind)
    assert_lin_equal(dev, ref)
    return dev


def test_worked_examples(cx):
    _check(cx, np.array([[1, -1, -1], [2, -1, -1]]), synth.TREE)
    _check(cx, np.array([[1, 2, -1, -1, 5, -1, -1], [4, 3, -1, -1, 6, -1, -1]]), synth.TREE)


def test_empty_and_single(cx):
    d = _check(cx, np.zeros((2, 0), np.int32), synth.TREE)
    assert d["num_levels"] == 0
    d = _check(cx, np.full((2, 1), -1, np.int32), synth.TREE)
    assert d["num_levels"] == 1 and d["first_leaf"] == 0


def test_fuzz_1000(cx):
    """>= 1000 random trees, forests, DAGs, chains (<= 200 nodes, ids shuffled)."""
    count = 0
    for seed in range(1000):
        n = 1 + (seed * 37) % 200
        r = seed % 4
        if r == 0:
            ch, kind = synth.random_dag(n, 1 + seed % 4, seed, p_edge=0.3), synth.DAG
        elif r == 3:
            ch, kind = synth.chains(1 + seed % 3, 1 + n // 3)[0], synth.SEQUENCE
        else:
            ch, kind = synth.random_forest(n, 1 + seed % 3, seed), synth.TREE
        if seed % 2:
            ch, _, _ = synth.shuffle_ids(ch, None, seed)
        _check(cx, ch, kind)
        count += 1
    assert count == 1000


@pytest.mark.parametrize("name", ["cfg1_treernn", "cfg2_treelstm_b10", "cfg3_treefc_b10",
                                  "cfg5_dagrnn_b10", "cfg5_treelstm_b4096",
                                  "cfg5_dagrnn_b4096"])
def test_baseline_configs(cx, name):
    w = synth.workload(name)
    _check(cx, w["children"], w["kind"])


def test_large_shuffled_forest(cx):
    ch, _ = synth.sst_shaped_forest(600, 3)
    ch, _, _ = synth.shuffle_ids(ch, None, 3)
    _check(cx, ch, synth.TREE)


@pytest.mark.parametrize("length,batch", [(10000, 1), (300, 40), (2500, 8)])
def test_long_chains(cx, length, batch):
    ch, _ = synth.chains(batch, length)
    _check(cx, ch, synth.SEQUENCE)


def test_error_cases_bit_exact(cx):
    T, D, S = synth.TREE, synth.DAG, synth.SEQUENCE
    cases = [
        ([[1, 5, -1], [2, -1, -1]], T), ([[-7, -1]], S), ([[-1, -1, -1], [1, -1, -1]], T),
        ([[2, 2, -1], [-1, -1, -1]], T), ([[2, 2, -1], [-1, -1, -1]], D),
        ([[1, -1], [1, -1]], D), ([[1, 2, 1]], D), ([[-1, 2, 1]], D), ([[0]], D),
        ([[-1, -1, 9], [1, -1, -1]], D), ([[1, 2, 1], [-1, -1, -1]], T),
    ]
    for ch, kind in cases:
        _check(cx, np.array(ch, np.int32), kind)
    # a large graph with a cycle deep inside (multi-CTA path)
    ch, _ = synth.grid_dags(200, 10, 10)
    ch = ch.copy()
    ch[1, 12345] = 12399  # (123, 4, 5) -> (123, 9, 9): creates a cycle through the grid
    _check(cx, ch, D)
    # a large tree with two parents somewhere
    ch2, _ = synth.sst_shaped_forest(400, 1)
    ch2 = ch2.copy()
    ch2[0, 9000] = 1  # node 1 (left child of root 0) gets a second parent
    _check(cx, ch2, T)


@pytest.mark.parametrize("batch", [15, 40, 60, 80, 100, 120])
def test_mid_size_forests(cx, batch):
    """Forests of 585..4680 nodes: the single-CTA linearizer with several
    nodes per thread (a leaf-start race in its walk-up once produced wrong
    heights here: pending counts were used to pick the start nodes while other
    walkers decremented them)."""
    for seed in range(3):
        ch, _ = synth.sst_shaped_forest(batch, seed)
        _check(cx, ch, synth.TREE)
        ch2, _, _ = synth.shuffle_ids(ch, None, seed + 10)
        _check(cx, ch2, synth.TREE)


@pytest.mark.parametrize("n", [600, 1500, 3000, 4700])
@pytest.mark.parametrize("maxc", [1, 2, 3, 4])
def test_mid_size_random(cx, n, maxc):
    ch = synth.random_forest(n, maxc, n + maxc)
    _check(cx, ch, synth.TREE)
    if 4 * n < 12000:
        _check(cx, synth.random_dag(n, maxc, n + maxc, p_edge=0.4), synth.DAG)


def test_tree_cycles_multi_cta(cx):
    """Tree-kind inputs with a cycle at multi-CTA size (n > 4.8k): a root made
    the child of one of its own leaves (walks from hanging leaves enter the
    cycle) and a leafless 3-ring appended to a valid forest; status and the
    lowest cycle node must match the oracle."""
    ch, off = synth.sst_shaped_forest(300, 5)
    n = ch.shape[1]
    c1 = ch.copy()
    r = int(off[137])                       # a root
    leaf = next(v for v in range(int(off[137]), int(off[138])) if c1[0, v] == -1)
    c1[0, leaf] = r                         # leaf -> root: a cycle through the tree
    _check(cx, c1, synth.TREE)
    c2 = np.full((2, n + 3), -1, np.int32)
    c2[:, :n] = ch
    c2[0, n], c2[0, n + 1], c2[0, n + 2] = n + 1, n + 2, n  # ring without leaves
    _check(cx, c2, synth.TREE)


@pytest.mark.parametrize("spine,shuffle", [(6000, False), (6000, True), (40000, False)])
def test_deep_caterpillar_multi_cta(cx, spine, shuffle):
    """Caterpillar trees (every spine node has one leaf child and the next
    spine node as children) far deeper than the walk limit, above the
    single-CTA size: the multi-CTA heights pass must be O(n) (pending-count
    peeling) and the structure pass pointer-jumps. Bit-exact
    vs the oracle, plus a short caterpillar forest next to it."""
    n = 2 * spine + 1
    ch = np.full((2, n), -1, np.int32)
    for i in range(spine):  # spine node 2i: children (2i + 1 = leaf, 2i + 2 = next spine)
        ch[0, 2 * i], ch[1, 2 * i] = 2 * i + 1, 2 * i + 2
    extra, _ = synth.sst_shaped_forest(20, 9)
    full = np.concatenate([ch, np.where(extra >= 0, extra + n, -1).astype(np.int32)], axis=1)
    if shuffle:
        full, _, _ = synth.shuffle_ids(full, None, 5)
    _check(cx, full, synth.TREE)


def test_tiny_fuzz_warp_path(cx):
    """n <= 32 (the one-warp linearizer, lin_warp.cuh): 1,500 random trees,
    forests, DAGs, chains with shuffled ids, plus corrupted inputs of every
    error kind -- bit-exact vs the oracle, errors included."""
    rng = np.random.default_rng(7)
    for seed in range(1500):
        n = 1 + seed % 32
        r = seed % 5
        maxc = 1 + seed % 4
        if r == 0:
            ch, kind = synth.random_dag(n, maxc, seed, p_edge=0.4), synth.DAG
        elif r == 1:
            ch, kind = synth.chains(1 + seed % 3, 1 + (n - 1) // 3)[0], synth.SEQUENCE
        else:
            ch, kind = synth.random_forest(n, maxc, seed), synth.TREE
        if seed % 2:
            ch, _, _ = synth.shuffle_ids(ch, None, seed)
        ch = np.ascontiguousarray(ch, dtype=np.int32)
        if seed % 7 == 3 and ch.size:  # corrupt: out of range, layout, duplicate, cycle
            ch = ch.copy()
            m, n2 = ch.shape
            v = int(rng.integers(n2))
            kk = int(rng.integers(m))
            op = (seed // 7) % 4
            if op == 0:
                ch[kk, v] = n2 + 3
            elif op == 1 and m > 1:
                ch[0, v], ch[m - 1, v] = -1, int(rng.integers(n2))
            elif op == 2 and m > 1:
                ch[0, v] = ch[1, v] = int(rng.integers(n2))
            else:
                ch[kk, v] = v  # self edge: a cycle
        _check(cx, ch, kind)
