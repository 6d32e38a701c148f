"""Seeded synthetic inputs for the Cortex hot path (SURVEY.md §8(d) "Generator specification").

This module is shared by the oracle (`oracle/`) and the CUDA path
(`paper_2011_01383_b200/`). It holds none of the method's arithmetic: it only
draws structures (child-index arrays), word ids, embedding tables and weights
from counter-based splitmix64 streams, so both sides receive bit-identical
inputs.

Conventions:
  * one splitmix64 stream per purpose, initial state (purpose << 32) | seed;
    purposes: 1 structure, 2 word ids, 3 Emb, 4 weights, 5 MV-RNN Mw;
  * u01 = (z >> 40) * 2^-24; randint(n) = ((z >> 32) * n) >> 32;
    U(a, b) = fp32(a + (b - a) * u01) computed in double;
  * structures are numbered per-structure pre-order (a parser's order),
    structures concatenated; children SoA [max_children][N], -1 = absent.

The paper's workloads (Table 2): perfect binary trees of
height 7 (TreeFC), synthetic 10x10 DAGs (DAG-RNN), Stanford Sentiment Treebank
parse trees (TreeLSTM/TreeGRU/MV-RNN; replaced by "SST-shaped" random binary
trees with 20 leaves because the dataset is not available).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
MASK64 = (1 << 64) - 1

P_STRUCT, P_WORDS, P_EMB, P_WEIGHTS, P_MW = 1, 2, 3, 4, 5

# cell ids, identical to cx_cell in include/cx.h
TREERNN, TREEFC, TREELSTM, TREEGRU, MVRNN, DAGRNN, SIMPLETREEGRU = range(7)
CELL_NAMES = {TREERNN: "treernn", TREEFC: "treefc", TREELSTM: "treelstm",
              TREEGRU: "treegru", MVRNN: "mvrnn", DAGRNN: "dagrnn",
              SIMPLETREEGRU: "simpletreegru"}
# structure kinds, identical to cx_kind
SEQUENCE, TREE, DAG = 0, 1, 2


class SplitMix64:
    """Counter-based splitmix64: output i is mix(state0 + (i+1)*GOLDEN)."""

    def __init__(self, purpose: int, seed: int):
        self.x = ((purpose << 32) | (seed & 0xFFFFFFFF)) & MASK64

    # -- scalar draws (used for structures, small and sequential) ---------
    def next(self) -> int:
        self.x = (self.x + 0x9E3779B97F4A7C15) & MASK64
        z = self.x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def randint(self, n: int) -> int:
        return ((self.next() >> 32) * n) >> 32

    # -- vectorised draws (numpy uint64 arithmetic wraps mod 2^64) --------
    def next_array(self, count: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            i = np.arange(1, count + 1, dtype=np.uint64)
            z = np.uint64(self.x) + i * GOLDEN
            self.x = (self.x + count * 0x9E3779B97F4A7C15) & MASK64
            z = (z ^ (z >> np.uint64(30))) * M1
            z = (z ^ (z >> np.uint64(27))) * M2
            return z ^ (z >> np.uint64(31))

    def uniform_array(self, count: int, a: float, b: float) -> np.ndarray:
        z = self.next_array(count)
        u01 = (z >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)
        return (a + (b - a) * u01).astype(np.float32)

    def randint_array(self, count: int, n: int) -> np.ndarray:
        z = self.next_array(count)
        return (((z >> np.uint64(32)) * np.uint64(n)) >> np.uint64(32)).astype(np.int64)


# ---------------------------------------------------------------------------
# Structures. Each builder returns children as int32 [max_children, N].
# ---------------------------------------------------------------------------

def sst_shaped_forest(batch: int, seed: int = 0, leaves: int = 20):
    """`batch` SST-shaped binary trees of `leaves` leaves each.

    A span of l > 1 leaves splits as k = 1 + randint(l - 1) leaves on the left.
    Ids are assigned in pre-order on entry; the split is drawn on entry too.
    Returns (children[2, N], is_leaf[N], tree_offsets[batch + 1]).
    """
    rng = SplitMix64(P_STRUCT, seed)
    left, right = [], []
    offsets = [0]

    for _ in range(batch):
        # explicit stack of (span, parent id, slot) to avoid Python recursion
        stack = [(leaves, -1, 0)]
        while stack:
            span, parent, slot = stack.pop()
            nid = len(left)
            left.append(-1)
            right.append(-1)
            if parent >= 0:
                (left if slot == 0 else right)[parent] = nid
            if span > 1:
                k = 1 + rng.randint(span - 1)
                # push right first so the left subtree is numbered first
                stack.append((span - k, nid, 1))
                stack.append((k, nid, 0))
        offsets.append(len(left))
    ch = np.array([left, right], dtype=np.int32)
    return ch, np.array(offsets, dtype=np.int64)


def perfect_forest(batch: int, height: int):
    """`batch` perfect binary trees whose root has height `height` (Q11):
    2^(height+1) - 1 nodes each, pre-order ids."""
    n_tree = (1 << (height + 1)) - 1
    left = np.full(batch * n_tree, -1, dtype=np.int32)
    right = np.full(batch * n_tree, -1, dtype=np.int32)
    offsets = [0]
    for b in range(batch):
        base = b * n_tree
        nid = [base]

        def build(h):
            me = nid[0]
            nid[0] += 1
            if h > 0:
                left[me] = build(h - 1)
                right[me] = build(h - 1)
            return me

        build(height)
        offsets.append(base + n_tree)
    return np.stack([left, right]), np.array(offsets, dtype=np.int64)


def grid_dags(batch: int, rows: int = 10, cols: int = 10):
    """`batch` rows x cols grid DAGs (Q12, Q22). Node (g, i, j) has id
    g*rows*cols + i*cols + j and depends on (i-1, j) and (i, j-1), packed
    as a prefix [up?, left?]."""
    n_g = rows * cols
    ch = np.full((2, batch * n_g), -1, dtype=np.int32)
    for g in range(batch):
        for i in range(rows):
            for j in range(cols):
                me = g * n_g + i * cols + j
                slot = 0
                if i > 0:
                    ch[slot, me] = me - cols
                    slot += 1
                if j > 0:
                    ch[slot, me] = me - 1
                    slot += 1
    offsets = np.arange(batch + 1, dtype=np.int64) * n_g
    return ch, offsets


def chains(batch: int, length: int):
    """`batch` sequences of `length` nodes; node 0 of each chain is its last
    element (the root) and node length-1 its first (the leaf)."""
    n = batch * length
    ch = np.full((1, n), -1, dtype=np.int32)
    for b in range(batch):
        base = b * length
        for t in range(length - 1):
            ch[0, base + t] = base + t + 1
    offsets = np.arange(batch + 1, dtype=np.int64) * length
    return ch, offsets


def random_dag(n: int, max_children: int, seed: int, p_edge: float = 0.5):
    """Small random DAG for fuzzing: child ids are always larger than the
    parent id before shuffling, so it is acyclic; children form a prefix."""
    rng = SplitMix64(P_STRUCT, seed)
    ch = np.full((max_children, n), -1, dtype=np.int32)
    for v in range(n):
        cands = list(range(v + 1, n))
        slot = 0
        while cands and slot < max_children:
            if rng.randint(1000) >= int(p_edge * 1000):
                break
            c = cands.pop(rng.randint(len(cands)))
            ch[slot, v] = c
            slot += 1
    return ch


def random_forest(n: int, max_children: int, seed: int, p_leaf: float = 0.4):
    """Small random forest (in-degree <= 1) for fuzzing, pre-order ids."""
    rng = SplitMix64(P_STRUCT, seed)
    ch = np.full((max_children, n), -1, dtype=np.int32)
    # attach node v (v >= 1) to a random earlier node with a free slot,
    # or start a new tree with probability p_leaf... simple Galton-Watson-ish
    fill = np.zeros(n, dtype=np.int64)
    for v in range(1, n):
        if rng.randint(1000) < 150:
            continue  # new root
        for _ in range(8):
            p = rng.randint(v)
            if fill[p] < max_children:
                ch[fill[p], p] = v
                fill[p] += 1
                break
    return ch


def shuffle_ids(children: np.ndarray, words: np.ndarray | None, seed: int):
    """Relabel nodes by a seeded permutation pi (new label of old node v is
    pi[v]); returns (children', words', pi). Used by the invariance tests."""
    n = children.shape[1]
    rng = SplitMix64(P_STRUCT, seed ^ 0x5A5A)
    keys = rng.next_array(n)
    order = np.argsort(keys, kind="stable")  # order[new] = old
    pi = np.empty(n, dtype=np.int64)
    pi[order] = np.arange(n)
    ch2 = np.full_like(children, -1)
    for k in range(children.shape[0]):
        src = children[k, order]
        ch2[k] = np.where(src >= 0, pi[np.maximum(src, 0)], -1)
    w2 = None if words is None else words[order]
    return ch2.astype(np.int32), w2, pi


# ---------------------------------------------------------------------------
# Payloads and parameters
# ---------------------------------------------------------------------------

def word_ids(children: np.ndarray, vocab: int, seed: int, all_nodes: bool = False):
    """randint(V) drawn in node-id order for leaves (every node if
    `all_nodes`, as DAG-RNN needs); -1 elsewhere."""
    n = children.shape[1]
    is_leaf = (children < 0).all(axis=0)
    need = np.ones(n, bool) if all_nodes else is_leaf
    rng = SplitMix64(P_WORDS, seed)
    w = np.full(n, -1, dtype=np.int32)
    idx = np.nonzero(need)[0]
    w[idx] = rng.randint_array(len(idx), vocab).astype(np.int32)
    return w


def embedding(vocab: int, hidden: int, seed: int):
    """Emb ~ U(-1, 1), [V][H] row-major, drawn in order."""
    return SplitMix64(P_EMB, seed).uniform_array(vocab * hidden, -1.0, 1.0).reshape(vocab, hidden)


def weight_shapes(cell: int, hidden: int, vocab: int):
    """(name, shape, fan_in or None for biases) in cx_weights order.
    SURVEY §8(b) weight table; MV-RNN p0 (Mw) is drawn from stream 5."""
    H = hidden
    if cell == TREERNN:
        return []
    if cell == TREEFC:
        return [("W", (H, 2 * H), 2 * H), ("b", (H,), None)]
    if cell == TREELSTM:
        return [("W_iou", (3 * H, H), H), ("U_iou", (3 * H, H), H), ("b_iou", (3 * H,), None),
                ("U_f", (H, H), H), ("b_f", (H,), None)]
    if cell in (TREEGRU, SIMPLETREEGRU):  # SimpleTreeGRU: same parameters
        return [("W_zh", (2 * H, H), H), ("U_z", (H, H), H), ("U_r", (H, H), H), ("U_h", (H, H), H),
                ("b_z", (H,), None), ("b_r", (H,), None), ("b_h", (H,), None)]
    if cell == MVRNN:
        return [("Mw", (vocab, H, H), "mw"), ("W", (H, 2 * H), 2 * H), ("beta", (H,), None),
                ("W_M", (H, 2 * H), 2 * H)]
    if cell == DAGRNN:
        return [("W_x", (H, H), H), ("U", (H, H), H), ("b", (H,), None)]
    raise ValueError(cell)


def weights(cell: int, hidden: int, vocab: int, seed: int | None = None):
    """Random-init weights of the cell's architecture, in cx_weights order.
    seed defaults to 1000 + cell id. Returns list of (name, float32 array)."""
    if seed is None:
        seed = 1000 + cell
    rng = SplitMix64(P_WEIGHTS, seed)
    out = []
    for name, shape, fan in weight_shapes(cell, hidden, vocab):
        count = int(np.prod(shape))
        if fan == "mw":
            mw = SplitMix64(P_MW, seed).uniform_array(count, -0.05, 0.05).reshape(shape)
            mw = mw + np.eye(hidden, dtype=np.float32)[None, :, :]
            out.append((name, mw.astype(np.float32)))
            continue
        bound = 1.0 / np.sqrt(fan if fan is not None else hidden)
        out.append((name, rng.uniform_array(count, -bound, bound).reshape(shape)))
    return out


# ---------------------------------------------------------------------------
# BASELINE.json configurations as concrete inputs
# ---------------------------------------------------------------------------

def workload(name: str, seed: int = 0):
    """Named workloads of SURVEY §8(d). Returns a dict with children, kind,
    words, cell, hidden, vocab, batch, offsets (structure boundaries)."""
    spec = {
        # configs[0]
        "cfg1_treernn": dict(cell=TREERNN, hidden=8, vocab=100, shape=("perfect", 1, 3)),
        # configs[1] (headline)
        "cfg2_treelstm_b10": dict(cell=TREELSTM, hidden=256, vocab=20000, shape=("sst", 10)),
        "cfg2_treelstm_b1": dict(cell=TREELSTM, hidden=256, vocab=20000, shape=("sst", 1)),
        # configs[2]
        "cfg3_treegru_b1": dict(cell=TREEGRU, hidden=512, vocab=20000, shape=("sst", 1)),
        "cfg3_treegru_b10": dict(cell=TREEGRU, hidden=512, vocab=20000, shape=("sst", 10)),
        "cfg3_treefc_b1": dict(cell=TREEFC, hidden=512, vocab=20000, shape=("perfect", 1, 7)),
        "cfg3_treefc_b10": dict(cell=TREEFC, hidden=512, vocab=20000, shape=("perfect", 10, 7)),
        # configs[3]
        "cfg4_mvrnn_b10": dict(cell=MVRNN, hidden=64, vocab=20000, shape=("sst", 10)),
        # configs[4]
        "cfg5_dagrnn_b1": dict(cell=DAGRNN, hidden=256, vocab=20000, shape=("grid", 1)),
        "cfg5_dagrnn_b10": dict(cell=DAGRNN, hidden=256, vocab=20000, shape=("grid", 10)),
        "cfg5_dagrnn_b4096": dict(cell=DAGRNN, hidden=256, vocab=20000, shape=("grid", 4096)),
        "cfg5_treelstm_b4096": dict(cell=TREELSTM, hidden=256, vocab=20000, shape=("sst", 4096)),
        # sequence workloads of the GRNN comparison (P:1535-1553,
        # "sequence length 100 and hidden and input sizes 256"): chains, kind sequence
        "f4_lstm_seq100_b1": dict(cell=TREELSTM, hidden=256, vocab=20000, shape=("chain", 1, 100)),
        "f4_lstm_seq100_b10": dict(cell=TREELSTM, hidden=256, vocab=20000, shape=("chain", 10, 100)),
        "f4_gru_seq100_b1": dict(cell=TREEGRU, hidden=256, vocab=20000, shape=("chain", 1, 100)),
        "f4_gru_seq100_b10": dict(cell=TREEGRU, hidden=256, vocab=20000, shape=("chain", 10, 100)),
    }[name]
    shape = spec["shape"]
    if shape[0] == "sst":
        ch, off = sst_shaped_forest(shape[1], seed)
        kind = TREE
    elif shape[0] == "perfect":
        ch, off = perfect_forest(shape[1], shape[2])
        kind = TREE
    elif shape[0] == "grid":
        ch, off = grid_dags(shape[1])
        kind = DAG
    elif shape[0] == "chain":
        ch, off = chains(shape[1], shape[2])
        kind = SEQUENCE
    else:
        raise ValueError(shape)
    cell = spec["cell"]
    words = word_ids(ch, spec["vocab"], seed, all_nodes=(cell == DAGRNN))
    return dict(name=name, children=ch, kind=kind, words=words, cell=cell,
                hidden=spec["hidden"], vocab=spec["vocab"], batch=len(off) - 1,
                offsets=off, seed=seed)
