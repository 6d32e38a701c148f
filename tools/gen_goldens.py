#!/usr/bin/env python
"""Brute-force golden values for every cell on tiny structures (SURVEY §8(c)
"Every cell on tiny trees (<= 7 nodes) at H = 1-2 evaluated by hand or
mpmath"). Writes tests/golden/brute_force.json.

This script is deliberately independent of both the oracle (oracle/) and the
CUDA path: it imports only mpmath (50-digit arithmetic) and json. Every
structure, word id, embedding and weight below is typed in by hand as a dyadic
rational (exact in fp32), and every cell is evaluated by plain recursion from
the root, written from the cell equations the paper names:

  TreeRNN        Listing 1: leaf Emb[word], h = tanh(h_l + h_r)
  TreeFC         T2 P:1290 ("TF Fold benchmarking model"), reading Q2:
                 h = tanh(W [h_l; h_r] + b)
  TreeLSTM       T2 P:1293 "Child-sum TreeLSTM" [Tai et al. 2015], reading Q1
  TreeGRU        P:1268-1270 ("similar to TreeLSTM, except GRU cell"), reading Q3:
                 per-child reset gate before U_h
  SimpleTreeGRU  footnote P:1638-1640: h = (1 - z) * h' instead of
                 z * h_{t-1} + (1 - z) * h', reading Q24
  MV-RNN         T2 P:1294 [Socher et al. 2012], reading Q9:
                 a = tanh(W [B a; A b] + beta), A = W_M [A; B]
  DAG-RNN        T2 P:1291 [Shuai et al.], reading Q8: h = tanh(W_x x + U sum h_pred + b)

Recursion recomputes shared DAG children (no memo): brute force, tiny inputs.
Run:  python tools/gen_goldens.py   (rewrites the JSON; commit the result)
"""
import json
import os

import mpmath as mp

mp.mp.dps = 50

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                   "golden", "brute_force.json")

TREERNN, TREEFC, TREELSTM, TREEGRU, MVRNN, DAGRNN, SIMPLETREEGRU = range(7)
SEQUENCE, TREE, DAG = 0, 1, 2


def M(x):
    return mp.mpf(x)


def sig(x):
    return 1 / (1 + mp.exp(-x))


# ---- tiny linear algebra on python lists of mpf (written out, no library) ----
def mv(W, x, c0=0):
    """y_r = sum_k W[r][c0 + k] x_k"""
    return [mp.fsum(M(W[r][c0 + k]) * x[k] for k in range(len(x))) for r in range(len(W))]


def rows(W, r0, r1):
    return W[r0:r1]


def add(*vs):
    return [mp.fsum(t) for t in zip(*vs)]


def mm(A, B):
    """(A B)_ij = sum_k A_ik B_kj"""
    return [[mp.fsum(M(A[i][k]) * M(B[k][j]) for k in range(len(B))) for j in range(len(B[0]))]
            for i in range(len(A))]


# ---- structures (children SoA [maxc][n], input ids, -1 absent) -------------
def kids(ch, v):
    out = []
    for k in range(len(ch)):
        if ch[k][v] == -1:
            break
        out.append(ch[k][v])
    return out


def eval_all(ch, node_fn):
    n = len(ch[0])
    memo = {}

    def ev(v):  # plain recursion; memo only keeps the table, values are recomputed
        val = node_fn(v, [ev(c) for c in kids(ch, v)])
        memo[v] = val
        return val

    return [ev(v) for v in range(n)]


# ---- the cells ---------------------------------------------------------------
def treernn(case):
    E, w = case["emb"], case["words"]

    def node(v, ks):
        if not ks:
            return [M(x) for x in E[w[v]]]
        hl, hr = ks
        return [mp.tanh(a + b) for a, b in zip(hl, hr)]
    return eval_all(case["children"], node)


def treefc(case):
    E, w = case["emb"], case["words"]
    W, b = case["weights"]
    H = case["H"]

    def node(v, ks):
        if not ks:
            return [M(x) for x in E[w[v]]]
        hl, hr = ks
        pre = add(mv(W, hl, 0), mv(W, hr, H), [M(x) for x in b])
        return [mp.tanh(x) for x in pre]
    return eval_all(case["children"], node)


def treelstm(case):
    """Child-sum TreeLSTM [Tai et al. 2015] (reading Q1): gate rows i, o, u."""
    E, w = case["emb"], case["words"]
    W_iou, U_iou, b_iou, U_f, b_f = case["weights"]
    H = case["H"]

    def node(v, ks):
        if not ks:
            x = [M(t) for t in E[w[v]]]
            g = add(mv(W_iou, x), [M(t) for t in b_iou])
        else:
            ht = add(*[k[0] for k in ks])
            g = add(mv(U_iou, ht), [M(t) for t in b_iou])
        i, o, u = g[:H], g[H:2 * H], g[2 * H:]
        c = [sig(i[j]) * mp.tanh(u[j]) for j in range(H)]
        for hk, ck in ks:
            f = add(mv(U_f, hk), [M(t) for t in b_f])
            c = [c[j] + sig(f[j]) * ck[j] for j in range(H)]
        h = [sig(o[j]) * mp.tanh(c[j]) for j in range(H)]
        return (h, c)
    return eval_all(case["children"], node)


def treegru(case, simple=False):
    """Child-sum TreeGRU (reading Q3); simple=True: SimpleTreeGRU (Q24)."""
    E, w = case["emb"], case["words"]
    W_zh, U_z, U_r, U_h, b_z, b_r, b_h = case["weights"]
    H = case["H"]

    def node(v, ks):
        if not ks:
            x = [M(t) for t in E[w[v]]]
            z = [sig(t) for t in add(mv(rows(W_zh, 0, H), x), [M(t) for t in b_z])]
            g = [mp.tanh(t) for t in add(mv(rows(W_zh, H, 2 * H), x), [M(t) for t in b_h])]
            return [(1 - z[j]) * g[j] for j in range(H)]
        ht = add(*ks)
        z = [sig(t) for t in add(mv(U_z, ht), [M(t) for t in b_z])]
        s = [M(0)] * H
        for hk in ks:
            r = [sig(t) for t in add(mv(U_r, hk), [M(t) for t in b_r])]
            s = [s[j] + r[j] * hk[j] for j in range(H)]
        g = [mp.tanh(t) for t in add(mv(U_h, s), [M(t) for t in b_h])]
        if simple:
            return [(1 - z[j]) * g[j] for j in range(H)]
        return [z[j] * ht[j] + (1 - z[j]) * g[j] for j in range(H)]
    return eval_all(case["children"], node)


def mvrnn(case):
    """MV-RNN [Socher et al. 2012] (reading Q9): left child (a, A), right (b, B)."""
    E, w = case["emb"], case["words"]
    Mw, W, beta, W_M = case["weights"]
    H = case["H"]

    def node(v, ks):
        if not ks:
            return ([M(t) for t in E[w[v]]], [[M(t) for t in row] for row in Mw[w[v]]])
        (a, A), (b, B) = ks
        p = mv(B, a) + mv(A, b)                     # [B a; A b]
        h = [mp.tanh(t) for t in add(mv(W, p), [M(t) for t in beta])]
        AB = A + B                                  # [A; B] stacked, 2H x H
        return (h, mm(W_M, AB))
    return eval_all(case["children"], node)


def dagrnn(case):
    E, w = case["emb"], case["words"]
    W_x, U, b = case["weights"]
    H = case["H"]

    def node(v, ks):
        x = [M(t) for t in E[w[v]]]
        ht = add(*ks) if ks else [M(0)] * H
        return [mp.tanh(t) for t in add(mv(W_x, x), mv(U, ht), [M(t) for t in b])]
    return eval_all(case["children"], node)


# ---- hand-typed inputs ---------------------------------------------------------
TRI = [[1, -1, -1], [2, -1, -1]]                            # 0(1, 2)
LEFT5 = [[1, 2, -1, -1, -1], [4, 3, -1, -1, -1]]            # 0(1(2, 3), 4), pre-order
PERFECT7 = [[1, 2, -1, -1, 5, -1, -1], [4, 3, -1, -1, 6, -1, -1]]  # 0(1(2,3), 4(5,6))
UNARY = [[1, 2, -1, -1], [3, -1, -1, -1]]                   # 0(1(2), 3): node 1 has 1 child
DIAMOND = [[1, 3, 3, -1], [2, -1, -1, -1]]                  # 0(1, 2), 1(3), 2(3): shared child
GRID22 = [[-1, 0, 0, 1], [-1, -1, -1, 2]]                   # (i,j) -> 2i+j, children [up, left]

# embeddings (V = 4) and word ids: dyadic, distinct, asymmetric
EMB1 = [["0.75"], ["-0.5"], ["0.25"], ["-0.875"]]
EMB2 = [["0.75", "-0.25"], ["-0.5", "0.625"], ["0.125", "0.375"], ["-0.875", "-0.1875"]]

MAT_A = [["0.5", "-0.25"], ["0.75", "0.125"]]
MAT_B = [["-0.375", "0.625"], ["0.25", "-0.5"]]
MAT_C = [["0.3125", "0.5625"], ["-0.6875", "0.1875"]]
MAT_D = [["-0.125", "-0.75"], ["0.4375", "0.875"]]
MAT_E = [["0.625", "0.0625"], ["-0.25", "-0.5625"]]
MAT_F = [["0.1875", "-0.4375"], ["0.9375", "-0.3125"]]


def case(name, cell, H, kind, children, words, emb, weights, cite):
    return dict(name=name, cell=cell, H=H, V=len(emb), kind=kind, children=children,
                words=words, emb=emb, weights=weights, cite=cite)


def cases():
    out = []
    # TreeRNN (Listing 1), H = 1 and 2
    out.append(case("treernn_h1_left5", TREERNN, 1, TREE, LEFT5, [-1, -1, 0, 3, 1], EMB1, [],
                    "Listing 1 P:853-871"))
    out.append(case("treernn_h2_perfect7", TREERNN, 2, TREE, PERFECT7,
                    [-1, -1, 0, 3, -1, 1, 2], EMB2, [], "Listing 1 P:853-871"))
    # TreeFC: W = [W_l W_r] with W_l != W_r, asymmetric (Q2)
    W_fc = [MAT_A[0] + MAT_B[0], MAT_A[1] + MAT_B[1]]
    out.append(case("treefc_h2_left5", TREEFC, 2, TREE, LEFT5, [-1, -1, 0, 3, 1], EMB2,
                    [W_fc, ["0.0625", "-0.125"]], "T2 P:1290, reading Q2"))
    out.append(case("treefc_h1_tri", TREEFC, 1, TREE, TRI, [-1, 2, 1], EMB1,
                    [[["0.5", "-1.25"]], ["0.25"]], "T2 P:1290, reading Q2"))
    # TreeLSTM: W_iou [3H][H], U_iou [3H][H], b_iou [3H], U_f [H][H], b_f [H]
    W_iou = MAT_A + MAT_B + MAT_C
    U_iou = MAT_D + MAT_E + MAT_F
    b_iou = ["0.125", "-0.25", "0.375", "-0.0625", "0.5", "-0.3125"]
    U_f = [["0.6875", "-0.5"], ["0.25", "0.8125"]]
    b_f = ["-0.125", "0.1875"]
    lstm_w = [W_iou, U_iou, b_iou, U_f, b_f]
    out.append(case("treelstm_h2_left5", TREELSTM, 2, TREE, LEFT5, [-1, -1, 0, 3, 1], EMB2,
                    lstm_w, "T2 P:1293 child-sum TreeLSTM, reading Q1"))
    out.append(case("treelstm_h2_unary", TREELSTM, 2, TREE, UNARY, [-1, -1, 2, 1], EMB2,
                    lstm_w, "T2 P:1293, reading Q1 (child-sum over 1 and 2 children)"))
    out.append(case("treelstm_h1_perfect7", TREELSTM, 1, TREE, PERFECT7,
                    [-1, -1, 0, 3, -1, 1, 2], EMB1,
                    [[["0.5"], ["-0.75"], ["0.625"]], [["-0.25"], ["0.875"], ["0.375"]],
                     ["0.125", "-0.25", "0.5"], [["0.6875"]], ["-0.125"]],
                    "T2 P:1293, reading Q1"))
    # TreeGRU: W_zh [2H][H], U_z, U_r, U_h [H][H], b_z, b_r, b_h [H]
    gru_w = [MAT_A + MAT_B, MAT_C, MAT_D, MAT_E, ["0.125", "-0.375"], ["0.25", "-0.0625"],
             ["-0.1875", "0.3125"]]
    out.append(case("treegru_h2_left5", TREEGRU, 2, TREE, LEFT5, [-1, -1, 0, 3, 1], EMB2,
                    gru_w, "P:1268-1270, reading Q3 (per-child reset gate)"))
    out.append(case("treegru_h2_unary", TREEGRU, 2, TREE, UNARY, [-1, -1, 2, 1], EMB2,
                    gru_w, "P:1268-1270, reading Q3"))
    out.append(case("treegru_h1_perfect7", TREEGRU, 1, TREE, PERFECT7,
                    [-1, -1, 0, 3, -1, 1, 2], EMB1,
                    [[["0.5"], ["-0.75"]], [["0.625"]], [["-1.5"]], [["0.875"]], ["0.125"],
                     ["0.25"], ["-0.375"]], "P:1268-1270, reading Q3"))
    out.append(case("simpletreegru_h2_left5", SIMPLETREEGRU, 2, TREE, LEFT5,
                    [-1, -1, 0, 3, 1], EMB2, gru_w, "footnote P:1638-1640, reading Q24"))
    # MV-RNN: Mw [V][H][H], W [H][2H], beta [H], W_M [H][2H]
    Mw2 = [MAT_A, MAT_B, MAT_C, MAT_D]
    W_mv = [MAT_E[0] + MAT_F[0], MAT_E[1] + MAT_F[1]]
    W_M = [MAT_B[0] + MAT_D[0], MAT_B[1] + MAT_D[1]]
    out.append(case("mvrnn_h2_left5", MVRNN, 2, TREE, LEFT5, [-1, -1, 0, 3, 1], EMB2,
                    [Mw2, W_mv, ["0.0625", "-0.1875"], W_M],
                    "T2 P:1294 [Socher et al. 2012], reading Q9"))
    out.append(case("mvrnn_h2_perfect7", MVRNN, 2, TREE, PERFECT7, [-1, -1, 0, 3, -1, 1, 2],
                    EMB2, [Mw2, W_mv, ["0.0625", "-0.1875"], W_M], "T2 P:1294, reading Q9"))
    out.append(case("mvrnn_h1_tri", MVRNN, 1, TREE, TRI, [-1, 0, 3], EMB1,
                    [[[["1.5"]], [["-0.5"]], [["0.75"]], [["2.0"]]], [["0.5", "-1.25"]],
                     ["0.125"], [["0.75", "0.375"]]], "T2 P:1294, reading Q9"))
    # DAG-RNN: W_x, U [H][H], b [H]; every node has a word (Q8, Q16)
    dag_w = [MAT_A, MAT_F, ["0.125", "-0.25"]]
    out.append(case("dagrnn_h2_diamond", DAGRNN, 2, DAG, DIAMOND, [0, 1, 2, 3], EMB2, dag_w,
                    "T2 P:1291, reading Q8 (shared child read by both parents)"))
    out.append(case("dagrnn_h2_grid22", DAGRNN, 2, DAG, GRID22, [3, 0, 2, 1], EMB2, dag_w,
                    "T2 P:1291, reading Q8/Q22 (2x2 grid)"))
    out.append(case("dagrnn_h1_left5", DAGRNN, 1, TREE, LEFT5, [1, 2, 0, 3, 1], EMB1,
                    [[["0.5"]], [["-0.75"]], ["0.25"]], "T2 P:1291, reading Q8"))
    return out


EVAL = {TREERNN: treernn, TREEFC: treefc, TREELSTM: treelstm, TREEGRU: treegru,
        MVRNN: mvrnn, DAGRNN: dagrnn, SIMPLETREEGRU: lambda c: treegru(c, simple=True)}


def fmt(x):
    return mp.nstr(x, 30)


def main():
    res = []
    for c in cases():
        vals = EVAL[c["cell"]](c)
        if c["cell"] == TREELSTM:
            c["h"] = [[fmt(x) for x in v[0]] for v in vals]
            c["aux"] = [[fmt(x) for x in v[1]] for v in vals]
        elif c["cell"] == MVRNN:
            c["h"] = [[fmt(x) for x in v[0]] for v in vals]
            c["aux"] = [[[fmt(x) for x in row] for row in v[1]] for v in vals]
        else:
            c["h"] = [[fmt(x) for x in v] for v in vals]
        res.append(c)
    doc = {"_source": "Written by tools/gen_goldens.py (mpmath, 50 digits; imports neither "
                      "oracle/ nor the CUDA package). Inputs are hand-typed dyadic rationals; "
                      "each case cites the passage / reading its cell follows.",
           "cases": res}
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)
    print(f"wrote {len(res)} cases to {OUT}")


if __name__ == "__main__":
    main()
