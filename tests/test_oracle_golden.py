"""Brute-force pins of the forward oracle (SURVEY §8(c) "Every cell on tiny
trees (<= 7 nodes) at H = 1-2 evaluated by hand or mpmath").

tests/golden/brute_force.json is written by tools/gen_goldens.py, which imports
only mpmath: 50-digit plain recursion from hand-typed dyadic inputs, each case
citing the passage / reading its cell follows. The matrices are asymmetric and
not the identity, so the MV-RNN pairing [B a; A b] (reading Q9) and the
TreeGRU per-child reset gate (reading Q3) are distinguished from
their alternatives (see test_alternatives_differ and the mutation check)."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "brute_force.json")))
CASES = {c["name"]: c for c in GOLD["cases"]}
TOL = 1e-13  # fp64 recursion vs 50-digit values of O(1) magnitude


def _inputs(c):
    f = lambda a: np.array(a, dtype=np.float64).astype(np.float32)
    ws = [f(w) for w in c["weights"]]
    for w, src in zip(ws, c["weights"]):  # the hand-typed values are exact in fp32
        assert np.array_equal(w.astype(np.float64), np.array(src, dtype=np.float64))
    return (np.array(c["children"], np.int32), np.array(c["words"], np.int32), f(c["emb"]), ws)


@pytest.mark.parametrize("name", sorted(CASES))
def test_brute_force_golden(name):
    c = CASES[name]
    ch, words, emb, ws = _inputs(c)
    lin = oracle.linearize(ch, c["kind"])
    assert lin["status"] == 0
    want_aux = "aux" in c
    st, bad, h, aux = oracle.forward(c["cell"], c["H"], c["V"], ws, emb, words, ch,
                                     want_aux=want_aux)
    assert st == 0, (st, bad)
    ref = np.array(c["h"], dtype=np.float64)
    assert np.abs(h - ref).max() < TOL, np.abs(h - ref).max()
    if want_aux:
        ra = np.array(c["aux"], dtype=np.float64)
        assert np.abs(aux - ra).max() < TOL


def _mv_alt(c, pairing):
    """MV-RNN root under an alternative pairing, numpy fp64 (test of the fixture
    only: it shows the golden inputs separate the readings)."""
    ch, words, emb, ws = _inputs(c)
    Mw, W, beta, WM = [w.astype(np.float64) for w in ws]

    def ev(v):
        l, r = ch[0, v], ch[1, v]
        if l < 0:
            return emb[words[v]].astype(np.float64), Mw[words[v]]
        (a, A), (b, B) = ev(l), ev(r)
        p = {"BaAb": np.r_[B @ a, A @ b], "AaBb": np.r_[A @ a, B @ b],
             "AbBa": np.r_[A @ b, B @ a]}[pairing]
        return np.tanh(W @ p + beta), WM @ np.vstack([A, B])
    return ev(0)[0]


def test_alternatives_differ():
    """The golden inputs separate the readings from their plausible alternatives."""
    c = CASES["mvrnn_h2_left5"]
    roots = {p: _mv_alt(c, p) for p in ("BaAb", "AaBb", "AbBa")}
    assert np.allclose(roots["BaAb"], np.array(c["h"][0], dtype=np.float64), atol=1e-13)
    assert np.abs(roots["BaAb"] - roots["AaBb"]).max() > 1e-3
    assert np.abs(roots["BaAb"] - roots["AbBa"]).max() > 1e-3
    # TreeGRU: per-child reset vs reset applied to h~ at the two-child root
    g = CASES["treegru_h2_left5"]
    ch, words, emb, ws = _inputs(g)
    W_zh, U_z, U_r, U_h, b_z, b_r, b_h = [w.astype(np.float64) for w in ws]
    h = np.array(g["h"], dtype=np.float64)
    hk = [h[ch[0, 0]], h[ch[1, 0]]]
    ht = hk[0] + hk[1]
    sg = lambda x: 1 / (1 + np.exp(-x))
    z = sg(U_z @ ht + b_z)
    per_child = sum(sg(U_r @ x + b_r) * x for x in hk)
    on_sum = sg(U_r @ ht + b_r) * ht
    root = lambda s: z * ht + (1 - z) * np.tanh(U_h @ s + b_h)
    assert np.allclose(root(per_child), h[0], atol=1e-13)
    assert np.abs(root(on_sum) - h[0]).max() > 1e-3
