"""Shared helpers for the -m gpu parity tests (call through the C ABI)."""
import numpy as np
import torch

import oracle
import synth

TOL_F32 = 1e-4  # BASELINE.json north_star: max relative error 1e-4 for the fp32 path


def dev_i32(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def dev_f32(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def lin_to_numpy(lin):
    """Device linearization -> dict in oracle.linearize layout (syncs)."""
    h = lin.header_dict()
    n, L, R = lin.n, h["num_levels"], h["num_roots"]
    out = dict(h)
    out.update(perm=lin.perm[:n].cpu().numpy(), inv=lin.inv[:n].cpu().numpy(),
               children=lin.children.cpu().numpy(), height=lin.height[:n].cpu().numpy(),
               level_begin=lin.level_begin[:L].cpu().numpy(),
               level_size=lin.level_size[:L].cpu().numpy(), roots=lin.roots[:R].cpu().numpy(),
               structure=lin.structure[:n].cpu().numpy())
    return out


LIN_FIELDS = ("status", "bad_node", "num_nodes", "num_levels", "num_leaves", "first_leaf",
              "max_level_size", "num_roots")


def assert_lin_equal(dev, ref):
    """Bit-exact comparison of every linearization output."""
    if ref["status"] != 0:
        assert (dev["status"], dev["bad_node"]) == (ref["status"], ref["bad_node"])
        return
    for f in LIN_FIELDS:
        assert dev[f] == ref[f], (f, dev[f], ref[f])
    for f in ("perm", "inv", "children", "height", "level_begin", "level_size", "roots",
              "structure"):
        assert np.array_equal(np.asarray(dev[f]), np.asarray(ref[f])), f


def normwise_rel_err(got, ref, rows=None):
    """Per-node e_n = max_i |g - r| / max(max_i |r|, 1e-6); returns max_n e_n
    (SURVEY §8(c) Q19)."""
    got = np.asarray(got, np.float64).reshape(len(got), -1)
    ref = np.asarray(ref, np.float64).reshape(len(ref), -1)
    if rows is not None:
        got, ref = got[rows], ref[rows]
    num = np.abs(got - ref).max(axis=1)
    den = np.maximum(np.abs(ref).max(axis=1), 1e-6)
    return float((num / den).max()) if len(num) else 0.0


def weights_dev(cell, hidden, vocab, seed=None):
    ws = synth.weights(cell, hidden, vocab, seed)
    return [w for _, w in ws], [dev_f32(w) for _, w in ws]


def run_both(cell, hidden, vocab, children, kind, words, emb, ws_np, ws_dev, want_aux=False,
             num_roots=None):
    import paper_2011_01383_b200 as cx
    lin = cx.linearize(dev_i32(children), kind)
    h, aux, roots = cx.forward(cell, hidden, ws_dev, dev_f32(emb), dev_i32(words), lin,
                               want_aux=want_aux, num_roots=num_roots)
    st, bad = cx.status(lin)
    rst, rbad, rh, raux = oracle.forward(cell, hidden, vocab, ws_np, emb, words, children,
                                         want_aux=want_aux)
    return lin, (st, bad), h, aux, roots, (rst, rbad), rh, raux
