"""Implicit workspaces (cx.py's cache) across calls of different shapes: the
synchronisation words' offsets depend on the shape (cx.h), so a cached buffer
reused for another shape must be zero-filled again. A call's results (and its
status) must not depend on what earlier calls of other shapes left behind."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _run(cx, name, dtype):
    w = synth.workload(name)
    dev = torch.device("cuda", 0)
    d = lambda a, t: torch.as_tensor(np.ascontiguousarray(a, dtype=t)).to(dev)
    H, V, cell = w["hidden"], w["vocab"], w["cell"]
    ws = [d(a, np.float32) for _, a in synth.weights(cell, H, V)]
    emb = d(synth.embedding(V, H, w["seed"]), np.float32)
    lin, h, _, _ = cx.linearize_forward(d(w["children"], np.int32), w["kind"], cell, H, ws, emb,
                                        d(w["words"], np.int32), dtype=dtype)
    assert cx.status(lin) == (0, -1), name
    return h.cpu().numpy()


@pytest.mark.parametrize("target", ["cfg2_treelstm_b10", "cfg3_treegru_b10", "cfg5_dagrnn_b10"])
def test_results_independent_of_workspace_history(target):
    import paper_2011_01383_b200 as cx
    h0 = _run(cx, target, cx.F32)
    for dirt, dt in [("cfg5_dagrnn_b4096", cx.BF16), ("cfg5_treelstm_b4096", cx.F32),
                     ("cfg3_treefc_b10", cx.F32), ("cfg4_mvrnn_b10", cx.F32)]:
        _run(cx, dirt, dt)
        assert np.array_equal(_run(cx, target, cx.F32), h0), f"{target} after {dirt}"
