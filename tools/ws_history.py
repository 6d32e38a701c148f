"""Does a forward depend on what an earlier call left in the cached workspace?
Runs workload A fresh, then each 'dirtying' workload, then A again (bitwise)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402


def run(name, dtype=cx.F32):
    w = synth.workload(name)
    dev = torch.device("cuda", 0)
    d = lambda a, t: torch.as_tensor(np.ascontiguousarray(a, dtype=t)).to(dev)
    H, V, cell = w["hidden"], w["vocab"], w["cell"]
    ws = [d(a, np.float32) for _, a in synth.weights(cell, H, V)]
    emb = d(synth.embedding(V, H, w["seed"]), np.float32)
    lin, h, _, _ = cx.linearize_forward(d(w["children"], np.int32), w["kind"], cell, H, ws, emb,
                                        d(w["words"], np.int32), dtype=dtype)
    st = cx.status(lin)
    if st != (0, -1):
        print(f"{name}: status {st} {cx.status_str(st[0])}", flush=True)
    return h.cpu().numpy()


target = sys.argv[1] if len(sys.argv) > 1 else "cfg3_treegru_b10"
h0 = run(target)
for dirt, dt in [("cfg3_treefc_b10", cx.F32), ("cfg5_treelstm_b4096", cx.F32), ("cfg5_dagrnn_b4096", cx.BF16),
                 ("cfg2_treelstm_b10", cx.F32), ("cfg4_mvrnn_b10", cx.F32), ("f3_simpletreegru_b10", cx.F32)]:
    try:
        run(dirt, dt)
    except KeyError:
        continue
    h1 = run(target)
    print(f"{target} after {dirt}: max|diff| {np.abs(h1 - h0).max():.3e}", flush=True)
