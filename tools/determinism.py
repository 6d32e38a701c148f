"""Run-to-run and shard-invariance probe of the CUDA path (one GPU): every
workload's linearize_forward is repeated R times (h compared bit for bit with
the first run), then each shard of G = 2 is run alone and its rows compared
with the unsharded result. Prints one line per workload."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402
from paper_2011_01383_b200 import shard  # noqa: E402


def run(w, children, words, dtype):
    dev = torch.device("cuda", 0)
    d = lambda a, t: torch.as_tensor(np.ascontiguousarray(a, dtype=t)).to(dev)
    H, V, cell = w["hidden"], w["vocab"], w["cell"]
    ws = [d(a, np.float32) for _, a in synth.weights(cell, H, V)]
    emb = d(synth.embedding(V, H, w["seed"]), np.float32)
    lin, h, _, _ = cx.linearize_forward(d(children, np.int32), w["kind"], cell, H, ws, emb,
                                        d(words, np.int32), dtype=dtype)
    assert cx.status(lin) == (0, -1)
    return h.cpu().numpy()


def main():
    names = sys.argv[1:] or ["cfg3_treegru_b10", "cfg2_treelstm_b10",
                             "cfg5_dagrnn_b10", "cfg3_treefc_b10", "cfg4_mvrnn_b10"]
    for name in names:
        w = synth.workload(name)
        for dt in (cx.F32,):
            h0 = run(w, w["children"], w["words"], dt)
            import os
            R = int(os.environ.get("REPEATS", "8"))
            diffs = [float(np.abs(run(w, w["children"], w["words"], dt) - h0).max()) for _ in range(R)]
            rep = max(diffs)
            nbad = sum(d > 0 for d in diffs)
            off = w["offsets"]
            sh = []
            for G in (2, 4):
                worst = 0.0
                for r in range(G):
                    sub, wl, (g0, g1), _ = shard.shard(w["children"], off, r, G, w["words"])
                    hr = run(w, sub, wl, dt)
                    worst = max(worst, float(np.abs(hr - h0[off[g0]:off[g1]]).max()))
                sh.append(worst)
            print(f"{name} f32: {R} repeats, {nbad} differ, max|diff| {rep:.3e}  shard G=2 {sh[0]:.3e} G=4 {sh[1]:.3e}",
                  flush=True)


if __name__ == "__main__":
    main()
