"""Debug: cluster kernel push vs pull mode, fused vs separate, per-level error vs the oracle."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth  # noqa
import paper_2011_01383_b200 as cx  # noqa

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_treelstm_b10"
w = synth.workload(name)
H, V, cell = w["hidden"], w["vocab"], w["cell"]
emb = synth.embedding(V, H, w["seed"])
ws = [a for _, a in synth.weights(cell, H, V)]
words = synth.word_ids(w["children"], V, w["seed"], all_nodes=(cell == synth.DAGRNN))
d = lambda a, t: torch.as_tensor(np.ascontiguousarray(a, dtype=t)).cuda()
st, _, rh, _ = oracle.forward(cell, H, V, ws, emb, words, w["children"])
ref = oracle.linearize(w["children"], w["kind"])
hin = ref["height"][ref["inv"]]
wsd = [d(a, np.float32) for a in ws]
for mode in ("1", "0"):
    os.environ["CX_PUSH"] = mode
    for fused in (True, False):
        if fused:
            lin, h, _, _ = cx.linearize_forward(d(w["children"], np.int32), w["kind"], cell, H, wsd,
                                                d(emb, np.float32), d(words, np.int32))
        else:
            lin = cx.linearize(d(w["children"], np.int32), w["kind"])
            h, _, _ = cx.forward(cell, H, wsd, d(emb, np.float32), d(words, np.int32), lin)
        torch.cuda.synchronize()
        g = h.cpu().numpy().astype(np.float64)
        e = np.abs(g - rh).max(axis=1) / np.maximum(np.abs(rh).max(axis=1), 1e-6)
        per = [float(e[hin == l].max()) for l in range(ref["num_levels"])]
        print(f"push={mode} fused={fused}: " + " ".join(f"{x:.1e}" for x in per), flush=True)
