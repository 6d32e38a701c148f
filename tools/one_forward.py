"""Three cx_linearize_forward calls of a workload (ncu target: the third
forward launch is the measured one): python tools/one_forward.py NAME [bf16]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402

name = sys.argv[1]
dt = cx.BF16 if len(sys.argv) > 2 and sys.argv[2] == "bf16" else cx.F32
w = synth.workload(name)
dev = torch.device("cuda", 0)
d = lambda a, t: torch.as_tensor(np.ascontiguousarray(a, dtype=t)).to(dev)
H, V, cell = w["hidden"], w["vocab"], w["cell"]
ws = [d(a, np.float32) for _, a in synth.weights(cell, H, V)]
emb = d(synth.embedding(V, H, w["seed"]), np.float32)
ch, words = d(w["children"], np.int32), d(w["words"], np.int32)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(3):
    flush.fill_(1.0)  # cold L2, as in the bench
    lin, h, _, _ = cx.linearize_forward(ch, w["kind"], cell, H, ws, emb, words, dtype=dt)
torch.cuda.synchronize()
print(name, "status", cx.status(lin), "family", cx.forward_family(cell, H, ch.shape[1], ch.shape[0], V, dt))
