"""I-cache hypothesis: a kernel replayed twice back-to-back in one graph."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402
from exp_overhead import timeit, t, dev  # noqa: E402

w = synth.workload("cfg2_treelstm_b10")
cell, H, V = synth.TREELSTM, 256, 20000
ch = w["children"]
emb = t(synth.embedding(V, H, 0), np.float32)
ws = [t(a, np.float32) for _, a in synth.weights(cell, H, V)]
chd, wd = t(ch, np.int32), t(w["words"], np.int32)
lin = cx.alloc_linearization(ch.shape[1], 2, w["kind"], dev)
h = torch.empty(ch.shape[1], H, device=dev)
cx.linearize(chd, w["kind"], out=lin)
cx.forward(cell, H, ws, emb, wd, lin, h_out=h)
L1 = lambda: cx.linearize(chd, w["kind"], out=lin)
F1 = lambda: cx.forward(cell, H, ws, emb, wd, lin, h_out=h)
for fl in (True, False):
    a = timeit(L1, do_flush=fl); b = timeit(lambda: (L1(), L1()), do_flush=fl)
    c = timeit(F1, do_flush=fl); d = timeit(lambda: (F1(), F1()), do_flush=fl)
    print(f"flush={fl}: lin x1 {a:6.2f}  lin x2 {b:6.2f} (2nd {b-a:6.2f}) | fwd x1 {c:6.2f}  fwd x2 {d:6.2f} (2nd {d-c:6.2f}) us")
