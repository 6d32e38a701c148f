"""fp32 forward time vs batch size, split-fp32 tensor-core kernel vs the FMA
kernels (CX_TC_F32_MIN_N), TreeLSTM / DAG-RNN / TreeFC: where should the
dispatch threshold sit? (events around linearize_forward, L2 flushed)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402

dev = torch.device("cuda", 0)
d = lambda a, t: torch.as_tensor(np.ascontiguousarray(a, dtype=t)).to(dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def timeit(cell, H, V, ch, kind, words):
    ws = [d(a, np.float32) for _, a in synth.weights(cell, H, V)]
    emb = d(synth.embedding(V, H, 1), np.float32)
    chd, wd = d(ch, np.int32), d(words, np.int32)
    ts = []
    for it in range(8):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lin, h, _, _ = cx.linearize_forward(chd, kind, cell, H, ws, emb, wd)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    assert cx.status(lin) == (0, -1)
    return min(ts), cx.forward_family(cell, H, ch.shape[1], ch.shape[0], V)


for name, cell, H, mk, kind in [("treelstm", synth.TREELSTM, 256, lambda b: synth.sst_shaped_forest(b, 1)[0], synth.TREE),
                                ("treefc", synth.TREEFC, 512, lambda b: synth.perfect_forest(b, 1)[0], synth.TREE),
                                ("dagrnn", synth.DAGRNN, 256, lambda b: synth.grid_dags(b, 10, 10)[0], synth.DAG)]:
    for b in (10, 20, 50, 100, 200, 400):
        ch = mk(b)
        V = 20000
        words = synth.word_ids(ch, V, 1, all_nodes=(cell == synth.DAGRNN))
        out = []
        for env in ("1", "1000000000"):
            os.environ["CX_TC_F32_MIN_N"] = env
            out.append(timeit(cell, H, V, ch, kind, words))
        print(f"{name} b{b} n={ch.shape[1]}: tc32 {out[0][0]:.1f} us ({out[0][1]})  fma {out[1][0]:.1f} us ({out[1][1]})", flush=True)
