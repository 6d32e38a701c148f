"""One small linearize + forward per kernel family, for compute-sanitizer
(tools/gpu/sanitize.sh): python tools/sanitize_case.py <case>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402

case = sys.argv[1]
dev = torch.device("cuda", 0)
d = lambda a, t: torch.as_tensor(np.ascontiguousarray(a, dtype=t)).to(dev)


def run(cell, H, V, ch, kind, fused=False, dtype=cx.F32, path=None):
    if path:
        os.environ["CX_FORWARD_PATH"] = path
    words = synth.word_ids(ch, V, 1, all_nodes=(cell == synth.DAGRNN))
    emb = synth.embedding(V, H, 1)
    ws = [d(w, np.float32) for _, w in synth.weights(cell, H, V)]
    if fused:
        lin, h, _, _ = cx.linearize_forward(d(ch, np.int32), kind, cell, H, ws, d(emb, np.float32),
                                            d(words, np.int32), dtype=dtype, want_aux=True, num_roots=1)
    else:
        lin = cx.linearize(d(ch, np.int32), kind)
        h, _, _ = cx.forward(cell, H, ws, d(emb, np.float32), d(words, np.int32), lin, dtype=dtype,
                             want_aux=True)
    torch.cuda.synchronize()
    print(case, "status", cx.status(lin), "family",
          cx.forward_family(cell, H, ch.shape[1], ch.shape[0], V, dtype), "h[0,:3]",
          h[0, :3].tolist())


forest = lambda b: synth.sst_shaped_forest(b, 3, leaves=9)[0]
if case == "lin_multi":  # multi-CTA linearizer
    ch, _ = synth.sst_shaped_forest(400, 3, leaves=9)
    lin = cx.linearize(d(ch, np.int32), synth.TREE)
    g, _ = synth.grid_dags(60, 9, 9)
    lin2 = cx.linearize(d(g, np.int32), synth.DAG)
    torch.cuda.synchronize()
    print(case, cx.status(lin), cx.status(lin2))
elif case == "cluster_lstm_fused":
    run(synth.TREELSTM, 64, 50, forest(3), synth.TREE, fused=True)
elif case == "cluster_lstm":
    run(synth.TREELSTM, 64, 50, forest(3), synth.TREE, path="cluster")
elif case == "cluster_dag_fused":
    run(synth.DAGRNN, 64, 50, synth.grid_dags(2, 4, 4)[0], synth.DAG, fused=True)
elif case == "rw_gru":
    run(synth.TREEGRU, 64, 50, forest(3), synth.TREE, path="rw")
elif case == "rw_fc":
    run(synth.TREEFC, 64, 50, synth.perfect_forest(2, 3)[0], synth.TREE, path="rw")
elif case == "smem_lstm":
    run(synth.TREELSTM, 64, 50, forest(3), synth.TREE, path="smem")
elif case == "big_lstm":
    run(synth.TREELSTM, 64, 50, forest(3), synth.TREE, path="big")
elif case == "mvrnn":
    run(synth.MVRNN, 16, 50, forest(3), synth.TREE)
elif case == "tc_lstm":
    run(synth.TREELSTM, 128, 50, forest(3), synth.TREE, dtype=cx.BF16, path="tc")
elif case == "tc_dag":
    run(synth.DAGRNN, 128, 50, synth.grid_dags(2, 4, 4)[0], synth.DAG, dtype=cx.BF16, path="tc")
elif case == "tc32_lstm":  # split-fp32 tensor-core kernel, hoisted leaves (2n > V)
    run(synth.TREELSTM, 128, 50, forest(3), synth.TREE, path="tc")
elif case == "tc32_dag":  # split-fp32, hoisted input projection (2n > V)
    run(synth.DAGRNN, 128, 50, synth.grid_dags(2, 4, 4)[0], synth.DAG, path="tc")
elif case == "tc32_dag_nohoist":  # split-fp32, per-node projection (node-order x rows)
    run(synth.DAGRNN, 128, 5000, synth.grid_dags(2, 4, 4)[0], synth.DAG, path="tc")
elif case == "tc32_fc":
    run(synth.TREEFC, 256, 50, synth.perfect_forest(2, 3)[0], synth.TREE, path="tc")
elif case == "single_rnn":
    run(synth.TREERNN, 8, 50, forest(2), synth.TREE, fused=True)
else:
    raise SystemExit(f"unknown case {case}")
