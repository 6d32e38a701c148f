import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, synth
import paper_2011_01383_b200 as cx
from gpu_helpers import dev_i32, lin_to_numpy
bad = []
for B in [1, 10, 20, 40, 60, 80, 100, 120, 128, 140, 200, 300]:
    for seed in (0, 1):
        ch, _ = synth.sst_shaped_forest(B, seed)
        dev = lin_to_numpy(cx.linearize(dev_i32(ch), synth.TREE))
        ref = oracle.linearize(ch, synth.TREE)
        diffs = [f for f in ("perm", "height", "level_begin", "level_size", "children", "roots", "structure")
                 if not np.array_equal(np.asarray(dev[f]), np.asarray(ref[f]))]
        hdr = [f for f in ("num_levels", "num_leaves", "first_leaf", "max_level_size") if dev[f] != ref[f]]
        print(B, seed, ch.shape[1], "DIFF" if diffs or hdr else "ok", diffs, hdr, flush=True)
for g in [10, 40, 80]:
    ch, _ = synth.grid_dags(g)
    dev = lin_to_numpy(cx.linearize(dev_i32(ch), synth.DAG)); ref = oracle.linearize(ch, synth.DAG)
    print("grid", g, "ok" if np.array_equal(dev["perm"], ref["perm"]) and np.array_equal(dev["children"], ref["children"]) else "DIFF")
