"""Per-level synchronisation and dependent-chain costs on this device
(cx_diag_sync_cycles + the empty-kernel launch floor), as JSON:
    python tools/sync_costs.py > profiles/r02_sync_costs.json"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402

dev = torch.device("cuda", 0)
mhz = float(os.environ.get("CX_SM_MHZ", "1965"))
out = {"device": torch.cuda.get_device_name(0), "sm_mhz_assumed": mhz, "kinds": {}}
for k, nm in [(0, "push"), (1, "cluster_barrier"), (2, "grid_barrier"), (3, "chain")]:
    reps = [cx.diag_sync_cycles(k, 4000 if k != 2 else 1000, dev) for _ in range(5)]
    out["kinds"][nm] = {"cycles_per_level": reps, "us_median": sorted(reps)[2] / mhz,
                        "what": bench.SYNC_KINDS.get(k, "dependent arithmetic of one level (H=256, one warp)")}
out["launch_floor_us"] = {"1_launch": bench.launch_floor_us(1, dev), "2_launches": bench.launch_floor_us(2, dev)}
print(json.dumps(out, indent=1))
