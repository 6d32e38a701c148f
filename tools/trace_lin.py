"""Phase timeline of cx_linearize (debug trace: %globaltimer and clock64 per
phase of CTA 0; slots 0..7 = lin_mark calls in linearize.cu).

    python tools/trace_lin.py [workload]
"""
import os as _os
_os.environ.setdefault("CX_TRACE", "1")  # debug timeline build (libcx_trace.so)
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_treelstm_b10"
inp = bench.make_inputs(name, 0, 1)
dev = torch.device("cuda", 0)
children = torch.as_tensor(np.ascontiguousarray(inp["children"], dtype=np.int32)).to(dev)
buf = torch.zeros(32, dtype=torch.int64, device=dev)
L = cx.lib()
L.cx_debug_set_lin_trace.argtypes = [ctypes.c_void_p]
lin = cx.linearize(children, inp["kind"])
torch.cuda.synchronize()
rows = []
for rep in range(20):
    buf.zero_()
    L.cx_debug_set_lin_trace(ctypes.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cx.linearize(children, inp["kind"], out=lin)
    e1.record()
    L.cx_debug_set_lin_trace(None)
    torch.cuda.synchronize()
    t = buf.cpu().numpy()
    rows.append((e0.elapsed_time(e1) * 1e3, t[:16].copy(), t[16:32].copy()))
ev = np.median([r[0] for r in rows])
t = np.median(np.stack([r[1] for r in rows]).astype(np.float64), axis=0)
c = np.median(np.stack([r[2] for r in rows]).astype(np.float64), axis=0)
print(f"{name}: n={children.shape[1]} event time {ev:.1f} us (median of 20, includes launch)")
names = ["load+init", "a1 validate", "a2 heights", "a3 counts", "a3 scans", "a4 scatter", "a5/a6 remap+sid"]
for k in range(1, 7):
    if t[k] and t[k - 1]:
        print(f"  {names[k-1]:18s} {(t[k]-t[k-1])/1000:6.2f} us  {(c[k]-c[k-1]):8.0f} cycles")

mnames = ["entry", "P0 init", "P1 validate+parents", "P2+P3 kind, heights", "P4 counts",
          "P5 offsets", "P6 scatter", "P7 remap", "P8 structures + header"]
if t[7]:
    print("multi-CTA phases (CTA 0):")
    for k in range(8, 16):
        if t[k] and t[k - 1]:
            print(f"  {mnames[k-7]:24s} {(t[k]-t[k-1])/1000:7.2f} us")
