"""Per-level timeline of one cx_forward launch (debug trace, %globaltimer per CTA).

    python tools/trace_forward.py [workload]
Slots: 0 entry, 1 leaf weights staged, 2 leaf phase done, 3+2j / 4+2j arrive / exit of
barrier j, 64+5j.. first-tile breakdown of level j (meta, gather, fma, reduce, end),
S-2 loop end, S-1 exit.
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
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
children, words, emb = t(inp["children"], np.int32), t(inp["words"], np.int32), t(inp["emb"], np.float32)
weights = [t(w, np.float32) for w in inp["weights"]]
cell, H = inp["cell"], inp["H"]
S = 256
info = cx.launch_info(cell, H)
buf = torch.zeros(info["ctas"] * (S + 2), dtype=torch.int64, device=dev)
L = cx.lib()
L.cx_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
lin = cx.linearize(children, inp["kind"])
cx.forward(cell, H, weights, emb, words, lin)
torch.cuda.synchronize()
res = []
for rep in range(5):
    flush.fill_(1.0)
    lin = cx.linearize(children, inp["kind"])
    L.cx_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), S)
    cx.forward(cell, H, weights, emb, words, lin)
    L.cx_debug_set_trace(None, 0)
    torch.cuda.synchronize()
    res.append(buf.view(info["ctas"], S).cpu().numpy().copy())
tr = res[-1].astype(np.int64)
hdr = lin.header_dict()
nl = hdr["num_levels"]
phases = 2 if cell == cx.TREEGRU else 1
t0 = tr[:, 0].min()
rel = lambda x: (x - t0) / 1000.0
print(f"{name}: ctas={info['ctas']} levels={nl} (us from earliest CTA entry)")
print(f"entry        min {rel(tr[:,0].min()):7.2f} max {rel(tr[:,0].max()):7.2f}")
print(f"leaf weights min {rel(tr[:,1].min()):7.2f} max {rel(tr[:,1].max()):7.2f}")
print(f"leaf done    min {rel(tr[:,2].min()):7.2f} max {rel(tr[:,2].max()):7.2f}")
lt = tr[:, 59:64]
okl = (lt > 0).all(axis=1)
if okl.any():
    d = np.diff(lt[okl], axis=1).mean(axis=0) / 1000
    m0 = (lt[okl][:, 0] - tr[okl, 1]).mean() / 1000
    print(f"first leaf tile: meta {m0:5.2f} gather {d[0]:5.2f} fma {d[1]:5.2f} red {d[2]:5.2f} epi {d[3]:5.2f}")
for j in range((nl - 1) * phases):
    arr, ex = tr[:, 3 + 2 * j], tr[:, 4 + 2 * j]
    b = 64 + 5 * j
    tile = tr[:, b:b + 5]
    ok = (tile > 0).all(axis=1)
    line = (f"barrier {j:2d}: arrive min {rel(arr.min()):7.2f} max {rel(arr.max()):7.2f} | "
            f"exit min {rel(ex.min()):7.2f} max {rel(ex.max()):7.2f} (last-arrive->first-exit "
            f"{(ex.min()-arr.max())/1000:5.2f})")
    if ok.any():
        d = np.diff(tile[ok], axis=1).mean(axis=0) / 1000
        m0 = (tile[ok][:, 0] - ex[ok]).mean() / 1000
        line += f" | tile: meta {m0:5.2f} gather {d[0]:5.2f} fma {d[1]:5.2f} red {d[2]:5.2f} epi {d[3]:5.2f}"
    print(line)
print(f"loop end     min {rel(tr[:,S-2].min()):7.2f} max {rel(tr[:,S-2].max()):7.2f}")
print(f"exit         min {rel(tr[:,S-1].min()):7.2f} max {rel(tr[:,S-1].max()):7.2f}")
