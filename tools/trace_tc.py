"""Per-level timeline of one bf16 tensor-core cx_forward launch (debug trace,
%globaltimer per CTA; slots documented at tc_mark in forward_tc.cu).

    python tools/trace_tc.py [workload]
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

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_treelstm_b4096"
DT = cx.F32 if len(sys.argv) > 2 and sys.argv[2] == "f32" else cx.BF16  # f32: the split-fp32 kernel
inp = bench.make_inputs(name, 0, 1)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
children, words, emb = t(inp["children"], np.int32), t(inp["words"], np.int32), t(inp["emb"], np.float32)
weights = [t(w, np.float32) for w in inp["weights"]]
cell, H = inp["cell"], inp["H"]
S = 256
info = cx.linearize_forward_launch_info(cell, H, inp["children"].shape[1], inp["children"].shape[0],
                                        inp["V"], DT)
buf = torch.zeros(info["ctas"] * (S + 2), dtype=torch.int64, device=dev)
L = cx.lib()
L.cx_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for rep in range(4):
    flush.fill_(1.0)
    lin = cx.linearize(children, inp["kind"])
    buf.zero_()
    L.cx_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), S)
    cx.forward(cell, H, weights, emb, words, lin, dtype=DT)
    L.cx_debug_set_trace(None, 0)
    torch.cuda.synchronize()
tr = buf[: info["ctas"] * S].view(info["ctas"], S).cpu().numpy().astype(np.int64)
hdr = lin.header_dict()
nl = hdr["num_levels"]
sizes = lin.level_size[:nl].cpu().numpy()
t0 = tr[:, 0].min()
rel = lambda x: (x - t0) / 1000.0
print(f"{name} {'f32 (split)' if DT == cx.F32 else 'bf16'}: ctas={info['ctas']} levels={nl} (us from earliest CTA entry)")
print(f"weights staged: min {rel(tr[:,60].min()):8.2f} max {rel(tr[:,60].max()):8.2f}; phase 0 done: max {rel(tr[:,61].max()):8.2f}")
print(f"prologue done: min {rel(tr[:,1].min()):8.2f} max {rel(tr[:,1].max()):8.2f}")
for l in range(nl):
    st, pr, mm, ep = (tr[:, 2 + 4 * l + k] for k in range(4))
    f = lambda v: f"{rel(v[v > 0].max()):8.2f}" if (v > 0).any() else "     -  "
    g = lambda v: f"{rel(v[v > 0].min()):8.2f}" if (v > 0).any() else "     -  "
    print(f"level {l:2d} M={sizes[l]:6d}: start {g(st)}..{f(st)}  prod done max {f(pr)}  "
          f"mma done max {f(mm)}  epi done min {g(ep)} max {f(ep)}")

if (tr[:, 63] > 0).any():
    print(f"leaf output copy: start max {rel(tr[:,62].max()):8.2f} end max {rel(tr[:,63].max()):8.2f}")
print("per-tile role timestamps, CTA 0 (us rel. to level start): prod [start,end] mma [start,end] epi [start,end]")
for l in range(2):
    ls = tr[0, 2 + 4 * l]
    for t_ in range(5):
        b = 128 + 12 * (t_ + 5 * l)
        v = tr[0, b:b + 6]
        if (v == 0).all():
            continue
        print(f"  level {l} tile {t_}: " + " ".join(f"{(x - ls) / 1000:7.2f}" if x else "    -  " for x in v))

print("per-stage, CTA 0, level 1 (us rel. to level start): TMA after empty-wait, TMA issued, MMA after full-wait, MMA committed")
ls = tr[0, 2 + 4 * 1]
for k in range(16):
    v = tr[0, 64 + 4 * k: 64 + 4 * k + 4]
    if (v == 0).all():
        continue
    print(f"  stage {k:2d}: " + " ".join(f"{(x - ls) / 1000:7.2f}" if x else "    -  " for x in v))
