"""Timeline of the cluster forward kernel (slots: 0 entry, 1 labels done,
2 leaf phase done, 3+l after level l's cluster barrier, S-1 exit)."""
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
fused = len(sys.argv) > 2 and sys.argv[2] == "fused"  # cx_linearize_forward (slot 20 = lin done)
DT = cx.BF16 if len(sys.argv) > 3 and sys.argv[3] == "bf16" else cx.F32  # bf16: rounded-operand FMA
inp = bench.make_inputs(name, 0, 1)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
children, words, emb = t(inp["children"], np.int32), t(inp["words"], np.int32), t(inp["emb"], np.float32)
weights = [t(w, np.float32) for w in inp["weights"]]
cell, H = inp["cell"], inp["H"]
S = 128
info = cx.launch_info(cell, H)
buf = torch.zeros(info["ctas"] * (S + 2), dtype=torch.int64, device=dev)
lbuf = torch.zeros(32, dtype=torch.int64, device=dev)
L = cx.lib()
L.cx_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
lin = cx.linearize(children, inp["kind"])
cx.forward(cell, H, weights, emb, words, lin)
torch.cuda.synchronize()
def run_once():
    global lin
    L.cx_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), S)
    if fused:
        lin = cx.linearize_forward(children, inp["kind"], cell, H, weights, emb, words, out=lin,
                                   h_out=h, dtype=DT)[0]
    else:
        L.cx_debug_set_lin_trace.argtypes = [ctypes.c_void_p]
        L.cx_debug_set_lin_trace(ctypes.c_void_p(lbuf.data_ptr()))
        cx.linearize(children, inp["kind"], out=lin)
        L.cx_debug_set_lin_trace(None)
        cx.forward(cell, H, weights, emb, words, lin, h_out=h, dtype=DT)
    L.cx_debug_set_trace(None, 0)


h = torch.empty(children.shape[1], H, device=dev)
run_once()
torch.cuda.synchronize()
# graph-replayed like bench.py (trace buffers are baked into the captured launches)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run_once()
for rep in range(3):
    flush.fill_(1.0)
    g.replay()
    torch.cuda.synchronize()
C = info["ctas"]
raw = buf.cpu().numpy().astype(np.int64)
clk = raw[:C * S].reshape(C, S)
gt = raw[C * S:C * S + 2 * C].reshape(C, 2)
MHZ = float(os.environ.get("CX_SM_MHZ", "1965"))
# per CTA: clock64 deltas from its entry mark (slot 0), placed on the common
# time axis by the CTA's entry %globaltimer
t0 = gt[:, 0].min()
tr = np.full((C, S), np.nan)
for c in range(C):
    ok = clk[c] != 0
    tr[c, ok] = (gt[c, 0] - t0) / 1000.0 + (clk[c, ok] - clk[c, 0]) / MHZ
nl = lin.header_dict()["num_levels"]
print(f"{name}: ctas={C} levels={nl} (clock64 marks at {MHZ:.0f} MHz, CTAs aligned by %globaltimer at entry)")
print(f"exit by %globaltimer: min {(gt[:, 1].min() - t0) / 1000:7.2f} max {(gt[:, 1].max() - t0) / 1000:7.2f} us")
for sl, nm in [(0, "entry"), (13, "e: compacted"), (14, "e: gathered"), (15, "e: tiles"), (21, "early leaves"), (20, "lin (fused)"), (1, "level lists"), (17, "push setup"), (18, "leaves ready"), (22, "leaf import"),
               (2, "leaf phase")] + [(3 + l, f"level {l}") for l in range(1, nl)] + [(S - 1, "exit")]:
    col = tr[:, sl]
    ok = ~np.isnan(col)
    if not ok.any():
        continue
    print(f"{nm:13s} min {col[ok].min():7.2f} max {col[ok].max():7.2f}")
print("first tile of each level, mean over CTAs with a tile (us): start->waited, waited->contracted, "
      "contracted->epilogue math (warp 0), ->pushed")
for l in range(1, nl):
    b = 24 + 5 * l
    blk = tr[:, [b, b + 1, b + 3, b + 2, b + 4]]
    ok = ~np.isnan(blk).any(axis=1)
    if ok.any():
        d = np.diff(blk[ok], axis=1).mean(axis=0)
        mx = np.diff(blk[ok], axis=1).max(axis=0)
        print(f"level {l:2d}: " + "  ".join(f"{x:5.2f}" for x in d) + "   max " + "  ".join(f"{x:5.2f}" for x in mx))
