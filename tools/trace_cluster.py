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
inp = bench.make_inputs(name, 0, 1)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
children, words, emb = t(inp["children"], np.int32), t(inp["words"], np.int32), t(inp["emb"], np.float32)
weights = [t(w, np.float32) for w in inp["weights"]]
cell, H = inp["cell"], inp["H"]
S = 128
info = cx.launch_info(cell, H)
buf = torch.zeros(info["ctas"] * S, dtype=torch.int64, device=dev)
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
                                   h_out=h)[0]
    else:
        L.cx_debug_set_lin_trace.argtypes = [ctypes.c_void_p]
        L.cx_debug_set_lin_trace(ctypes.c_void_p(lbuf.data_ptr()))
        cx.linearize(children, inp["kind"], out=lin)
        L.cx_debug_set_lin_trace(None)
        cx.forward(cell, H, weights, emb, words, lin, h_out=h)
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
tr = buf.view(info["ctas"], S).cpu().numpy().astype(np.int64)
nl = lin.header_dict()["num_levels"]
t0 = tr[:, 0].min()
rel = lambda x: (x - t0) / 1000.0
print(f"{name}: ctas={info['ctas']} levels={nl}")
if not fused:
    lt = lbuf.cpu().numpy().astype(np.int64)
    print(f"cx_linearize (CTA 0): entry {rel(lt[0]):7.2f}  end {rel(lt[6]):7.2f} us (relative to the forward's entry)")
for sl, nm in [(0, "entry"), (20, "lin (fused)"), (1, "labels"), (12, "leaf words"), (13, "leaf gather"), (2, "leaf phase")] + [(3 + l, f"level {l}") for l in range(1, nl)] + [(S - 1, "exit")]:
    col = tr[:, sl]
    ok = col > 0
    if not ok.any():
        continue
    print(f"{nm:12s} min {rel(col[ok].min()):7.2f} max {rel(col[ok].max()):7.2f}")
print("first tile of each level, mean over CTAs with a tile (us): list->meta, meta->pulled, pulled->contracted, ->epilogue")
for l in range(1, nl):
    b = 24 + 5 * l
    blk = tr[:, b:b + 5]
    ok = (blk > 0).all(axis=1)
    if ok.any():
        d = np.diff(blk[ok], axis=1).mean(axis=0) / 1000
        pre = (blk[ok][:, 0] - tr[ok, 2 + l]).mean() / 1000 if l > 1 else (blk[ok][:, 0] - tr[ok, 2]).mean() / 1000
        print(f"level {l}: barrier->list {pre:5.2f}  " + "  ".join(f"{x:5.2f}" for x in d))
