"""Timeline of the fused single-CTA kernel (forward_single.cu), clock64 marks:
0 entry, 20 linearized, 21 setup, 22 leaves, 2+l after the band starting at l, S-1 exit."""
import os as _os
_os.environ.setdefault("CX_TRACE", "1")
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1_treernn"
inp = bench.make_inputs(name, 0, 1)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
children, words, emb = t(inp["children"], np.int32), t(inp["words"], np.int32), t(inp["emb"], np.float32)
weights = [t(w, np.float32) for w in inp["weights"]]
cell, H = inp["cell"], inp["H"]
n = children.shape[1]
info = cx.linearize_forward_launch_info(cell, H, n, children.shape[0], inp["V"])
C, S = info["ctas"], 64
buf = torch.zeros(C * (S + 2), dtype=torch.int64, device=dev)
L = cx.lib()
L.cx_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
lin = cx.alloc_linearization(n, children.shape[0], inp["kind"], dev)
h = torch.empty(n, H, device=dev)


def run_once():
    L.cx_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), S)
    cx.linearize_forward(children, inp["kind"], cell, H, weights, emb, words, out=lin, h_out=h)
    L.cx_debug_set_trace(None, 0)


run_once()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run_once()
for _ in range(3):
    flush.fill_(1.0)
    g.replay()
    torch.cuda.synchronize()
raw = buf.cpu().numpy().astype(np.int64)
clk = raw[:C * S].reshape(C, S)
MHZ = 1965.0
print(f"{name}: ctas={C} levels={lin.header_dict()['num_levels']}")
for sl, nm in [(20, "linearized"), (21, "setup"), (22, "leaves")] + [(2 + l, f"band @{l}") for l in range(1, 20)] + [(S - 1, "exit")]:
    col = clk[:, sl]
    ok = col != 0
    if ok.any():
        d = (col[ok] - clk[ok, 0]) / MHZ
        print(f"{nm:12s} {d.min():7.2f} .. {d.max():7.2f} us after entry")
