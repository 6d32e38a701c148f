"""Fixed-overhead experiment: graph-replayed linearize / forward on tiny and
headline inputs, with and without an L2 flush between replays."""
import os as _os
_os.environ.setdefault("CX_TRACE", "1")  # debug timeline build (libcx_trace.so)
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2011_01383_b200 as cx  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def timeit(fn, reps=100, do_flush=True):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if do_flush:
            flush.fill_(1.0)
        e0.record()
        g.replay()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
    return v[len(v) // 2]


def case(name, ch, kind, cell=synth.TREELSTM, H=256, V=20000):
    words = synth.word_ids(ch, V, 0, all_nodes=(cell == synth.DAGRNN))
    emb = t(synth.embedding(V, H, 0), np.float32)
    ws = [t(w, np.float32) for _, w in synth.weights(cell, H, V)]
    chd, wd = t(ch, np.int32), t(words, np.int32)
    lin = cx.alloc_linearization(ch.shape[1], ch.shape[0], kind, dev)
    h = torch.empty(ch.shape[1], H, device=dev)
    cx.linearize(chd, kind, out=lin)
    cx.forward(cell, H, ws, emb, wd, lin, h_out=h)
    torch.cuda.synchronize()
    lin_f = lambda: cx.linearize(chd, kind, out=lin)
    fwd_f = lambda: cx.forward(cell, H, ws, emb, wd, lin, h_out=h)
    both = lambda: (lin_f(), fwd_f())
    for fl in (True, False):
        print(f"{name:28s} flush={fl!s:5s} lin {timeit(lin_f, do_flush=fl):7.2f} us  "
              f"fwd {timeit(fwd_f, do_flush=fl):7.2f} us  both {timeit(both, do_flush=fl):7.2f} us")


if __name__ == "__main__":
  case("treelstm N=1", np.full((2, 1), -1, np.int32), synth.TREE)
  case("treelstm N=3", np.array([[1, -1, -1], [2, -1, -1]], np.int32), synth.TREE)
  w = synth.workload("cfg2_treelstm_b10")
  case("treelstm b10 (N=390)", w["children"], w["kind"])
  case("treernn b10 H=256", w["children"], w["kind"], cell=synth.TREERNN)
  os.environ["CX_FORWARD_PATH"] = "smem"
  case("treelstm b10 smem-path", w["children"], w["kind"])

  # ---- launch overhead of an empty kernel, and the linearizer phase timeline
  import ctypes  # noqa: E402
  L = cx.lib()
  L.cx_debug_empty.argtypes = [ctypes.c_int32] * 3 + [ctypes.c_void_p, ctypes.c_void_p]
  L.cx_debug_set_lin_trace.argtypes = [ctypes.c_void_p]
  st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
  for ctas, thr, coop in ((1, 32, 0), (1, 1024, 0), (144, 512, 0), (144, 512, 1), (148, 1024, 1)):
      us = timeit(lambda: L.cx_debug_empty(ctas, thr, coop, None, st()))
      print(f"empty kernel ctas={ctas:3d} threads={thr:4d} coop={coop}: {us:6.2f} us")
  buf = torch.zeros(32, dtype=torch.int64, device=dev)
  for name, ch, kind in (("N=1", np.full((2, 1), -1, np.int32), synth.TREE),
                         ("b10", w["children"], w["kind"])):
      chd = t(ch, np.int32)
      lin = cx.alloc_linearization(ch.shape[1], 2, kind, dev)
      cx.linearize(chd, kind, out=lin)
      torch.cuda.synchronize()
      L.cx_debug_set_lin_trace(ctypes.c_void_p(buf.data_ptr()))
      for _ in range(3):
          cx.linearize(chd, kind, out=lin)
      torch.cuda.synchronize()
      L.cx_debug_set_lin_trace(None)
      tr = buf.cpu().numpy()
      print(name, "lin phases (us from entry):", [round((tr[i] - tr[0]) / 1000, 2) for i in range(7)])
      print(name, "lin phases (cycles from entry):", [int(tr[8 + i] - tr[8]) for i in range(7)])
