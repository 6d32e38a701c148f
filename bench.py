#!/usr/bin/env python
"""Benchmark of the Cortex hot path on B200.

One step = cx_linearize_forward over one batch of synthetic structures (the
whole hot path, reading Q17 of DESIGN.md): the linearizer fused into the
forward kernel, one launch, where the batch allows it, else
cx_linearize + cx_forward. Default workload =
BASELINE.json configs[1]: TreeLSTM (child-sum, binary SST-shaped trees),
batch 10 per GPU, H = 256, fp32. Multi-GPU: one process per GPU (torchrun),
each rank evaluates its own independent batch (weak scaling, no data-path
collective); timing is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
    python bench.py --impl reference ...   # the CPU oracle on the host cores
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "TreeLSTM fwd latency µs (batch 10, H=256) and trees/s at 1/2/4/8 B200"
UNIT = "trees/s"
FMA_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4: SMs x FP32 lanes x 2 x max clock

WORKLOADS = {
    # name: (generator, cell, hidden, vocab, per-GPU batch or total batch, scaling)
    "cfg2_treelstm_b10": ("sst", synth.TREELSTM, 256, 20000, 10, "weak"),
    "cfg2_treelstm_b1": ("sst", synth.TREELSTM, 256, 20000, 1, "weak"),
    "cfg3_treegru_b10": ("sst", synth.TREEGRU, 512, 20000, 10, "weak"),
    "cfg3_treegru_b1": ("sst", synth.TREEGRU, 512, 20000, 1, "weak"),
    "cfg3_treefc_b10": ("perfect7", synth.TREEFC, 512, 20000, 10, "weak"),
    "cfg3_treefc_b1": ("perfect7", synth.TREEFC, 512, 20000, 1, "weak"),
    "cfg4_mvrnn_b10": ("sst", synth.MVRNN, 64, 20000, 10, "weak"),
    "cfg5_dagrnn_b10": ("grid", synth.DAGRNN, 256, 20000, 10, "weak"),
    "cfg5_dagrnn_b1": ("grid", synth.DAGRNN, 256, 20000, 1, "weak"),
    "cfg1_treernn": ("perfect3", synth.TREERNN, 8, 100, 1, "weak"),
    # GRNN-comparison sequences (length 100, H = 256)
    "f4_lstm_seq100_b10": ("chain100", synth.TREELSTM, 256, 20000, 10, "weak"),
    "f4_lstm_seq100_b1": ("chain100", synth.TREELSTM, 256, 20000, 1, "weak"),
    "f4_gru_seq100_b10": ("chain100", synth.TREEGRU, 256, 20000, 10, "weak"),
    "f4_gru_seq100_b1": ("chain100", synth.TREEGRU, 256, 20000, 1, "weak"),
    # strong scaling: the batch is split across ranks
    "cfg5_treelstm_b4096": ("sst", synth.TREELSTM, 256, 20000, 4096, "strong"),
    "cfg5_dagrnn_b4096": ("grid", synth.DAGRNN, 256, 20000, 4096, "strong"),
}


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------
def make_inputs(name, rank, world, seed=0):
    gen, cell, H, V, batch, scaling = WORKLOADS[name]
    total = batch * world if scaling == "weak" else batch
    if gen == "sst":
        ch, off = synth.sst_shaped_forest(total, seed)
    elif gen == "perfect7":
        ch, off = synth.perfect_forest(total, 7)
    elif gen == "perfect3":
        ch, off = synth.perfect_forest(total, 3)
    elif gen == "chain100":
        ch, off = synth.chains(total, 100)
    else:
        ch, off = synth.grid_dags(total)
    kind = synth.DAG if gen == "grid" else synth.SEQUENCE if gen == "chain100" else synth.TREE
    # this rank's contiguous block of structures, ids rebased to 0 (shard.py)
    from paper_2011_01383_b200 import shard
    words_all = synth.word_ids(ch, V, seed, all_nodes=(cell == synth.DAGRNN))
    sub, words, (g0, g1), a = shard.shard(ch, off, rank, world, words_all)
    emb = synth.embedding(V, H, seed)
    ws = [w for _, w in synth.weights(cell, H, V)]
    return dict(children=sub, kind=kind, words=words, emb=emb, weights=ws, cell=cell, H=H, V=V,
                batch=g1 - g0, total=total, scaling=scaling, offsets=off[g0:g1 + 1] - a,
                g0=g0, g1=g1)


def algorithmic_work(cell, H, n, n_leaves, n_internal, batch, maxc=2):
    """Algorithmic flops and bytes per step."""
    leaf_f = {synth.TREELSTM: 6 * H * H, synth.TREEGRU: 4 * H * H, synth.DAGRNN: 2 * H * H}.get(cell, 0)
    int_f = {synth.TREERNN: H, synth.TREEFC: 4 * H * H, synth.TREELSTM: 10 * H * H,
             synth.TREEGRU: 8 * H * H, synth.MVRNN: 4 * H ** 3 + 8 * H * H,
             synth.DAGRNN: 2 * H * H}[cell]
    flops = leaf_f * n_leaves + int_f * n_internal
    if cell == synth.DAGRNN:
        flops += 2 * H * H * n_internal  # every node has an input projection
    emb_rows = n if cell == synth.DAGRNN else n_leaves
    bytes_ = 4 * maxc * n + 4 * n + 4 * H * emb_rows + 4 * H * n  # children, words, Emb, h_out
    if cell == synth.MVRNN:
        bytes_ += 4 * H * H * n_leaves
    return flops, bytes_


def measured_peaks():
    """MEASURED_PEAKS.json (driver-written, per pod) or None."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polling thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.NAMES.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle on the host cores
# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    name = args.workload
    inp = make_inputs(name, 0, 1)
    gen, cell, H, V, batch, scaling = WORKLOADS[name]
    ch, off = inp["children"], inp["offsets"]
    # bounded sample: at most `cap` structures per step (whole batch when small)
    cap = 16 if batch > 64 else batch
    a, b = 0, int(off[cap])
    sub, words = ch[:, a:b], inp["words"][a:b]
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        lin = oracle.linearize(sub, inp["kind"])
        st, _, _, _ = oracle.forward(cell, H, V, inp["weights"], inp["emb"], words, sub)
        t1 = time.perf_counter()
        assert lin["status"] == 0 and st == 0
        if i >= args.warmup:
            times.append(t1 - t0)
    per = sum(times) / len(times)
    value = cap / per
    sample = f"{cap} of {batch} structures of {name} per step (oracle linearize + forward, fp64)"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": name, "batch_per_step": cap, "hidden": H},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(name, seconds=12.0):
    """The oracle as it stands, timed on one host core, on a bounded sample."""
    import oracle
    inp = make_inputs(name, 0, 1)
    gen, cell, H, V, batch, _ = WORKLOADS[name]
    cap = min(batch, 16)
    b = int(inp["offsets"][cap])
    sub, words = inp["children"][:, :b], inp["words"][:b]
    done, t0 = 0, time.perf_counter()
    while True:
        lin = oracle.linearize(sub, inp["kind"])
        oracle.forward(cell, H, V, inp["weights"], inp["emb"], words, sub)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds or (done >= 3 and el * (done + 1) / done > seconds * 1.5):
            break
    return {"value": done * cap / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{done} x {cap} structures of {name} in {el:.1f}s (fp64 naive recursion, 1 thread)"}


# ---------------------------------------------------------------------------
# secondary: batch-4096 throughput (SURVEY §8(d) "headline trees/s = cfg5b")
# ---------------------------------------------------------------------------
def throughput_b4096(dtype_name, rank, world, local_rank, steps=30, warmup=5):
    """cx_linearize + cx_forward over this rank's block of the 4096 SST trees
    (strong scaling), CUDA-graph replayed, L2 flushed between steps, events on
    the launch stream; trees/s = 4096 / max-over-ranks mean step time."""
    import torch
    import torch.distributed as dist
    import paper_2011_01383_b200 as cx
    name = "cfg5_treelstm_b4096"
    dev = torch.device("cuda", local_rank)
    inp = make_inputs(name, rank, world)
    cell, H = inp["cell"], inp["H"]
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
    children, words = t(inp["children"], np.int32), t(inp["words"], np.int32)
    emb = t(inp["emb"], np.float32)
    weights = [t(w, np.float32) for w in inp["weights"]]
    n = inp["children"].shape[1]
    dtype = cx.BF16 if dtype_name == "bf16" else cx.F32
    lin = cx.alloc_linearization(n, inp["children"].shape[0], inp["kind"], dev)
    h = torch.empty(n, H, dtype=torch.float32, device=dev)
    roots = torch.empty(inp["batch"], H, dtype=torch.float32, device=dev)

    def step():
        cx.linearize(children, inp["kind"], out=lin)
        cx.forward(cell, H, weights, emb, words, lin, dtype=dtype, h_out=h, root_out=roots)

    step()
    cx.check(lin)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        g.replay()
        flush.fill_(1.0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for a0, a1 in evs:
        a0.record(stream)
        g.replay()
        a1.record(stream)
        flush.fill_(1.0)
    torch.cuda.synchronize()
    total = sum(a0.elapsed_time(a1) for a0, a1 in evs)
    if world > 1:
        tt = torch.tensor([total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    ms = total / steps
    return {"workload": name, "dtype": dtype_name, "trees_per_s": inp["total"] / (ms / 1e3),
            "ms_per_step": ms, "trees": inp["total"], "trees_per_gpu": inp["batch"],
            "scaling": "strong", "timing": "graph replay of linearize+forward, max over ranks"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2011_01383_b200 as cx

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    name = args.workload
    inp = make_inputs(name, rank, world)
    cell, H, V = inp["cell"], inp["H"], inp["V"]
    ch_np = inp["children"]
    n = ch_np.shape[1]
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
    children = t(ch_np, np.int32)
    words = t(inp["words"], np.int32)
    emb = t(inp["emb"], np.float32)
    weights = [t(w, np.float32) for w in inp["weights"]]
    R = inp["batch"]
    stream = torch.cuda.current_stream()

    # preallocated outputs (reused every step; no allocation inside a step)
    lin = cx.alloc_linearization(n, ch_np.shape[0], inp["kind"], dev)
    h = torch.empty(n, H, dtype=torch.float32, device=dev)
    roots = torch.empty(R, H, dtype=torch.float32, device=dev)
    dtype = cx.BF16 if args.dtype == "bf16" else cx.F32
    cx.linearize(children, inp["kind"], out=lin)
    cx.forward(cell, H, weights, emb, words, lin, dtype=dtype, h_out=h, root_out=roots)
    cx.check(lin)
    hdr = lin.header_dict()
    L = hdr["num_levels"]
    n_leaves = hdr["num_leaves"]

    def lin_call():
        cx.linearize(children, inp["kind"], out=lin)

    def fwd_call():
        cx.forward(cell, H, weights, emb, words, lin, dtype=dtype, h_out=h, root_out=roots)

    # one step = cx_linearize_forward: ONE launch (linearizer fused into the
    # forward kernel) where it applies, else the two kernels
    fused = cx.fused_applies(cell, H, n, ch_np.shape[0], V, dtype)
    ws_lf = torch.zeros(cx.lib().cx_linearize_forward_workspace_bytes(
        ctypes.byref(cx._cx._model(cell, H, V, dtype)), n, ch_np.shape[0]), dtype=torch.uint8,
        device=dev)

    def step():
        cx.linearize_forward(children, inp["kind"], cell, H, weights, emb, words, dtype=dtype,
                             out=lin, h_out=h, root_out=roots, workspace=ws_lf)

    def step2():
        lin_call()
        fwd_call()

    step()
    cx.check(lin)

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    # one step = one CUDA graph (2 kernel nodes); breakdown graphs for each call
    g_step, g_lin, g_fwd = capture(step), capture(lin_call), capture(fwd_call)
    g_step2 = capture(step2)
    stream = torch.cuda.current_stream()

    # L2 flush buffer (> 126 MB L2): written between timed steps, outside the events
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    for _ in range(args.warmup):
        g_step.replay()
        flush.fill_(1.0)
    torch.cuda.synchronize()

    # timed region: K graph replays, per-step events, flush between steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    with sampler:
        for k in range(args.steps):
            ev[k][0].record(stream)
            g_step.replay()
            ev[k][1].record(stream)
            flush.fill_(1.0)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
    total_ms = sum(step_ms)
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    trees_total = inp["batch"] * world if inp["scaling"] == "weak" else inp["total"]
    value = trees_total / (ms_per_step / 1e3)

    # breakdown: linearize and forward graphs timed separately (same protocol)
    nb = min(args.steps, 200)
    evb = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(nb)]
    for k in range(nb):
        evb[k][0].record(stream)
        g_lin.replay()
        evb[k][1].record(stream)
        g_fwd.replay()
        evb[k][2].record(stream)
        flush.fill_(1.0)
    torch.cuda.synchronize()
    lin_ms = [evb[k][0].elapsed_time(evb[k][1]) for k in range(nb)]
    fwd_ms = [evb[k][1].elapsed_time(evb[k][2]) for k in range(nb)]
    # the two-launch step (cx_linearize + cx_forward graph), for comparison
    ev2 = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(nb)]
    for k in range(nb):
        ev2[k][0].record(stream)
        g_step2.replay()
        ev2[k][1].record(stream)
        flush.fill_(1.0)
    torch.cuda.synchronize()
    two_ms = [ev2[k][0].elapsed_time(ev2[k][1]) for k in range(nb)]

    # eager (no graph) latency through the Python API, for reference
    eager_ms = []
    for k in range(min(args.steps, 100)):
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        step()
        a1.record(stream)
        flush.fill_(1.0)
        eager_ms.append((a0, a1))
    torch.cuda.synchronize()
    eager_ms = [x.elapsed_time(y) for x, y in eager_ms]

    # optional NCCL all-gather of the packed root states (the only collective)
    allgather_us = None
    if world > 1 and args.allgather:
        from paper_2011_01383_b200 import shard
        for _ in range(3):
            shard.all_gather_roots(roots, inp["total"])
        torch.cuda.synchronize()
        dist.barrier()
        ag = []
        for _ in range(50):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            shard.all_gather_roots(roots, inp["total"])
            a1.record(stream)
            ag.append((a0, a1))
        torch.cuda.synchronize()
        allgather_us = statistics.median(x.elapsed_time(y) for x, y in ag) * 1e3

    # ---- end to end through the public API with host buffers --------------
    # the step's inputs packed in one pinned buffer (children [maxc, n] then words [n]):
    # one H2D copy per step; the device views are what the API call takes
    maxc_ = ch_np.shape[0]
    in_host = torch.as_tensor(np.ascontiguousarray(np.concatenate(
        [np.asarray(ch_np, np.int32).ravel(), np.asarray(inp["words"], np.int32)]))).pin_memory()
    in_dev = torch.empty_like(in_host, device=dev)
    roots_host = torch.empty((R, H), dtype=torch.float32).pin_memory()
    ch_dev = in_dev[:maxc_ * n].view(maxc_, n)
    w_dev = in_dev[maxc_ * n:]
    e2e_steps = max(5, min(args.steps, 200))
    # the serving form of the public API: a prepared cx_linearize_forward call
    # on fixed device buffers (one C call per step)
    plan = cx.LinearizeForwardPlan(ch_dev, inp["kind"], cell, H, weights, emb, w_dev,
                                   dtype=dtype, num_roots=R)
    for _ in range(3):
        in_dev.copy_(in_host, non_blocking=True)
        plan()
        roots_host.copy_(plan.root_out, non_blocking=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = []
    for _ in range(e2e_steps):
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        in_dev.copy_(in_host, non_blocking=True)
        plan()
        roots_host.copy_(plan.root_out, non_blocking=True)
        s1.record(stream)
        s1.synchronize()  # the host reads the step's result
        e2e_ms.append(s0.elapsed_time(s1))
        flush.fill_(1.0)
    torch.cuda.synchronize()
    e2e_total = sum(e2e_ms)
    if world > 1:
        tt = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_total = float(tt.item())
    e2e_value = trees_total / (e2e_total / e2e_steps / 1e3)
    h2d = in_host.numel() * 4
    d2h = roots_host.numel() * 4

    secondary = None
    if args.secondary and name == "cfg2_treelstm_b10":
        secondary = [throughput_b4096(dt, rank, world, local_rank) for dt in ("bf16", "f32")]

    if rank != 0:
        return
    # the dominant kernel: the fused kernel (= the whole step) or cx_forward's
    fwd_mean = sum(step_ms) / len(step_ms) if fused else sum(fwd_ms) / len(fwd_ms)
    flops, alg_bytes = algorithmic_work(cell, H, n, n_leaves, n - n_leaves, R, ch_np.shape[0])
    achieved = flops / (fwd_mean / 1e3) / 1e12
    info = cx.launch_info(cell, H, V, dtype)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "forward_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(
                f"{name}:fused" if fused else name if args.dtype == "f32" else f"{name}:bf16")
        except Exception:
            traffic = None
    if args.dtype == "bf16":
        peaks = measured_peaks()
        peak, src = (peaks["bf16_tflops"], "MEASURED_PEAKS.json bf16_tflops (burst)") if peaks \
            else (2250.0, "B200 nominal dense bf16 (MEASURED_PEAKS.json absent)")
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "kernel": "tc_kernel (cx_forward, dtype bf16)", "flops_per_launch": flops,
                    "alg_bytes_per_launch": alg_bytes,
                    "hbm_frac": alg_bytes / (fwd_mean / 1e3) / 1e9 /
                                (peaks["hbm_gbs"] if peaks else 7700.0),
                    "note": f"peak = {src}; algorithmic flops (SURVEY 8(d)), not the MMA's "
                            "(child-sum by linearity issues 16H^2 per TreeLSTM node)"}
    else:
        roofline = {"bound": "alu", "achieved": achieved, "peak": FMA_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": achieved / FMA_PEAK_TFLOPS, "traffic": traffic,
                    "kernel": "ck_kernel<fused> (cx_linearize_forward, one launch per step)"
                              if fused else "fwd_kernel (cx_forward)", "flops_per_launch": flops,
                    "alg_bytes_per_launch": alg_bytes,
                    "note": "fp32 FMA peak = 148 SM x 128 lanes x 2 x 1.965 GHz; the step is "
                            "critical-path (levels x barrier) bound, see DESIGN.md"}
    clocks = sampler.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": inp["scaling"], "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": name, "cell": synth.CELL_NAMES[cell], "hidden": H, "vocab": V,
                   "structures_per_gpu": R, "nodes_per_gpu": n, "levels": L,
                   "parallelism": f"dp{world} (independent structures per rank)",
                   "l2": "flushed between timed steps (256 MiB write, outside the events)"},
        "latency_us": statistics.median(step_ms) * 1e3,
        "latency_p10_us": float(np.percentile(step_ms, 10)) * 1e3,
        "latency_p90_us": float(np.percentile(step_ms, 90)) * 1e3,
        "linearize_us": statistics.median(lin_ms) * 1e3,
        "forward_us": statistics.median(fwd_ms) * 1e3,
        "eager_latency_us": statistics.median(eager_ms) * 1e3,
        "two_launch_latency_us": statistics.median(two_ms) * 1e3,
        "fused": fused,
        "timing": "CUDA graph replay of cx_linearize_forward per step (one fused launch where "
                  "it applies), events on the launch stream; linearize_us / forward_us / "
                  "two_launch_latency_us time the separate cx_linearize and cx_forward launches",
        "gpu_launches": (1 if fused else 2) * args.steps,
        "allgather_roots_us": allgather_us,
        "launch": info,
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "clocks": clocks,
    }
    if secondary:
        line["throughput_b4096"] = secondary
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(name)
    print(json.dumps(line), flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=500)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--workload", default="cfg2_treelstm_b10", choices=sorted(WORKLOADS))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-secondary", dest="secondary", action="store_false",
                   help="skip the batch-4096 throughput lines (bf16, f32) of the default run")
    p.add_argument("--dtype", default="f32", choices=["f32", "bf16"],
                   help="compute precision of cx_forward (bf16 = tcgen05 tensor-core path)")
    p.add_argument("--allgather", action="store_true",
                   help="N>1: also time the NCCL all-gather of root states")
    args = p.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world == 1 and args.gpus > 1:
        print("bench.py: launch N>1 under torchrun (one process per GPU)", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
