"""Summarise ncu reports into profiles/ (text + JSON):
    python tools/ncu_summary.py <launches.csv> <name=report.ncu-rep> ... --out profiles/r01"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Achieved Occupancy", "L2 Hit Rate", "One or More Eligible", "No Eligible"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_bytes.sum", "sm__inst_executed.sum", "smsp__inst_executed_op_ffma.sum"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    ki = h.index("Kernel Name")
    d, kname = {}, None
    for r in rows[1:]:
        kname = r[ki]
        if r[mi] in KEYS and r[mi] not in d:
            d[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rr[0], rr[1], rr[2]
    for k in RAW:
        if k in hdr:
            i = hdr.index(k)
            d[k] = f"{vals[i]} {units[i]}".strip()
    stalls = subprocess.run(["python", "tools/ncu_lines.py", rep, "12"], capture_output=True, text=True).stdout
    return kname, d, stalls


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [j for j, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[i + 1:]:
        v = float(r[vi].replace(",", ""))
        if r[ui] in ("nsecond", "ns"):
            v /= 1000.0
        elif r[ui] in ("msecond", "ms"):
            v *= 1000.0
        agg[r[ki].split("(")[0][:90]].append(v)
    return {k: {"count": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v)} for k, v in agg.items()}


if __name__ == "__main__":
    args = sys.argv[1:]
    out = args[args.index("--out") + 1]
    lines, js = [], {}
    L = launches(args[0])
    tot = sum(v["total_us"] for v in L.values())
    lines.append(f"# launch list ({args[0]}), ncu gpu__time_duration.sum, cold-cache serialised\n")
    for k, v in sorted(L.items(), key=lambda x: -x[1]["total_us"]):
        lines.append(f"{v['count']:5d} x {v['mean_us']:10.2f} us  share {100 * v['total_us'] / tot:5.1f}%  {k}")
    js["launches"] = L
    for spec in args[1:]:
        if "=" not in spec:
            continue
        name, rep = spec.split("=", 1)
        k, d, stalls = details(rep)
        js[name] = {"kernel": k, **d}
        lines.append(f"\n# {name}: {k}")
        lines += [f"  {a:38s} {b}" for a, b in d.items()]
        lines.append("  top source lines by warp-stall samples:")
        lines += ["    " + l for l in stalls.splitlines()]
    open(out + ".txt", "w").write("\n".join(lines) + "\n")
    json.dump(js, open(out + ".json", "w"), indent=1)
    print("\n".join(lines))
