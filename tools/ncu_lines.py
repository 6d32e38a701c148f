"""Aggregate ncu source-page warp-stall samples per CUDA source line.
    python tools/ncu_lines.py report.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, agg, hdr = None, {}, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        s, ie = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    stalls = {hdr[i]: int(r[i] or 0) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and r[i].isdigit()}
    agg[(cur, int(r[0]))] = (s, ie, r[1].strip(), stalls)
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    st = sorted(v[3].items(), key=lambda x: -x[1])[:2]
    st = " ".join(f"{a[6:]}={b}" for a, b in st if b)
    print(f"{v[0]:6d} {v[1]:9d} {k[0]}:{k[1]:4d} {v[2][:70]:70s} {st}")
