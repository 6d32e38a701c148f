"""Stall samples per source line from an ncu report (SASS rows summed under the
source line they belong to): python tools/ncu_srcstall.py REPORT [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, cur_line, agg, text = None, None, {}, {}
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Line No", "Function Name"):
        continue
    if r[0]:
        try:
            cur_line = int(r[0])
            text[(cur_file, cur_line)] = r[1][:90]
        except ValueError:
            pass
        continue
    if len(r) > 4 and r[2].startswith("0x"):
        try:
            s = int(r[4])
        except ValueError:
            continue
        k = (cur_file, cur_line)
        agg[k] = agg.get(k, 0) + s
tot = sum(agg.values()) or 1
print(f"total samples {tot}")
for (f, l), s in sorted(agg.items(), key=lambda x: -x[1])[:N]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  {f}:{l}  {text.get((f, l), '')}")
