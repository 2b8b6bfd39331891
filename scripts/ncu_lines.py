"""Per-source-line instruction counts and stall samples from an ncu report (--set full
with -lineinfo): python scripts/ncu_lines.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")])
        stall = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    rows.append((inst, stall, fname, int(r[0]), r[1][:90]))
tot_i = sum(x[0] for x in rows) or 1
tot_s = sum(x[1] for x in rows) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
key = (lambda x: x[1]) if "--by-stall" in sys.argv else (lambda x: x[0])
for inst, stall, f, ln, src in sorted(rows, key=key, reverse=True)[:N]:
    print(f"{inst / tot_i:6.3f} {stall / tot_s:6.3f}  {f}:{ln}  {src}")
