#!/usr/bin/env python
"""Summarise ncu captures (run here, no GPU) into profiles/ text files.

    python scripts/ncu_summary.py REPORT.ncu-rep [--out profiles/NAME.txt] [--algo-bytes N]
    python scripts/ncu_summary.py --launches LAUNCHES.csv [--out ...]
"""
import argparse
import csv
import io
import json
import subprocess
import sys
from collections import Counter, defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second", "sm__inst_executed.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    kernels = []
    for v in r[2:]:
        kernels.append({h[i]: (v[i], u[i]) for i in range(len(h))})
    return kernels


def sass_mix(rep):
    """Per kernel: executed-instruction mix and stall samples from the SASS source page."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res, cur, h = [], None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1] if len(r) > 1 else "?", "ops": Counter(), "stalls": Counter()}
            res.append(cur)
            h = None
            continue
        if cur is None:
            continue
        if h is None:
            h = r
            idx = {n: i for i, n in enumerate(h)}
            continue
        if len(r) < 5 or r[0] == "Address":
            continue
        t = r[idx["Source"]].strip().split()
        if not t:
            continue
        o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        cur["ops"][o] += int(r[idx["Instructions Executed"]] or 0)
        for k in h:
            if k.startswith("stall_") and "Not Issued" not in k:
                cur["stalls"][k] += int(r[idx[k]] or 0)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--out")
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--elements", type=float, default=None)
    a = ap.parse_args()
    lines = []
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        h = rows[hi]
        idx = {n: j for j, n in enumerate(h)}
        agg = defaultdict(list)
        for r in rows[hi + 1:]:
            if len(r) >= len(h) and r[idx["Metric Name"]] == "gpu__time_duration.sum":
                agg[r[idx["Kernel Name"]]].append(float(r[idx["Metric Value"]].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        lines.append(f"# launch list (ncu gpu__time_duration.sum, cold-cache serialised): {a.launches}")
        lines.append(f"{'kernel':70s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"{k[:70]:70s} {len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / tot:7.3f}")
    if a.report:
        for kern in raw(a.report):
            name = kern.get("Kernel Name", ("?", ""))[0]
            lines.append(f"# ncu --set full: {a.report}\n# kernel: {name}")
            for m in METRICS:
                if m in kern:
                    lines.append(f"{m:60s} {kern[m][0]:>16s} {kern[m][1]}")
            try:
                rd = float(kern["dram__bytes_read.sum"][0].replace(",", ""))
                unit = kern["dram__bytes_read.sum"][1]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                wr = float(kern["dram__bytes_write.sum"][0].replace(",", ""))
                wunit = kern["dram__bytes_write.sum"][1]
                wscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(wunit, 1)
                traffic = rd * scale + wr * wscale
                lines.append(f"{'traffic = dram read + write (bytes)':60s} {traffic:16.0f}")
                if a.algo_bytes:
                    lines.append(f"{'algorithmic bytes per launch':60s} {a.algo_bytes:16.0f}")
                    lines.append(f"{'traffic / algorithmic':60s} {traffic / a.algo_bytes:16.4f}")
                if a.out and "rows" in name:  # the dominant kernel's traffic, read by bench.py
                    js = a.out.rsplit(".", 1)[0] + ".json"
                    json.dump({"kernel": name, "dram_bytes_per_launch": traffic,
                               "algorithmic_bytes": a.algo_bytes}, open(js, "w"), indent=1)
            except Exception:
                pass
        for k in sass_mix(a.report):
            ops, stalls = k["ops"], k["stalls"]
            tot = sum(ops.values())
            lines.append(f"# SASS mix of {k['name'][:80]}: executed warp instructions {tot}")
            if a.elements and "rows" in k["name"]:
                lines.append(f"# thread instructions per element: {tot * 32 / a.elements:.2f}")
            for o, n in ops.most_common(14):
                lines.append(f"  {o:10s} {n:14d} {n / max(tot, 1):6.3f}")
            st = sum(stalls.values())
            lines.append("# warp stall samples")
            for o, n in stalls.most_common(8):
                lines.append(f"  {o:28s} {n:10d} {n / max(st, 1):6.3f}")
    txt = "\n".join(lines) + "\n"
    if a.out:
        open(a.out, "w").write(txt)
    sys.stdout.write(txt)


if __name__ == "__main__":
    main()
