#!/usr/bin/env python
"""Per-source-line instruction and stall-sample totals from an ncu report (profiling tooling).

    python scripts/ncu_lines.py REPORT.ncu-rep [min_pct]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
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
    if hdr and r[0] and r[0] != "":
        try:
            ln = int(r[0])
        except ValueError:
            continue
        d = dict(zip(hdr[4:], r[-(len(hdr) - 4):]))  # numeric columns, aligned from the right
        num = lambda k: float(d.get(k, "0")) if d.get(k, "-") not in ("", "-") else 0.0
        ie = num("Instructions Executed")
        sm = num("Warp Stall Sampling (All Samples)")
        rows.append((fname, ln, r[1].strip()[:90], ie, sm))
ti = sum(x[3] for x in rows) or 1
ts = sum(x[4] for x in rows) or 1
print(f"total warp instructions {ti:.4g}, samples {ts:.4g}")
for f, ln, s, ie, sm in rows:
    if 100 * ie / ti >= minp or 100 * sm / ts >= minp:
        print(f"{f}:{ln:<4d} inst {100*ie/ti:5.1f}%  stall {100*sm/ts:5.1f}%  {s}")
