#!/usr/bin/env python
"""Per-SASS-block instruction shares of an ncu report with source lines.
usage: python scripts/ncu_blocks.py report.ncu-rep [min_share]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; mins = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hh = rows[1]; data = rows[2:]
ia = hh.index("Instructions Executed"); iavg = hh.index("Avg. Threads Executed")
isamp = hh.index("Warp Stall Sampling (All Samples)")
isrc = hh.index("Source")
tot = sum(float(r[ia] or 0) for r in data) or 1; ts = sum(float(r[isamp] or 0) for r in data) or 1
blocks = []; cur = None
for k, r in enumerate(data):
    e = float(r[ia] or 0)
    if cur and cur[1] == e:
        cur[2] += 1; cur[3] += float(r[isamp] or 0); cur[4] += float(r[iavg] or 0)
    else:
        cur = [k, e, 1, float(r[isamp] or 0), float(r[iavg] or 0)]; blocks.append(cur)
print(f"total warp instructions {tot:.4e}; static instructions {len(data)}")
acc = 0
for b in blocks:
    sh = b[1] * b[2] / tot
    acc += sh
    if sh >= mins:
        print(f"sass@{b[0]:5d} len {b[2]:4d} exec {b[1]:.3e} share {sh:.3f} cum {acc:.3f} stall {b[3]/ts:.3f} thr {b[4]/b[2]:5.1f} | {data[b[0]][isrc].strip()[:60]}")
