#!/usr/bin/env python
"""Per-basic-block instruction counts of an ncu --set full report (source
page, SASS view): start line, length, executions, share, threads, stalls.
usage: python scripts/sass_blocks.py report.ncu-rep [min_share] [--dump file]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
mins = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 0.003
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
h = rows[1]; d = rows[2:]
ia = h.index("Instructions Executed"); it = h.index("Avg. Threads Executed")
isamp = h.index("Warp Stall Sampling (All Samples)")
if "--dump" in sys.argv:
    with open(sys.argv[sys.argv.index("--dump") + 1], "w") as f:
        for k, r in enumerate(d):
            f.write(f"{k:5d} {float(r[ia] or 0)/1e6:10.1f} {r[it]:>6} {r[isamp]:>7} {r[1]}\n")
out = []; prev = None
for k, r in enumerate(d):
    c = float(r[ia] or 0)
    if c != prev:
        out.append([k, 0, c, 0.0, 0, r[1].strip()]); prev = c
    b = out[-1]; b[1] += 1; b[3] += float(r[it] or 0); b[4] += int(r[isamp] or 0)
tot = sum(b[1] * b[2] for b in out) or 1
print(f"total warp instructions {tot:.4e}")
for b in out:
    if b[2] > 0 and b[1] * b[2] / tot > mins:
        print(f"{b[0]:5d} n={b[1]:3d} cnt={b[2]/1e6:8.1f}M share={b[1]*b[2]/tot:.3f} "
              f"thr={b[3]/b[1]:4.1f} stall={b[4]:7d} {b[5][:48]}")
