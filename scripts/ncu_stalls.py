#!/usr/bin/env python
"""Top instructions by a stall reason in an ncu report.
usage: python scripts/ncu_stalls.py report.ncu-rep [stall_long_sb] [N]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; col = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"; N = int(sys.argv[3]) if len(sys.argv) > 3 else 14
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out))); hh = rows[1]; data = rows[2:]
ic = hh.index(col); isrc = hh.index("Source"); ia = hh.index("Instructions Executed"); isamp = hh.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ic] or 0) for r in data); ts = sum(float(r[isamp] or 0) for r in data)
print(f"{col}: {tot:.0f} samples of {ts:.0f} ({tot/ts:.3f})")
for k in sorted(range(len(data)), key=lambda k: -float(data[k][ic] or 0))[:N]:
    r = data[k]
    print(f"{k:5d} {float(r[ic] or 0)/ts:.4f} exec {r[ia]:>10s} | {r[isrc].strip()[:70]}  <- prev: {data[k-1][isrc].strip()[:40]}")
