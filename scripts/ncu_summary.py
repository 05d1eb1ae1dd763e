#!/usr/bin/env python
"""Summarise an ncu --set full report: key metrics + hottest SASS blocks.
usage: python scripts/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(raw)))
h, units, vals = rd[0], rd[1], rd[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sectors_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
out = {}
for w in want:
    if w in h:
        k = h.index(w)
        out[w] = (vals[k], units[k])
        print(f"{w:70s} {vals[k]} {units[k]}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hh = rows[1]; data = rows[2:]
ia = hh.index("Instructions Executed"); iavg = hh.index("Avg. Threads Executed")
isamp = hh.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ia] or 0) for r in data) or 1; ts = sum(float(r[isamp] or 0) for r in data) or 1
blocks = []; cur = None
for k, r in enumerate(data):
    e = float(r[ia] or 0)
    if cur and cur[1] == e:
        cur[2] += 1; cur[3] += float(r[isamp] or 0); cur[4] += float(r[iavg] or 0)
    else:
        cur = [k, e, 1, float(r[isamp] or 0), float(r[iavg] or 0)]; blocks.append(cur)
blocks.sort(key=lambda b: -b[1] * b[2])
print(f"total warp instructions {tot:.3e}")
hot = []
for b in blocks[:14]:
    line = (f"sass@{b[0]:4d} len {b[2]:3d} share {b[1]*b[2]/tot:.3f} stall {b[3]/ts:.3f} "
            f"threads {b[4]/b[2]:.1f} first: {data[b[0]][1].strip()[:48]}")
    print(line); hot.append(line)
if len(sys.argv) > 3 and sys.argv[2] == "--json":
    out["hot_blocks"] = hot
    json.dump(out, open(sys.argv[3], "w"), indent=1)
