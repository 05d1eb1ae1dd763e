#!/usr/bin/env python
"""Condense one ncu --set full report of the walker kernel into the JSON
bench.py's roofline reads (profiles/r02/ncu_cfg<i>.json): DRAM bytes and
l1tex global-load sectors per launch, hit rates, issue activity, and the
hash of the kernel sources the capture was taken at.
usage: python scripts/ncu_to_profile.py report.ncu-rep CFG out.json [capture-note]"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (source_sha)

rep, cfg, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
note = sys.argv[4] if len(sys.argv) > 4 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(raw)))
h, vals = rd[0], rd[2]


def g(name):
    return float(vals[h.index(name)].replace(",", ""))


def unit(name):
    return rd[1][h.index(name)]


def to_bytes(name):
    u = unit(name).lower()
    f = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}[u]
    return g(name) * f


def to_ms(name):
    u = unit(name).lower()
    f = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "second": 1e3}[u]
    return g(name) * f


d = {
    "config": cfg,
    "kernel": vals[h.index("Kernel Name")],
    "capture": note or os.path.basename(rep),
    "source_sha": bench.source_sha(),
    "kernel_ms_under_ncu": to_ms("gpu__time_duration.sum"),
    "dram_bytes_per_launch": to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum"),
    "l1tex_ld_sectors_per_launch": g("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    "l1tex_ld_requests_per_launch": g("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    "l2_hit_rate": g("lts__t_sector_hit_rate.pct"),
    "l1_hit_rate": g("l1tex__t_sector_hit_rate.pct"),
    "issue_active": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "warp_instructions": g("smsp__inst_executed.sum"),
    "registers": g("launch__registers_per_thread"),
    "lts_tex_read_sectors": g("lts__t_sectors_srcunit_tex_op_read.sum"),
}
with open(out, "w") as f:
    json.dump(d, f, indent=1)
print(json.dumps(d, indent=1))
