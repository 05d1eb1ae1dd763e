#!/usr/bin/env python
"""Markdown table of the round's bench lines (profiles/r02/bench_cfg<i>.json).
usage: python scripts/readme_table.py profiles/r02"""
import json
import os
import sys

d0 = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02"
names = {1: "FD2D 64², 4096 × 1e4 walkers", 2: "BA 1e5, 1e5 × 1e4", 3: "WS 1e6, 1e6 × 2e3",
         4: "FD3D 256³, 1e6 rows × 1e4", 5: "BA 1e7 m=8, 1e7 × 1e3, N=512"}
print("| cfg | workload | kernel ms | transitions/s | e2e transitions/s | roofline (bound: frac) | K3 / K6 | CPU reference (as-is / path-only) | e2e / CPU as-is | e2e / CPU path-only |")
print("|---|---|---|---|---|---|---|---|---|---|")
for c in (1, 2, 3, 4, 5):
    d = json.loads(open(os.path.join(d0, f"bench_cfg{c}.json")).read().strip().splitlines()[-1])
    r, e, cb, g = d["roofline"], d["e2e"], d["cpu_baseline"], d.get("gather_ceiling") or {}
    po = cb.get("path_only_value")
    bold = "**" if c == 5 else ""
    print(f"| {c} | {names[c]} | {bold}{r['kernel_ms']:.4g}{bold} | {bold}{d['value']:.3g}{bold} | "
          f"{bold}{e['value']:.3g}{bold} | {r['bound']}: {r['frac']:.2f} | {g.get('frac_of_ceiling', float('nan')):.2f} | "
          f"{cb['value']:.3g} / {po:.3g} | {e['value'] / cb['value']:.3g}× | {e['value'] / po:.3g}× |")
