#!/usr/bin/env python
"""Measured L2 random-gather ceiling: K6 (walk_fast.cu, memory-only walker,
hash RNG) in long chains over the config-2 BA graph, whose 32-MB fat Edge
table is L2-resident.  Written to profiles/r02/l2_gather_peak.json and used
by bench.py as the roofline peak of the cache-resident configs (1-4).
usage (GPU box): python scripts/l2_gather_peak.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_12759_b200 as pb

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/l2_gather_peak.json"
cfg = pb.build_config(2, 1.0)
m = pb.split(cfg.csr)
pb.set_v_device  # noqa: B018 (API presence)
rows = torch.arange(cfg.csr.n, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
best = None
for chains, length in ((256, 64), (512, 64), (1024, 32), (2048, 16)):
    for _ in range(2):
        pb.gather_ceiling_device(m, rows.data_ptr(), cfg.csr.n, chains, length, st.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record(st)
    for _ in range(reps):
        pb.gather_ceiling_device(m, rows.data_ptr(), cfg.csr.n, chains, length, st.cuda_stream)
    b.record(st)
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / reps / 1e3
    jumps = cfg.csr.n * chains * length
    r = {"chains_per_row": chains, "chain_len": length, "ms": t * 1e3, "jumps_per_s": jumps / t,
         "gbs_sector_32B": 32.0 * jumps / t / 1e9, "gbs_model_64B": 64.0 * jumps / t / 1e9}
    print(r)
    if best is None or r["jumps_per_s"] > best["jumps_per_s"]:
        best = r
best["how"] = ("K6 gather_ceiling_kernel, chains of dependent 32-B Edge gathers over the "
               "config-2 BA graph (n=1e5, 32-MB Edge table, L2-resident), best of 4 shapes, "
               "CUDA events, 5 launches")
best["table_bytes"] = int(cfg.csr.nnz) * 32
best["gpu"] = torch.cuda.get_device_name(0)
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump(best, f, indent=1)
print("wrote", out)
