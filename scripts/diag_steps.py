#!/usr/bin/env python
"""Diagnose time between walker launches in the bench loop: host enqueue
cost of entries_device vs GPU-side gaps (CUDA events)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_12759_b200 as pb  # noqa: E402

cfg = pb.build_config(int(sys.argv[1]) if len(sys.argv) > 1 else 1,
                      float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
m = pb.split(cfg.csr)
rows = np.arange(cfg.csr.n, dtype=np.uint32) if cfg.rows is None else cfg.rows
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream()
sp = s.cuda_stream
v = torch.from_numpy(cfg.v).to(dev)
rd = torch.from_numpy(rows.astype(np.int32)).to(dev)
val = torch.empty(len(rows), dtype=torch.float64, device=dev)
se = torch.empty_like(val)
jm = torch.empty(len(rows), dtype=torch.int64, device=dev)
pb.set_v_device(m, v.data_ptr(), cfg.csr.n, sp)
p = pb.PathParams(cfg.beta, cfg.n_steps, cfg.walkers, pb.Splitting.Strang, 3)
for _ in range(3):
    pb.entries_device(m, rd.data_ptr(), len(rows), p, val.data_ptr(), se.data_ptr(),
                      jm.data_ptr(), sp)
torch.cuda.synchronize()
K = 10
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
      for _ in range(K)]
host = []
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record(s)
for k in range(K):
    ev[k][0].record(s)
    a = time.perf_counter()
    pb.entries_device(m, rd.data_ptr(), len(rows), p, val.data_ptr(), se.data_ptr(),
                      jm.data_ptr(), sp)
    host.append(time.perf_counter() - a)
    ev[k][1].record(s)
t1.record(s)
torch.cuda.synchronize()
kern = [a.elapsed_time(b) for a, b in ev]
gaps = [ev[k][0].elapsed_time(ev[k + 1][0]) - kern[k] for k in range(K - 1)]
print(f"config {cfg.name}: total {t0.elapsed_time(t1) / K:.3f} ms/step, kernel "
      f"{np.mean(kern):.3f} ms, gap {np.mean(gaps):.3f} ms, host enqueue "
      f"{1e3 * np.mean(host):.3f} ms (max {1e3 * np.max(host):.3f})")
