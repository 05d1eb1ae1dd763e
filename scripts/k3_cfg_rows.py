"""K3 on the first R sampled rows of a config (ncu captures of long-walk
configs without profiling a multi-second launch).
usage: python scripts/k3_cfg_rows.py CFG R"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1904_12759_b200 as pb

idx, R = int(sys.argv[1]), int(sys.argv[2])
cfg = pb.build_config(idx, 1.0)
m = pb.split(cfg.csr)
pool = cfg.rows if cfg.rows is not None else np.arange(cfg.csr.n)
rows = np.ascontiguousarray(pool[:R], np.uint32)
p = pb.PathParams(cfg.beta, cfg.n_steps, cfg.walkers, pb.Splitting.Strang, 3)
for k in range(3):
    t = time.perf_counter()
    r = pb.entries_estimate(m, cfg.v, rows, p)
    print(f"cfg{idx} rows {R}: {1e3 * (time.perf_counter() - t):.1f} ms, jumps {r.total_jumps}")
