import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1904_12759_b200 as pb
# long walks with few walkers per entry: task slots recycle through the gate
csr = pb.gen_fd(3, 64, 4225.0)   # 64^3 grid, rate ~ 6*4225
v = pb.gen_vector(0, csr.n, 2)
m = pb.split(csr)
rows = np.arange(0, csr.n, 2, dtype=np.uint32)
for W in (16, 64, 1000):
    p = pb.PathParams(1e-3, 32, W, pb.Splitting.Strang, 3)
    pb.entries_estimate(m, v, rows, p)
    t = time.perf_counter(); r = pb.entries_estimate(m, v, rows, p); dt = time.perf_counter() - t
    print(f"W={W}: {1e3*dt:.1f} ms, jumps {r.total_jumps}, {r.total_jumps/dt:.3e} jumps/s")
