"""K4 tc_estimate on config 5 with M = n W (the entries workload's walker
count): jumps/s of the grouped-start walker on the BA 1e7 graph."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_12759_b200 as pb
cfg = pb.build_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5, 1.0)
m = pb.split(cfg.csr)
M = cfg.csr.n * cfg.walkers
for seed in (1, 2, 3):
    p = pb.PathParams(cfg.beta, cfg.n_steps, M, pb.Splitting.Strang, seed)
    t = time.perf_counter()
    r = pb.tc_estimate(m, p)
    dt = time.perf_counter() - t
    print(f"tc cfg M={M:.3g} {1e3*dt:.1f} ms jumps={r.total_jumps:.4g} {r.total_jumps/dt:.3g} jumps/s jumpers={pb.last_jumpers(m):.4g}", flush=True)
