"""One warm-up + one timed vector_estimate / tc_estimate call on a config
(for ncu launch lists of the K4 pipeline)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_12759_b200 as pb
idx = int(sys.argv[1]); est = sys.argv[2] if len(sys.argv) > 2 else "vector"
cfg = pb.build_config(idx, 1.0)
m = pb.split(cfg.csr)
M = int(min(cfg.csr.n * cfg.walkers, 2e9))
for seed in (1, 2):
    p = pb.PathParams(cfg.beta, cfg.n_steps, M, pb.Splitting.Strang, seed)
    t = time.perf_counter()
    r = pb.vector_estimate(m, cfg.v, p) if est == "vector" else pb.tc_estimate(m, p)
    print(est, idx, seed, "%.2f ms" % (1e3 * (time.perf_counter() - t)), r.total_jumps)
