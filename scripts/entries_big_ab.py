"""Entry estimator on config 5 through the host API: K3 (default) or the
grouped-start walk K3L (EXPMC_FORCE_BIG=1, experiments only).  Wall time
per call, jumps/s."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_12759_b200 as pb
cfg = pb.build_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5, 1.0)
m = pb.split(cfg.csr)
p = pb.PathParams(cfg.beta, cfg.n_steps, cfg.walkers, pb.Splitting.Strang, 3)
tag = "K3L" if os.environ.get("EXPMC_FORCE_BIG") else "K3"
for k in range(4):
    t = time.perf_counter()
    r = pb.entries_estimate(m, cfg.v, cfg.rows, p)
    dt = time.perf_counter() - t
    print(f"{tag} cfg{cfg.index if hasattr(cfg, 'index') else ''} {1e3 * dt:.1f} ms "
          f"jumps {r.total_jumps:.4g} {r.total_jumps / dt:.4g} jumps/s")
