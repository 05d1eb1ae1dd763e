"""Workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): K1 split_pack (+ alias tables on a weighted graph), K3 entry
walker, K2 PCG-compat walker, K4 vector / tc walkers, K3L (W >= 2^29 path
through a tiny graph).  Sized so racecheck (which instruments every shared
access) finishes in minutes.

  python scripts/sanitize_cases.py {cfg1|cfg2|weighted} [--rows R] [--walkers W]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_12759_b200 as pb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--walkers", type=int, default=2000)
    ap.add_argument("--vector-samples", type=int, default=2_000_000)
    a = ap.parse_args()
    if a.case == "cfg1":
        cfg = pb.build_config(1)
        csr, v, beta, N = cfg.csr, cfg.v, cfg.beta, cfg.n_steps
    elif a.case == "cfg2":
        cfg = pb.build_config(2, 0.05)
        csr, v, beta, N = cfg.csr, cfg.v, cfg.beta, cfg.n_steps
    elif a.case == "weighted":
        # FD2D 24x24 with order-sensitive U(0,1] weights (symmetric): every
        # row non-uniform -> alias tables in K1, alias jumps in K3/K4
        csr = pb.gen_fd(2, 24, 1.0)
        rng = np.random.default_rng(5)
        w = {}
        for i in range(csr.n):
            for k in range(int(csr.row_ptr[i]), int(csr.row_ptr[i + 1])):
                j = int(csr.col[k])
                key = (min(i, j), max(i, j))
                if key not in w:
                    w[key] = rng.uniform(1e-3, 1.0)
                csr.val[k] = w[key]
        v = pb.gen_vector(0, csr.n, 2)
        beta, N = 1.0, 32
    else:
        raise SystemExit("unknown case")
    m = pb.split(csr, device=0)
    rows = np.linspace(0, csr.n - 1, min(a.rows, csr.n)).astype(np.uint32)
    r3 = pb.entries_estimate(m, v, rows, pb.PathParams(beta, N, a.walkers, pb.Splitting.Strang, 3))
    r3l = pb.entries_estimate(m, v, rows[:2],
                              pb.PathParams(beta, N, a.walkers, pb.Splitting.Lie, 4))
    p2 = pb.PathParams(beta, N, min(a.walkers, 500), pb.Splitting.Strang, 3, pb.Rng.PCG_COMPAT)
    r2 = pb.entries_estimate(m, v, rows[:32], p2)
    pv = pb.PathParams(beta, N, a.vector_samples, pb.Splitting.Strang, 5)
    ve = pb.vector_estimate(m, np.abs(v), pv)
    tc = pb.tc_estimate(m, pv)
    print(f"{a.case}: K3 jumps {int(r3.jumps.sum())} K3(lie) {int(r3l.jumps.sum())} "
          f"K2 jumps {int(r2.jumps.sum())} vector jumps {ve.total_jumps} tc {tc.value:.6g}",
          flush=True)


if __name__ == "__main__":
    main()
