#!/usr/bin/env python
"""Accuracy leg for the Theorem-2 estimators (SURVEY §8c iii, rows a13/a14) at
full configuration size: K4 vector_estimate / tc_estimate against the
deterministic splitting product they sample (K5, fp64):

  E[values] = x_split = (e^{dtD/2} e^{-dtL} e^{dtD/2})^N v        (vector)
  E[tc]     = 1^T (e^{dtD/2} e^{-dtL} e^{dtD/2})^N 1               (tc)

Reported per config (v >= 0 configs 1-4, M = n W capped at --max-paths):
  * z_global: (sum(values) - sum(x_split)) / std_error_global — the
    reference's own global SE (estimator.cpp:268-272); |z| <= 4 expected;
  * eps_a, eps_b: sum|values - x_split| / sum|x_split| for two independent
    seeds, and eps_pair = sum|a - b| / sum|x_split| / sqrt(2): for an unbiased
    per-entry law eps_a ~ eps_b ~ eps_pair (independent noise adds in
    quadrature); a per-entry bias would push eps_a, eps_b above eps_pair;
  * z_tc: (tc - 1^T x_split(1)) / SE.
One JSON line per config.

usage: python scripts/accuracy_vector.py [--configs 1 2 3 4] [--max-paths 2e9]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1904_12759_b200 as pb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4])
    ap.add_argument("--max-paths", type=float, default=2e9)
    args = ap.parse_args()
    for c in args.configs:
        t0 = time.time()
        cfg = pb.build_config(c, 1.0)
        m = pb.split(cfg.csr)
        n = cfg.csr.n
        M = int(min(n * cfg.walkers, args.max_paths))
        pa = pb.PathParams(cfg.beta, cfg.n_steps, M, pb.Splitting.Strang, 11)
        pbb = pb.PathParams(cfg.beta, cfg.n_steps, M, pb.Splitting.Strang, 12)
        a = pb.vector_estimate(m, cfg.v, pa)
        fixed = pb.last_k4_stats(m)[1]
        b = pb.vector_estimate(m, cfg.v, pbb)
        x = pb.splitting_product(m, cfg.v, pa)
        den = np.abs(x).sum()
        eps_a = float(np.abs(a.values - x).sum() / den)
        eps_b = float(np.abs(b.values - x).sum() / den)
        eps_pair = float(np.abs(a.values - b.values).sum() / den / math.sqrt(2.0))
        z_global = float((a.values.sum() - x.sum()) / a.std_error_global)
        t = pb.tc_estimate(m, pa)
        x1 = pb.splitting_product(m, np.ones(n), pa)
        z_tc = float((t.value - x1.sum()) / t.std_error)
        out = {"config": f"cfg{c}_{cfg.name}", "n": n, "paths": M, "n_steps": cfg.n_steps,
               "beta": cfg.beta, "fixed_point_sums": bool(fixed == 1),
               "z_global": z_global, "eps_a": eps_a, "eps_b": eps_b, "eps_pair": eps_pair,
               "eps_ratio": max(eps_a, eps_b) / eps_pair if eps_pair > 0 else None,
               "tc": t.value, "tc_exact": float(x1.sum()), "z_tc": z_tc,
               "ok": bool(abs(z_global) <= 4 and abs(z_tc) <= 4 and
                          max(eps_a, eps_b) <= 1.1 * eps_pair + 1e-12),
               "secs": round(time.time() - t0, 1)}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
