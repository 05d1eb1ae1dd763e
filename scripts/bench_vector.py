#!/usr/bin/env python
"""Theorem-2 estimators (SURVEY §8a rows a13 vector_estimate, a14
tc_estimate) on the BASELINE configurations with v >= 0 (1-4): the GPU
Philox walker K4 through the host API (H2D of v, D2H of the n-vector inside
the timed region) beside the unmodified reference (oracle/_ref) with
workers = all host cores on a bounded M.  One JSON line per (estimator,
config) on stdout.

M follows SURVEY §8d (M = n * W) capped at --max-paths so one call stays in
seconds; the CPU sample is sized to ~--cpu-seconds.  Metric: path
transitions/s (total jumps / s) and paths/s.

usage: python scripts/bench_vector.py [--configs 1 2 3 4] [--steps 3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_GBps", "copy_gbs"):
            if k in d:
                return float(d[k])
    except (OSError, ValueError):
        pass
    return 7700.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--max-paths", type=float, default=2e9)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    import paper_1904_12759_b200 as pb

    cores = os.cpu_count() or 1
    for idx in args.configs:
        cfg = pb.build_config(idx, 1.0)  # config 2: beta = 0.5 / lambda_max (GPU stats)
        m = pb.split(cfg.csr)
        n = cfg.csr.n
        M = int(min(n * cfg.walkers, args.max_paths))
        for est in ("vector", "tc"):
            def run(seed, samples=M):
                p = pb.PathParams(cfg.beta, cfg.n_steps, samples, pb.Splitting.Strang, seed)
                if est == "vector":
                    r = pb.vector_estimate(m, cfg.v, p)
                else:
                    r = pb.tc_estimate(m, p)
                return r.total_jumps
            run(1)  # warm-up (module load, scratch allocation)
            t = time.perf_counter()
            jumps = sum(run(2 + k) for k in range(args.steps))
            secs = time.perf_counter() - t
            line = {"estimator": f"{est}_estimate", "config": f"cfg{idx}_{cfg.name}", "n": n,
                    "paths_per_call": M, "n_steps": cfg.n_steps, "beta": cfg.beta,
                    "gpu": {"transitions_per_s": jumps / secs,
                            "paths_per_s": M * args.steps / secs,
                            "ms_per_call": 1e3 * secs / args.steps,
                            "api": f"expmc_cuda_{est}_estimate (host buffers, wall clock, "
                                   "H2D/D2H included)"}}
            if not args.no_cpu:
                import oracle

                rm = oracle.Ref().matrix_from_csr(cfg.csr)
                # calibrate, then one bounded sample of ~cpu_seconds
                Mc = max(cores * 100, 10_000)
                t = time.perf_counter()
                if est == "vector":
                    rm.vector_estimate(cfg.v, cfg.beta, cfg.n_steps, Mc, 1, 7, workers=cores)
                else:
                    rm.tc_estimate(cfg.beta, cfg.n_steps, Mc, 1, 7, workers=cores)
                tc = max(time.perf_counter() - t, 1e-3)
                Mc = int(Mc * max(1.0, args.cpu_seconds / tc))
                t = time.perf_counter()
                if est == "vector":
                    _, _, j, _ = rm.vector_estimate(cfg.v, cfg.beta, cfg.n_steps, Mc, 1, 8,
                                                    workers=cores)
                else:
                    _, _, j = rm.tc_estimate(cfg.beta, cfg.n_steps, Mc, 1, 8, workers=cores)
                secs_c = time.perf_counter() - t
                line["cpu_reference"] = {"transitions_per_s": j / secs_c,
                                         "paths_per_s": Mc / secs_c, "cores": cores,
                                         "kind": "reference",
                                         "sample": f"M = {Mc} paths, workers = {cores}, "
                                                   f"{secs_c:.1f} s"}
                line["speedup_transitions"] = line["gpu"]["transitions_per_s"] / \
                    line["cpu_reference"]["transitions_per_s"]
            # roofline of the whole call (SURVEY §8d bytes, K4 form): 64 B per
            # jump + 48 B per jumper (start record + 16-B result record)
            jumpers = pb.last_jumpers(m)
            b_alg = 64.0 * jumps / args.steps + 48.0 * jumpers
            peak = _hbm_peak()
            ach = b_alg / (secs / args.steps) / 1e9
            line["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                                "frac": ach / peak, "traffic": None,
                                "algorithmic_bytes_per_call": b_alg,
                                "jumpers_per_call": jumpers,
                                "scope": "whole host call (wall clock)"}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
