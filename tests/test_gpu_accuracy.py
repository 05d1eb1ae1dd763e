"""Accuracy leg of the correctness contract (BASELINE north_star; SURVEY
§8c iii), mirroring the reference's decompose_error
(/root/reference/proj/src/oracle.cpp:237-260): the Monte Carlo estimate
(K3) against the deterministic GPU references (K5)

  x_exact = exp(beta A) v      (scaled Taylor, fp64)
  x_split = the splitting product the walkers sample

eps_split = the method's bias (the paper's eps_1), eps_stat = the Monte Carlo
error (eps_2).  Tolerance, stated and asserted per configuration, as mean
relative errors sum|.| / sum|x| (robust to the signed v of config 5):

  eps_total <= eps_split + 4 * mean relative SE,  and
  |sum(x_mc - x_split)| <= 4 sqrt(sum SE^2)   (unbiased in aggregate).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("idx,scale,max_rows", [(1, 1.0, 4096), (2, 0.2, 20_000),
                                                (3, 0.05, 20_000), (4, 1.0 / 64, 20_000),
                                                (5, 0.01, 20_000)])
def test_mc_within_stated_tolerance_of_exact(pb, idx, scale, max_rows):
    cfg = pb.build_config(idx, scale)
    m = pb.split(cfg.csr)
    rows = cfg.rows if cfg.rows is not None else np.arange(cfg.csr.n, dtype=np.uint32)
    if len(rows) > max_rows:
        rows = np.sort(np.random.default_rng(7).choice(rows, max_rows, replace=False)
                       ).astype(np.uint32)
    p = pb.PathParams(cfg.beta, cfg.n_steps, cfg.walkers, pb.Splitting.Strang, 5)
    mc = pb.entries_estimate(m, cfg.v, rows, p)
    x_exact = pb.expmv(m, cfg.v, cfg.beta)[rows]
    x_split = pb.splitting_product(m, cfg.v, p)[rows]
    den = np.abs(x_exact).sum()
    eps_split = np.abs(x_split - x_exact).sum() / den
    eps_total = np.abs(mc.values - x_exact).sum() / den
    se_rel = mc.std_errors.sum() / den
    z_agg = (mc.values - x_split).sum() / math.sqrt((mc.std_errors ** 2).sum())
    print(f"cfg{idx} scale {scale}: eps_split {eps_split:.3e} eps_total {eps_total:.3e} "
          f"se {se_rel:.3e} z_agg {z_agg:.2f}")
    assert eps_split < 1e-3  # the splitting error at the configs' N rule
    assert eps_total <= eps_split + 4.0 * se_rel
    assert abs(z_agg) <= 4.0
