"""Law of the walkers' Exp(1) draws (the reference's exp_time,
/root/reference/proj/src/sampler.cpp:10-16, draws -log(u) from a 53-bit
uniform in fp64; the B200 walkers use neg_ln_u, csrc/common.cuh: fp32 from
the 31-bit midpoint uniform u = (w | 1) 2^-32 of one Philox word).

Over 2^30 draws on the GPU:
  * Kolmogorov-Smirnov on the bin edges of a 0.05-wide histogram: the
    largest CDF gap is within the KS 99.9% band 1.95/sqrt(n);
  * tail masses P(E > y) for y = 4, 8, 12, 16, 17, 20 within 4 binomial SE
    of e^-y (the round-1 transform, a 23-bit uniform, had no mass above
    16.6: P(E > 17) = 4.1e-8 would read 0 instead of ~44 draws here);
  * mean 1 and variance 1 within 4 SE.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_exp1_transform_law(pb):
    n = 1 << 30
    width, nb = 0.05, 512  # bins up to 25.6 (the transform's max is 22.18)
    hist, mom = pb.exp_law(n, seed=12345, bin_width=width, nbins=nb)
    assert int(hist.sum()) == n
    edges = width * np.arange(1, nb)
    cdf_emp = np.cumsum(hist[:-1]) / n
    D = float(np.max(np.abs(cdf_emp - (1.0 - np.exp(-edges)))))
    assert D < 1.95 / math.sqrt(n), D
    for y in (4, 8, 12, 16, 17, 20):
        k = int(round(y / width))
        tail = int(hist[k:].sum())
        p = math.exp(-y)
        se = math.sqrt(n * p * (1 - p))
        assert abs(tail - n * p) <= 4 * se + 1, (y, tail, n * p)
    assert int(hist[int(round(22.2 / width)):].sum()) == 0  # max 32 ln 2 = 22.18
    mean = mom[0] / n
    var = mom[1] / n - mean * mean
    assert abs(mean - 1.0) < 4 * math.sqrt(1.0 / n) + 1e-7
    assert abs(var - 1.0) < 4 * math.sqrt(8.0 / n) + 1e-6
