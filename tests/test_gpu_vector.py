"""K4 (vector_estimate / tc_estimate by grouped starts, csrc/walk_vec.cu) on the GPU.

K4 draws the reference's M i.i.d. walkers (estimator.cpp:208-318) grouped by
start row: multinomial start counts down a binomial tree, a binomial split of
each row's walkers into never-jumpers and jumpers, walks for the jumpers only.
These tests pin the two samplers that replace the per-walker start draw
against their exact laws, then the estimators against the reference.

Tolerances (written here, per the contract):
  * Binomial sampler: chi-square goodness of fit against scipy.stats.binom,
    p-value > 1e-4 per case (cells with expected count >= 20), and the sample
    mean within 5 standard errors of n p.
  * Start counts: sum exactly M; chi-square of the counts against M v / V
    (one multinomial draw: n - 1 degrees of freedom), p-value > 1e-4.
  * Estimates: global functional within 4 combined SE of the reference's own
    vector_estimate / tc_estimate; per entry, against the splitting product x
    the walkers sample (K5): the mean of R = 8 GPU runs within 1.5 / sqrt(R)
    of a single run's L1 distance (no per-entry bias), and the reference's
    L1 distance within a factor 1.6 of a GPU run's; total jumps within 1%.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

stats = pytest.importorskip("scipy.stats")


def _chi2_binom(x, n, p):
    dist = stats.binom(n, p)
    lo, hi = int(x.min()), int(x.max())
    ks = np.arange(lo, hi + 1)
    pmf = dist.pmf(ks)
    # merge tails into the edge cells, then merge cells until expected >= 20
    pmf[0] += dist.cdf(lo - 1)
    pmf[-1] += dist.sf(hi)
    obs = np.bincount((x - lo).astype(np.int64), minlength=len(ks)).astype(float)
    exp = pmf * len(x)
    cells_o, cells_e, ao, ae = [], [], 0.0, 0.0
    for o, e in zip(obs, exp):
        ao += o
        ae += e
        if ae >= 20:
            cells_o.append(ao)
            cells_e.append(ae)
            ao = ae = 0.0
    if ae > 0 and cells_e:
        cells_o[-1] += ao
        cells_e[-1] += ae
    cells_o, cells_e = np.array(cells_o), np.array(cells_e)
    cells_e *= cells_o.sum() / cells_e.sum()
    if len(cells_o) < 2:
        return 1.0
    return stats.chisquare(cells_o, cells_e).pvalue


@pytest.mark.parametrize("n,p", [
    (1, 0.3), (7, 0.5), (40, 0.1), (1000, 0.005),      # inversion (n p < 10)
    (30, 0.4), (1000, 0.02), (10_000, 0.5),            # BTRS
    (123_456_789, 1e-7), (2_000_000_000, 0.3),         # BTRS, large n
    (500, 0.97), (10_000_000_000, 0.999999),           # p > 1/2 (symmetry)
])
def test_binomial_sampler_law(pb, n, p):
    x = pb.binomial_samples(n, p, 400_000, seed=11).astype(np.float64)
    assert x.min() >= 0 and x.max() <= n
    mean, var = n * p, n * p * (1 - p)
    assert abs(x.mean() - mean) <= 5 * math.sqrt(var / len(x)) + 1e-12
    if var > 0:
        assert abs(x.var() / var - 1) < 0.02
    if var < 1e7:  # pmf cells resolvable
        assert _chi2_binom(x, n, p) > 1e-4


def test_binomial_sampler_edges(pb):
    assert np.all(pb.binomial_samples(0, 0.5, 100) == 0)
    assert np.all(pb.binomial_samples(50, 0.0, 100) == 0)
    assert np.all(pb.binomial_samples(50, 1.0, 100) == 50)
    a = pb.binomial_samples(1000, 0.3, 1000, seed=3)
    b = pb.binomial_samples(1000, 0.3, 1000, seed=3)
    c = pb.binomial_samples(1000, 0.3, 1000, seed=4)
    assert np.array_equal(a, b) and not np.array_equal(a, c)


@pytest.mark.parametrize("n", [1, 2, 3, 37, 1000, 4097])
def test_start_counts_multinomial(pb, n):
    rng = np.random.default_rng(n)
    csr = pb.gen_ws(max(n, 12), 2, 0.1, 3) if n >= 12 else pb.csr_from_dense(
        np.ones((n, n)) - np.eye(n) if n > 1 else np.zeros((1, 1)))
    m = pb.split(csr)
    nn = m.n
    M = 10_000_000
    for v in (None, rng.uniform(0, 1, nn) * (rng.uniform(size=nn) > 0.2)):
        if v is not None and v.sum() == 0:
            v[0] = 1.0
        c = pb.start_counts(m, v, M, seed=5)
        assert c.sum() == M
        w = np.ones(nn) if v is None else v
        if v is not None:
            assert np.all(c[w == 0] == 0)
        e = M * w / w.sum()
        keep = e > 0
        if keep.sum() > 1:
            assert stats.chisquare(c[keep], e[keep]).pvalue > 1e-4
        c2 = pb.start_counts(m, v, M, seed=5)
        assert np.array_equal(c, c2)


def test_start_counts_many_seeds_mean(pb):
    """Across seeds, each row's count averages M p_i (unbiased tree)."""
    csr = pb.gen_ws(300, 2, 0.1, 1)
    m = pb.split(csr)
    v = np.linspace(0.1, 3.0, m.n)
    M = 100_000
    acc = np.zeros(m.n)
    S = 200
    for s in range(S):
        acc += pb.start_counts(m, v, M, seed=100 + s)
    p = v / v.sum()
    z = (acc / S - M * p) / np.sqrt(M * p * (1 - p) / S)
    assert abs(z.mean()) < 4 / math.sqrt(m.n) * 2 and 0.7 < z.var() < 1.3


@pytest.mark.parametrize("splitting", [0, 1])
@pytest.mark.parametrize("name", ["ba_2000", "weighted_40", "ws_3000"])
def test_vector_and_tc_vs_reference(pb, ref, name, splitting):
    from test_gpu_parity import _graphs

    csr = _graphs(pb)[name]
    rm = ref.matrix_from_csr(csr)
    m = pb.split(csr)
    rng = np.random.default_rng(7)
    v = rng.uniform(0, 1, csr.n)
    v[rng.uniform(size=csr.n) < 0.1] = 0.0
    beta = {"ba_2000": 0.05, "weighted_40": 0.7, "ws_3000": 0.3}[name]
    M = 4_000_000
    p = pb.PathParams(beta, 32, M, pb.Splitting(splitting), 9)
    got = pb.vector_estimate(m, v, p)
    rv, rse, rj, rvs = rm.vector_estimate(v, beta, 32, M, splitting, 10, workers=16)
    z = (got.values.sum() - rv.sum()) / math.sqrt(got.std_error_global ** 2 + rse ** 2)
    assert abs(z) < 4.0, z
    # per-entry law: E[values] is the splitting product x (K5, deterministic).
    # R independent GPU runs: their mean must close in on x as 1/sqrt(R) (no
    # per-entry bias), and the reference's distance to x must match a single
    # GPU run's (same per-entry noise).
    x = pb.splitting_product(m, v, p)
    R = 8
    runs = [got.values] + [pb.vector_estimate(
        m, v, pb.PathParams(beta, 32, M, pb.Splitting(splitting), 1000 + r)).values
        for r in range(R - 1)]
    l1 = lambda y: np.abs(y - x).sum() / np.abs(x).sum()
    e_single = np.mean([l1(y) for y in runs])
    e_mean = l1(np.mean(runs, axis=0))
    e_ref = l1(rv)
    assert e_mean < 1.5 * e_single / math.sqrt(R), (e_mean, e_single)
    assert e_single / 1.6 < e_ref < 1.6 * e_single, (e_ref, e_single)
    assert abs(got.total_jumps / rj - 1) < 0.01
    t = pb.tc_estimate(m, p)
    tv, tse, tj = rm.tc_estimate(beta, 32, M, splitting, 10, workers=16)
    assert abs(t.value - tv) < 4.0 * math.sqrt(t.std_error ** 2 + tse ** 2)


def test_vector_matches_splitting_product(pb):
    """K4 values against the deterministic splitting product (K5) the walkers
    sample, on a graph with hubs: per-entry z over the rows that collect many
    walkers, and the global functional."""
    csr = pb.gen_ba(3000, 4, 2)
    m = pb.split(csr)
    v = pb.gen_vector(0, csr.n, 5) + 0.05
    p = pb.PathParams(0.05, 32, 30_000_000, pb.Splitting.Strang, 3)
    got = pb.vector_estimate(m, v, p)
    x = pb.splitting_product(m, v, p)
    assert abs(got.values.sum() - x.sum()) < 4 * got.std_error_global
    rel = np.abs(got.values - x).sum() / np.abs(x).sum()
    assert rel < 0.03, rel


def test_isolated_rows_and_single_row(pb, ref):
    """Rows with rate 0 never jump (exp_time returns +inf, sampler.cpp:12):
    all their walkers score at their start."""
    a = np.zeros((5, 5))
    a[0, 1] = a[1, 0] = 2.0
    np.fill_diagonal(a, [0.1, -0.2, 0.3, -0.4, 0.5])
    csr = pb.csr_from_dense(a)
    m = pb.split(csr)
    v = np.array([1.0, 2.0, 3.0, 0.0, 5.0])
    p = pb.PathParams(1.0, 16, 2_000_000, pb.Splitting.Strang, 4)
    got = pb.vector_estimate(m, v, p)
    V = v.sum()
    for i in (2, 3, 4):  # isolated: value_i = v_i e^{β a_ii} exactly in law; counts ~ v_i / V
        exp_i = v[i] * math.exp(a[i, i])
        if v[i] == 0:
            assert got.values[i] == 0
        else:
            sd = V * math.exp(a[i, i]) * math.sqrt(v[i] / V * (1 - v[i] / V) / p.samples)
            assert abs(got.values[i] - exp_i) < 5 * sd
    rm = ref.matrix_from_csr(csr)
    rv, rse, rj, _ = rm.vector_estimate(v, 1.0, 16, 2_000_000, 1, 4, workers=16)
    z = (got.values.sum() - rv.sum()) / math.sqrt(got.std_error_global ** 2 + rse ** 2)
    assert abs(z) < 4
    one = pb.split(pb.csr_from_dense(np.array([[0.25]])))
    r = pb.vector_estimate(one, [2.0], pb.PathParams(2.0, 8, 1000, seed=1))
    assert r.values[0] == pytest.approx(2.0 * math.exp(0.5), rel=1e-14)
    assert r.std_error_global <= 1e-6 * r.values[0] and r.total_jumps == 0


@pytest.mark.parametrize("shards", [2, 3, 7])
def test_start_row_shards_reproduce_unsharded(pb, shards):
    """Multi-GPU path of the Theorem-2 estimators, on one GPU:
    the row shards run exactly the unsharded call's walkers, so their
    rank-ordered combination equals vector_estimate / tc_estimate up to fp
    summation order (1e-12), with identical jump counts."""
    from paper_1904_12759_b200.shard import combine_tc_shards, combine_vector_shards, plan_shards

    csr = pb.gen_ba(5000, 4, 3)
    m = pb.split(csr)
    v = pb.gen_vector(0, csr.n, 8) + 0.01
    p = pb.PathParams(0.08, 32, 20_000_000, pb.Splitting.Strang, 21)
    full = pb.vector_estimate(m, v, p)
    parts = [pb.vector_estimate_rows(m, v, p, lo, hi) for lo, hi in plan_shards(csr.n, shards)]
    got = combine_vector_shards(parts, p.samples, full.v_sum)
    assert got.total_jumps == full.total_jumps
    np.testing.assert_allclose(got.values, full.values, rtol=1e-12, atol=1e-14 * full.values.max())
    assert got.std_error_global == pytest.approx(full.std_error_global, rel=1e-9)
    t = pb.tc_estimate(m, p)
    tp = combine_tc_shards([pb.tc_estimate_rows(m, p, lo, hi)
                            for lo, hi in plan_shards(csr.n, shards)], p.samples)
    assert tp.total_jumps == t.total_jumps
    assert tp.value == pytest.approx(t.value, rel=1e-12)
    assert tp.std_error == pytest.approx(t.std_error, rel=1e-9)


def test_shard_argument_checks(pb):
    m = pb.split(pb.gen_fd(2, 4, 1.0))
    v = np.ones(m.n)
    with pytest.raises(ValueError, match="row range out of bounds"):
        pb.vector_estimate_rows(m, v, pb.PathParams(samples=10), 3, 2)
    with pytest.raises(ValueError, match="row shards need the Philox engine"):
        pb.tc_estimate_rows(m, pb.PathParams(samples=10, rng=pb.Rng.PCG_COMPAT), 0, 4)


def test_tiny_horizon_jump_counts(pb):
    """λ = rate β ~ 1e-6: almost every walker stays put; the number of
    jumpers (and jumps) must follow M E[1 - e^{-λ_start}] — the small-λ end
    of the never-jumper split (jump probability from expm1, no cancellation)."""
    csr = pb.gen_ws(2000, 5, 0.1, 9)
    m = pb.split(csr)
    beta = 1e-7
    M = 200_000_000
    rate = m.export()["rate"]
    lam = rate * beta
    expect = M * np.mean(-np.expm1(-lam))          # uniform starts (tc)
    t = pb.tc_estimate(m, pb.PathParams(beta, 8, M, pb.Splitting.Strang, 5))
    jumpers = pb.last_jumpers(m)
    assert abs(jumpers - expect) < 5 * math.sqrt(expect), (jumpers, expect)
    # second jumps within 1e-7 are ~λ times rarer: jumps ≈ jumpers
    assert jumpers <= t.total_jumps < jumpers + 5 + 5 * math.sqrt(expect * lam.max() + 1)


@pytest.mark.parametrize("name,beta", [("ba_2000", 0.05), ("weighted_40", 0.7),
                                       ("fd3d_10", 0.004)])
def test_fixed_point_and_sort_reductions_agree(pb, name, beta, monkeypatch):
    """vector_estimate's two per-end reductions — exact 128-bit fixed point
    (order-independent integer sums) and the sort-based sequential fp64 sums —
    reduce the same walkers: per entry they agree to fp64 summation error,
    and tallies / jumps are identical."""
    from test_gpu_parity import _graphs

    csr = _graphs(pb)[name]
    m = pb.split(csr)
    v = pb.gen_vector(0, csr.n, 4) + 0.02
    p = pb.PathParams(beta, 32, 3_000_000, pb.Splitting.Lie, 17)
    monkeypatch.delenv("EXPMC_K4_SORT", raising=False)
    a = pb.vector_estimate(m, v, p)
    assert pb.last_k4_stats(m)[1] == 1
    monkeypatch.setenv("EXPMC_K4_SORT", "1")
    b = pb.vector_estimate(m, v, p)
    assert pb.last_k4_stats(m)[1] == 0
    assert a.total_jumps == b.total_jumps and a.std_error_global == b.std_error_global
    np.testing.assert_allclose(a.values, b.values, rtol=1e-12, atol=0)


def test_fixed_point_falls_back_on_wide_weight_range(pb, ref):
    """When e^{β (d_max - d_min)} times M does not fit the 128-bit window
    (BA hubs at a large β), vector_estimate uses the sort-based reduction and
    still agrees with the reference."""
    csr = pb.gen_ba(2000, 5, 1)
    m = pb.split(csr)
    v = pb.gen_vector(0, csr.n, 4) + 0.02
    beta = 0.6  # d_max ~ 150 -> e^{90}
    p = pb.PathParams(beta, 64, 400_000, pb.Splitting.Strang, 2)
    got = pb.vector_estimate(m, v, p)
    assert pb.last_k4_stats(m)[1] == 0
    rv, rse, _, _ = ref.matrix_from_csr(csr).vector_estimate(v, beta, 64, 400_000, 1, 3,
                                                             workers=16)
    z = (got.values.sum() - rv.sum()) / math.sqrt(got.std_error_global ** 2 + rse ** 2)
    assert abs(z) < 4.0


@pytest.mark.parametrize("splitting", [0, 1])
def test_entries_beyond_2_29_walkers(pb, splitting):
    """entry_estimate accepts any `samples` (estimator.hpp:19): W >= 2^29
    takes the grouped large-W path.  Against the K3 walker just below the
    threshold (same law) and against the splitting product x (the exact mean)
    within 5 combined SE; signed v, rows with never-jumper majority (K = f0)
    and with jumper majority (K = 0)."""
    a = np.zeros((6, 6))
    for i, j, w in [(0, 1, 1.0), (1, 2, 2.0), (2, 3, 0.5), (3, 4, 3.0), (4, 5, 1.0), (0, 5, 0.25)]:
        a[i, j] = a[j, i] = w
    np.fill_diagonal(a, [0.1, -0.3, 0.2, 0.0, -0.1, 0.4])
    csr = pb.csr_from_dense(a)
    m = pb.split(csr)
    v = np.array([1.0, -0.5, 2.0, 0.3, -1.2, 0.7])
    beta = 0.2   # λ from 0.05 (row 0: K = f0) to 0.8 (row 3: K = 0)
    rows = np.arange(6, dtype=np.uint32)
    big = pb.entries_estimate(m, v, rows, pb.PathParams(beta, 16, 1 << 29, pb.Splitting(splitting), 7))
    Ws = 1 << 25  # K3 (the threshold's other side; few rows => slow at 2^29 - 1)
    small = pb.entries_estimate(m, v, rows, pb.PathParams(beta, 16, Ws, pb.Splitting(splitting), 8))
    x = pb.splitting_product(m, v, pb.PathParams(beta, 16, 10, pb.Splitting(splitting)))
    assert np.all(big.std_errors > 0)
    z = (big.values - small.values) / np.sqrt(big.std_errors ** 2 + small.std_errors ** 2)
    assert np.all(np.abs(z) < 5), z
    zx = (big.values - x) / big.std_errors
    assert np.all(np.abs(zx) < 5), zx
    # jump counts: same law as K3's (mean jumps per walker)
    jb, js = big.jumps / float(1 << 29), small.jumps / float(Ws)
    assert np.all(np.abs(jb - js) < 6 * np.sqrt(2.0 * np.maximum(js, 1e-9) / Ws) + 1e-12)
    # the single-entry call routes the same way: the same walkers (keyed by
    # row and walker), summed with a different piece alignment
    e = pb.entry_estimate(m, v, 3, pb.PathParams(beta, 16, 1 << 29, pb.Splitting(splitting), 7))
    assert e.total_jumps == big.jumps[3]
    assert e.value == pytest.approx(big.values[3], rel=1e-11)
    assert e.std_error == pytest.approx(big.std_errors[3], rel=1e-9)


def test_entries_beyond_2_29_walkers_hub_and_leaf_rows(pb):
    """Regression (round-1 advisor finding): the W >= 2^29 path once summed
    in a 128-bit fixed-point window sized from e^{beta d_max} max|v| of the
    whole matrix; with a hub at e^{beta d} ~ 1e139 every O(1) deviation of an
    ordinary row truncated to 0 (value = K, SE = 0).  Now each row's
    deviations are summed in fp64 by the deterministic run-sum passes.
    Ordinary rows of a small component next to a 2000-leaf star hub: W = 2^29
    against K3 at W = 2^25 and against the splitting product."""
    D = 2000
    n = D + 1 + 5
    rows_, cols_, w_ = [], [], []
    for k in range(1, D + 1):  # star: hub 0, leaves 1..D
        rows_ += [0, k]
        cols_ += [k, 0]
        w_ += [1.0, 1.0]
    path = list(range(D + 1, n))  # a separate 5-node weighted path
    for a, b, w in zip(path[:-1], path[1:], [1.0, 0.5, 2.0, 1.5]):
        rows_ += [a, b]
        cols_ += [b, a]
        w_ += [w, w]
    order = np.lexsort((np.array(cols_), np.array(rows_)))
    r_, c_, ww = np.array(rows_)[order], np.array(cols_)[order], np.array(w_)[order]
    rp = np.zeros(n + 1, np.uint64)
    np.add.at(rp, r_ + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    csr = pb.Csr(n, rp, c_.astype(np.uint32), ww, np.zeros(n))
    m = pb.split(csr)
    v = np.ones(n)
    v[path] = [0.3, -1.0, 0.8, 0.5, -0.2]
    beta = 0.16  # hub: e^{beta d} = e^{320}
    rows = np.array(path, np.uint32)
    big = pb.entries_estimate(m, v, rows, pb.PathParams(beta, 32, 1 << 29, pb.Splitting.Strang, 7))
    Ws = 1 << 25
    small = pb.entries_estimate(m, v, rows, pb.PathParams(beta, 32, Ws, pb.Splitting.Strang, 8))
    x = pb.splitting_product(m, v, pb.PathParams(beta, 32, 10, pb.Splitting.Strang))[path]
    assert np.all(big.std_errors > 0), big.std_errors
    z = (big.values - small.values) / np.sqrt(big.std_errors ** 2 + small.std_errors ** 2)
    assert np.all(np.abs(z) < 5), z
    assert np.all(np.abs((big.values - x) / big.std_errors) < 5)
    # the hub row itself: every walker leaves at once (K = 0), huge values
    hub = pb.entries_estimate(m, v, np.array([0], np.uint32),
                              pb.PathParams(beta, 32, 1 << 29, pb.Splitting.Strang, 7))
    assert np.isfinite(hub.values[0]) and hub.std_errors[0] > 0


@pytest.mark.parametrize("M", [1, 2, 3, 33, 1000])
def test_small_sample_counts(pb, ref, M):
    """Tiny M (down to one walker): the start tree, the never-jumper split
    and the jumper batches handle empty rows and empty batches; tallies obey
    finalize (SE 0 for M = 1)."""
    from test_gpu_parity import _graphs

    csr = _graphs(pb)["weighted_40"]
    m = pb.split(csr)
    v = pb.gen_vector(0, csr.n, 6)
    v[[0, -1]] = 0.0  # zero mass at both ends of the cumulative table
    p = pb.PathParams(0.5, 16, M, pb.Splitting.Strang, 3)
    r = pb.vector_estimate(m, v, p)
    assert np.all(np.isfinite(r.values)) and r.samples_used == M
    assert r.values[0] >= 0 and (r.values > 0).sum() <= M
    # Σ values = mean of V w over the M walkers, whose SE is std_error_global
    if M == 1:
        assert r.std_error_global == 0.0
    t = pb.tc_estimate(m, p)
    assert np.isfinite(t.value) and t.samples_used == M
    c = pb.start_counts(m, v, M, seed=3)
    assert c.sum() == M and c[0] == 0 and c[-1] == 0
