"""Randomised bit-exact parity of the entry walker against its CPU model:
seeded random graphs (weighted and unweighted, with isolated rows, hubs and
leaves), random horizons from "nobody jumps" to "everybody jumps many times",
random walker counts across the part-count thresholds, both splittings, every
launch shape.  The result contract (oracle/fast_model.c) does not depend on
the schedule, so any mismatch is a scheduling or bookkeeping bug."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _random_graph(pb, rng, n, weighted):
    a = np.zeros((n, n))
    m = int(rng.integers(n, 4 * n))
    for _ in range(m):
        i, j = rng.integers(0, n, 2)
        if i != j:
            a[i, j] = a[j, i] = float(rng.integers(1, 8)) * 0.25 if weighted else 1.0
    hub = int(rng.integers(0, n))           # one hub row
    for j in rng.choice(n, size=n // 2, replace=False):
        if j != hub:
            a[hub, j] = a[j, hub] = 1.0 if not weighted else 0.75
    iso = int(rng.integers(0, n))           # one isolated row
    if iso != hub:
        a[iso, :] = 0.0
        a[:, iso] = 0.0
    np.fill_diagonal(a, rng.normal(size=n))
    return pb.csr_from_dense(a)


# EXPMC_SOAK_CASES=N widens the sweep (profiles/r02/soak.txt: 600 cases)
@pytest.mark.parametrize("case", range(int(os.environ.get("EXPMC_SOAK_CASES", "24"))))
def test_entry_walker_random_cases_match_cpu_model(pb, orc, case, monkeypatch):
    rng = np.random.default_rng(9000 + case)
    n = int(rng.integers(8, 90))
    csr = _random_graph(pb, rng, n, weighted=bool(case % 2))
    m = pb.split(csr)
    s = orc.split(csr)
    v = rng.normal(size=n)
    beta = float(10.0 ** rng.uniform(-4, 0.6))
    W = int(rng.choice([1, 3, 127, 128, 129, 1000, 4095, 4096, 4097, 8192, 9001]))
    N = int(rng.choice([1, 8, 32, 512]))
    splitting = int(rng.integers(0, 2))
    rows = np.sort(rng.choice(n, size=min(n, int(rng.integers(1, 40))), replace=False)).astype(
        np.uint32)
    seed = int(rng.integers(0, 2 ** 40))
    mv, ms, mj = orc.fast_entries(s, v, rows, beta, N, W, splitting, seed, pb.entry_slots(W))
    p = pb.PathParams(beta, N, W, pb.Splitting(splitting), seed, pb.Rng.PHILOX)
    for shape in ("0", "1", "3"):
        monkeypatch.setenv("EXPMC_ENTRY_SHAPE", shape)
        got = pb.entries_estimate(m, v, rows, p)
        tag = (case, shape, n, beta, W, N, splitting)
        assert np.array_equal(got.values, mv), (tag, np.max(np.abs(got.values - mv)))
        assert np.array_equal(got.std_errors, ms), tag
        assert np.array_equal(got.jumps, mj), tag
