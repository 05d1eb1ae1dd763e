"""CPU tests: pin the oracle (oracle/liboracle.so, the C restatement of the
reference hot path) against the golden fixtures generated from the compiled
reference (tests/golden/make_golden.py), and check the CPU model of the
Philox walker against curand's Philox and against the reference's law.

Tolerances: the restatement must reproduce the reference BIT FOR BIT
(same algorithm, same operation order, same glibc libm, workers = 1)."""
import json
import math
import os
from types import SimpleNamespace

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def hx(a):
    return np.array([float.fromhex(x) for x in a])


def csr_from_gold(g):
    return SimpleNamespace(n=g["n"], row_ptr=np.array(g["row_offset"], np.uint64),
                           col=np.array(g["neighbor"], np.uint32), val=hx(g["weight"]),
                           diag=hx(g["diag"]))


def test_pcg32_public_sequence(orc):
    # RngStream(42, 54) reproduces the public pcg32 demo output
    got = orc.rng_draws(42, 54, 0, 4)
    assert [hex(x) for x in got] == ["0xa15c02b7", "0x7b47f409", "0xba1d3330", "0x83d2f293"]


def test_rng_matches_reference_golden(orc):
    g = load("rng.json")
    assert list(orc.rng_draws(42, 54, 0, 8)) == g["pcg32_demo_42_54_u32"]
    s = g["s1_0"]
    assert list(orc.rng_draws(1, 0, 0, 6)) == s["u32"]
    assert [str(int(x)) for x in orc.rng_draws(1, 0, 1, 6)] == s["u64"]
    assert np.array_equal(orc.rng_draws(1, 0, 2, 6), hx(s["uniform"]))
    assert np.array_equal(orc.rng_draws(1, 0, 3, 6), hx(s["uniform_pos"]))
    assert list(orc.rng_draws(1, 0, 4, 6, 10)) == s["uniform_index_10"]
    assert np.array_equal(orc.rng_draws(7, 3, 2, 6), hx(g["s7_3_uniform"]))
    assert list(orc.rng_draws(2024, 99, 4, 6, 1000)) == g["s2024_99_uniform_index_1000"]
    assert np.array_equal(orc.exp_times(1, 0, 2.0, 6), hx(g["exp_time_1_0_rate2"]))
    assert np.array_equal(orc.exp_times(5, 8, 0.5, 6), hx(g["exp_time_5_8_rate0_5"]))
    assert math.isinf(orc.exp_times(1, 0, 0.0, 1)[0])  # rate 0 -> +inf


def test_split_bit_exact_vs_reference_golden(orc):
    for name, g in load("split.json").items():
        s = orc.split(csr_from_gold(g))
        for k in ("d", "rate", "cum", "diag"):
            assert np.array_equal(s[k], hx(g[k])), (name, k)
        assert list(s["uniform_row"]) == g["uniform_row"], name
        assert s["dbar"] == float.fromhex(g["dbar"]) and s["dmax"] == g["dmax"], name


def test_estimators_bit_exact_vs_reference_golden(orc):
    splits = load("split.json")
    for name, e in load("estimates.json").items():
        s = orc.split(csr_from_gold(splits[name]))
        v, vpos = hx(e["v"]), hx(e["vpos"])
        for c in e["cases"]:
            if c["kind"] == "entry":
                val, se, j = orc.entry_estimate(s, v, c["i"], c["beta"], c["n_steps"],
                                                c["samples"], c["splitting"], c["seed"])
                assert val == float.fromhex(c["value"]) and se == float.fromhex(c["se"]), (name, c)
                assert j == c["jumps"]
            elif c["kind"] == "vector":
                vals, se, j, vs = orc.vector_estimate(s, vpos, c["beta"], c["n_steps"],
                                                      c["samples"], c["splitting"], c["seed"])
                assert np.array_equal(vals, hx(c["values"])), name
                assert se == float.fromhex(c["se"]) and j == c["jumps"]
                assert vs == float.fromhex(c["v_sum"])
            else:
                val, se, j = orc.tc_estimate(s, c["beta"], c["n_steps"], c["samples"],
                                             c["splitting"], c["seed"])
                assert val == float.fromhex(c["value"]) and se == float.fromhex(c["se"])
                assert j == c["jumps"]


def test_advance_vs_reference_golden(orc):
    splits = load("split.json")
    for name, a in load("advance.json").items():
        s = orc.split(csr_from_gold(splits[name]))
        end, jumps = orc.advance_many(s, a["seed"], a["start"], a["dt"], len(a["end"]))
        assert list(end) == a["end"] and list(jumps) == a["jumps"], name


def test_survey_p3_fixture(orc):
    """entry_estimate(i=1, v=(1,2,-0.5), beta=1, N=8, M=1e5,
    seed=2024, workers=1) on the P3 graph."""
    g = load("split.json")["p3"]
    s = orc.split(csr_from_gold(g))
    v = [1.0, 2.0, -0.5]
    assert orc.entry_estimate(s, v, 1, 1.0, 8, 100_000, 1, 2024)[0] == 31.248671410962384
    assert orc.entry_estimate(s, v, 1, 1.0, 8, 100_000, 0, 2024)[0] == 30.938284991716518
    assert orc.entry_estimate(s, v, 1, 1.0, 8, 100_000, 1, 2024)[2] == 308153


def test_spec_kats(orc):
    """SPEC.md KATs on the oracle: single edge entry (0,0) ~ cosh 1 (:191),
    TC of a regular graph is deterministic 2e (:210), Exp(2) mean (:120)."""
    g = load("split.json")["single_edge"]
    s = orc.split(csr_from_gold(g))
    val, se, _ = orc.entry_estimate(s, [1.0, 0.0], 0, 1.0, 32, 200_000, 1, 7)
    assert abs(val - math.cosh(1.0)) < 4 * se
    tc, tse, _ = orc.tc_estimate(s, 1.0, 32, 10_000, 1, 7)
    assert abs(tc - 2 * math.e) < 1e-12 and tse < 1e-12
    x = orc.exp_times(3, 1, 2.0, 1_000_000)
    assert abs(x.mean() - 0.5) < 3 * x.std() / 1000.0
    # 2-state chain P(end != start) at dt = 0.5 = (1 - e^-1)/2
    end, _ = orc.advance_many(s, 11, 0, 0.5, 100_000)
    p = (1 - math.exp(-1.0)) / 2
    assert abs(end.mean() - p) < 4 * math.sqrt(p * (1 - p) / 100_000)


def test_alias_tables_represent_row_weights(orc):
    g = load("split.json")["rand25_weighted"]
    s = orc.split(csr_from_gold(g))
    s.update(row_offset=np.array(g["row_offset"], np.uint64),
             neighbor=np.array(g["neighbor"], np.uint32), weight=hx(g["weight"]))
    thr, al = orc.alias_build(s)
    ro = s["row_offset"]
    for i in range(g["n"]):
        lo, hi = int(ro[i]), int(ro[i + 1])
        if hi == lo:
            continue
        deg = hi - lo
        prob = np.zeros(deg)
        for k in range(deg):
            keep = thr[lo + k] / 2.0 ** 32
            prob[k] += keep / deg
            prob[al[lo + k]] += (1 - keep) / deg
        np.testing.assert_allclose(prob, s["weight"][lo:hi] / s["rate"][i], atol=1e-9)


def test_model_philox_matches_curand(orc):
    for c in load("philox.json")["cases"]:
        assert list(orc.philox(c["ctr"], c["key"])) == c["out"]


def test_model_neg_ln_accuracy(orc):
    """neg_ln_u(w) = -ln(u), u = (w | 1) 2^-32 (31-bit midpoint uniform), to
    1.5e-7 max(1, E) absolute (fp32: x is rounded to 24 bits); never negative."""
    ws = np.random.default_rng(0).integers(0, 2**32, 40000, dtype=np.uint64)
    edge = [0, 1, 2, 3, 511, 512, 2**24 - 1, 2**24, 2**24 + 1, 2**31, 2**32 - 129, 2**32 - 128,
            2**32 - 2, 2**32 - 1]
    for w in list(ws) + edge:
        w = int(w)
        want = 32 * math.log(2.0) - math.log(w | 1)
        got = orc.neg_ln_u(w)
        assert got >= 0.0
        assert abs(got - want) <= 1.5e-7 * max(1.0, want), (w, got, want)
    assert orc.neg_ln_u(0) == pytest.approx(32 * math.log(2.0), rel=1e-7)


def test_model_exp_det_accuracy(orc):
    """The walker's deterministic exp (exp_det / fm_exp) is within 1 ulp of
    glibc exp over the whole finite range, including subnormal results."""
    import ctypes

    f = orc.L.fm_exp
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-745, 709.78, 20000), rng.uniform(-3, 3, 20000),
                         [0.0, 709.43, 709.44, 709.78, -708.4, -744.9]])
    for x in xs:
        a, b = f(float(x)), math.exp(float(x))
        assert abs(a - b) <= math.ulp(b), (x, a, b)
    assert math.isinf(f(710.0)) and f(-800.0) == 0.0


def test_model_law_matches_reference(orc, ref):
    """The continuous-clock Philox walker (CPU model of K3) samples the same
    law as the reference: per-entry z-scores over several graphs."""
    import paper_1904_12759_b200 as pb

    zs = []
    for csr, beta in ((pb.gen_fd(2, 8, 1.0), 1.0), (pb.gen_ba(400, 3, 2), 0.2)):
        s = orc.split(csr)
        rm = ref.matrix_from_csr(csr)
        v = pb.gen_vector(0, csr.n, 5) + 0.2
        rows = np.arange(0, csr.n, max(1, csr.n // 40), dtype=np.uint32)
        for split_mode in (0, 1):
            mv, ms, _ = orc.fast_entries(s, v, rows, beta, 16, 4000, split_mode, 9, 32)
            rv, rse, _ = rm.entries(v, rows, beta, 16, 4000, split_mode, 10, workers=1,
                                    threads=8)
            zs.append((mv - rv) / np.sqrt(ms ** 2 + rse ** 2))
    z = np.concatenate(zs)
    assert np.sum(np.abs(z) > 4) <= 1
    assert abs(z.mean()) < 0.25 and 0.6 < z.var() < 1.5


def test_model_jump_count_matches_rate(orc):
    """AC7: jumps per path ~ beta * rate on a regular graph."""
    import paper_1904_12759_b200 as pb

    csr = pb.gen_ws(500, 2, 0.0, 1)  # 4-regular ring
    s = orc.split(csr)
    rows = np.arange(0, 500, 25, dtype=np.uint32)
    _, _, j = orc.fast_entries(s, np.ones(500), rows, 1.5, 32, 5000, 1, 3, 32)
    per_path = j.sum() / (len(rows) * 5000)
    assert abs(per_path - 1.5 * 4) / 6.0 < 0.05


@pytest.mark.parametrize("lam", [1e-4, 0.02, 0.3, 2.0, 12.0])
def test_model_gap_decisions_poisson_law(orc, lam):
    """Gap decisions (E = λK + R) keep the per-walker law: on a 2-regular
    ring every state has rate 2, so a walker's jump count is Poisson(2β).
    Covers sparse jumpers (λ = 1e-4: gaps of ~1e4 walkers), the regime of
    the headline config (λ ~ 0.3) and walkers that all jump (λ = 12)."""
    import paper_1904_12759_b200 as pb

    csr = pb.gen_ws(64, 1, 0.0, 1)  # ring: every row degree 2, weight 1
    s = orc.split(csr)
    assert np.all(s["rate"] == 2.0)
    beta = lam / 2.0
    rows = np.arange(0, 64, 8, dtype=np.uint32)
    W = 20011  # parts of unequal size (WPR = 4)
    _, _, j = orc.fast_entries(s, np.ones(64), rows, beta, 32, W, 1, 5, pb.entry_slots(W))
    n = len(rows) * W
    mean, sd = n * lam, math.sqrt(n * lam)
    assert abs(float(j.sum()) - mean) < 5 * sd + 1, (float(j.sum()), mean)
