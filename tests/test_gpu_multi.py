"""Multi-replica entry path (C ABI expmc_cuda_entries_multi), the staged-v
cache and the per-handle serialisation of concurrent callers, on one GPU.

The multi-GPU contract is that the gathered vector is bitwise
identical for any shard count: walker streams are keyed by (seed, row,
walker) and each row's reduction order is fixed.  On one GPU the shards are
separate replicas (handles) on the same device, run concurrently by the
library's host threads — the same code path as one replica per GPU."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(pb):
    csr = pb.gen_ba(20_000, 4, 3)
    v = pb.gen_vector(1, csr.n, 5)
    return csr, v


@pytest.mark.parametrize("nh", [2, 3, 7])
def test_entries_multi_bitwise_equals_single(pb, nh):
    csr, v = _cfg(pb)
    ms = [pb.split(csr) for _ in range(nh)]
    p = pb.PathParams(0.05, 32, 1000, pb.Splitting.Strang, 9)
    rows = np.random.default_rng(1).choice(csr.n, 5000, replace=False).astype(np.uint32)
    one = pb.entries_estimate(ms[0], v, rows, p)
    many = pb.entries_estimate_multi(ms, v, rows, p)
    assert np.array_equal(one.values, many.values)
    assert np.array_equal(one.std_errors, many.std_errors)
    assert np.array_equal(one.jumps, many.jumps)
    assert one.total_jumps == many.total_jumps
    # the full vector (rows = None) as well
    full1 = pb.entries_estimate(ms[0], v, None, p)
    fullm = pb.entries_estimate_multi(ms, v, None, p)
    assert np.array_equal(full1.values, fullm.values) and full1.total_jumps == fullm.total_jumps


def test_entries_multi_errors(pb):
    csr, v = _cfg(pb)
    m = pb.split(csr)
    p = pb.PathParams(0.05, 32, 100, pb.Splitting.Strang, 9)
    with pytest.raises(ValueError, match="distinct"):
        pb.entries_estimate_multi([m, m], v, None, p)
    other = pb.split(pb.gen_fd(2, 8))
    with pytest.raises(ValueError, match="different matrices"):
        pb.entries_estimate_multi([m, other], v, None, p)
    with pytest.raises(ValueError, match="entry index out of range"):
        pb.entries_estimate_multi([m, pb.split(csr)], v, [0, csr.n], p)
    bad = v.copy()
    bad[17] = np.nan
    with pytest.raises(ValueError, match="non-finite entry in v"):
        pb.entries_estimate_multi([m, pb.split(csr)], bad, None, p)


def test_staged_v_cache(pb):
    csr, v = _cfg(pb)
    m = pb.split(csr)
    p = pb.PathParams(0.05, 32, 2000, pb.Splitting.Strang, 4)
    ref = [pb.entry_estimate(m, v, i, p) for i in (0, 5, 17)]
    s0 = pb.v_stagings(m)
    assert s0 == 3  # cache off: every call stages v
    pb.set_v_cache(m, True)
    got = [pb.entry_estimate(m, v, i, p) for i in (0, 5, 17)]
    assert pb.v_stagings(m) == s0 + 1  # one staging, then reuse
    assert [g.value for g in got] == [r.value for r in ref]
    # a new array (other pointer) restages; in-place changes need invalidate_v
    w = v * 2.0
    e2 = pb.entry_estimate(m, w, 5, p)
    assert pb.v_stagings(m) == s0 + 2
    w *= 0.5  # now equal to v, in place: stale until invalidated
    pb.invalidate_v(m)
    e3 = pb.entry_estimate(m, w, 5, p)
    assert pb.v_stagings(m) == s0 + 3 and e3.value == ref[1].value
    assert e2.value != e3.value
    pb.set_v_cache(m, False)
    pb.entry_estimate(m, v, 5, p)
    pb.entry_estimate(m, v, 5, p)
    assert pb.v_stagings(m) == s0 + 5


def test_concurrent_callers_share_a_handle(pb):
    """Two host threads on one handle with different v: each gets exactly
    its serial result (calls on a handle are serialised by the library)."""
    csr, v = _cfg(pb)
    m = pb.split(csr)
    p = pb.PathParams(0.05, 32, 1000, pb.Splitting.Strang, 2)
    vs = [v, np.abs(v) + 0.5, -v]
    want = [pb.entries_estimate(m, x, None, p).values for x in vs]
    got = [[None] * 4 for _ in vs]
    errs = []

    def run(k):
        try:
            for r in range(4):
                got[k][r] = pb.entries_estimate(m, vs[k], None, p).values
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=run, args=(k,)) for k in range(len(vs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    for k in range(len(vs)):
        for r in range(4):
            assert np.array_equal(got[k][r], want[k])


_PIECES_SCRIPT = r"""
import sys, numpy as np
import paper_1904_12759_b200 as pb
csr = pb.gen_ba(20_000, 4, 3)
v = pb.gen_vector(1, csr.n, 5)
m = pb.split(csr)
p = pb.PathParams(0.05, 32, 1000, pb.Splitting.Strang, 9)
rows = np.random.default_rng(1).choice(csr.n, 5003, replace=False).astype(np.uint32)
a = pb.entries_estimate(m, v, rows, p)
b = pb.entries_estimate(m, v, None, p)
np.savez(sys.argv[1], av=a.values, ase=a.std_errors, aj=a.jumps, at=a.total_jumps,
         bv=b.values, bse=b.std_errors, bj=b.jumps, bt=b.total_jumps)
"""


def test_host_call_result_pieces_do_not_change_a_bit(tmp_path):
    """The host entry call walks large requests in pieces (halves, so that
    only a small last piece's copy-back is exposed: api.cu run_entries); the
    pieces are a row sharding, so any piece count gives the same bits.
    EXPMC_PIECES forces the piece path on a small request."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for pieces in ("1", "6", "13"):
        f = tmp_path / f"p{pieces}.npz"
        env = dict(os.environ, EXPMC_PIECES=pieces, PYTHONPATH=root)
        subprocess.run([sys.executable, "-c", _PIECES_SCRIPT, str(f)], check=True, env=env,
                       cwd=root, timeout=600)
        out[pieces] = np.load(f)
    for pieces in ("6", "13"):
        for k in out["1"].files:
            assert np.array_equal(out["1"][k], out[pieces][k]), (pieces, k)
