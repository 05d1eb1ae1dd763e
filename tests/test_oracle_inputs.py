"""The reference arm's inputs (oracle/inputs.py: the reference's own BA
generator plus plain-C restatements of FD / WS / vectors / row sample) are
byte-identical to the product's (paper_1904_12759_b200.inputs), so both
benchmark arms walk the same matrices, vectors and rows.  CPU only."""
import numpy as np
import pytest


def _same_csr(a, b):
    assert a.n == b.n
    for k in ("row_ptr", "col", "val", "diag"):
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and np.array_equal(x, y), k


@pytest.mark.parametrize("dim,side,scale", [(2, 1, 1.0), (2, 7, 1.0), (2, 64, 1.0),
                                            (3, 5, 1.0), (3, 9, 66049.0)])
def test_fd_matches_product(pb, dim, side, scale):
    from oracle import inputs as oi

    _same_csr(oi.gen_fd(dim, side, scale), pb.gen_fd(dim, side, scale))


@pytest.mark.parametrize("n,hk,p,seed", [(12, 1, 0.5, 3), (1000, 5, 0.1, 1), (5000, 3, 1.0, 7),
                                         (300, 2, 0.0, 2)])
def test_ws_matches_product(pb, n, hk, p, seed):
    from oracle import inputs as oi

    _same_csr(oi.gen_ws(n, hk, p, seed), pb.gen_ws(n, hk, p, seed))


def test_vectors_and_rows_match_product(pb):
    from oracle import inputs as oi

    for kind, n, side in [(0, 4096, 0), (1, 10000, 0), (2, 1000, 10), (2, 27, 3)]:
        a = oi.gen_vector(kind, n, 2, side=side, sigma=0.1)
        b = pb.gen_vector(kind, n, 2, side=side, sigma=0.1)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), kind
    for n, k in [(10, 10), (1000, 37), (4096, 1)]:
        assert np.array_equal(oi.gen_row_sample(n, k, 4), pb.gen_row_sample(n, k, 4))


@pytest.mark.parametrize("idx,scale", [(1, 1.0), (2, 0.02), (3, 0.002), (4, 0.0005),
                                       (5, 0.0003)])
def test_reference_arm_configs_match_product(pb, ref, idx, scale):
    """Every field the benchmark config dict reports, plus the arrays."""
    from oracle import inputs as oi

    a = oi.build_config(idx, scale)
    b = pb.build_config(idx, scale, lambda_max=(a.matrix.lambda_max(100) if idx == 2 else None))
    assert (a.name, a.n, a.nnz, a.walkers, a.n_steps) == (b.name, b.csr.n, b.csr.nnz,
                                                          b.walkers, b.n_steps)
    assert a.beta == b.beta
    assert np.array_equal(a.v, b.v)
    assert (a.rows is None) == (b.rows is None)
    if a.rows is not None:
        assert np.array_equal(a.rows, b.rows)
    s = a.matrix.split()
    assert np.array_equal(s["row_offset"], b.csr.row_ptr)
    assert np.array_equal(s["neighbor"], b.csr.col)
    assert np.array_equal(s["weight"], b.csr.val)


def test_config2_beta_agrees_with_product_lambda(pb, ref):
    """The product arm's beta (GPU-free here: the reference's lambda feeds
    both) — and the printed beta is rounded to 10 significant digits, so a
    last-bit difference between the two power iterations cannot split the
    config dicts."""
    from oracle import inputs as oi

    a = oi.build_config(2, 0.02)
    assert float(f"{a.beta:.10g}") == pytest.approx(a.beta, rel=1e-10)
