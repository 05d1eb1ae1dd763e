"""TEST INFRASTRUCTURE ONLY — BASELINE.json config inputs built WITHOUT the
product library, for bench.py's reference arm (``--impl reference``) and
``cpu_baseline`` leg: the process that times the reference must not load
``libexpmc_b200.so``.

* Barabási–Albert (configs 2, 5): the reference's own
  ``generate({ScaleFree, n, m0, seed})`` (proj/src/generators.cpp:58-103)
  through ``oracle/_ref`` — the unmodified reference builds and splits it.
* FD2D / FD3D, Watts–Strogatz, the seeded vectors and the row sample: the
  plain-C restatements in ``oracle/inputs_gen.c`` (liboracle.so).
* config 2's beta = 0.5 / lambda_max from the reference's own
  ``stats(m, 100)`` (proj/src/sparse_matrix.cpp:176-217).

``tests/test_oracle_inputs.py`` pins these byte-for-byte against the
product's builders (paper_1904_12759_b200.inputs), so both arms of the
benchmark walk identical matrices, vectors and rows.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import HERE, Ref, RefMatrix, _f64p, _load, _u32p, _u64p


class _Gen:
    def __init__(self):
        L = _load(os.environ.get("EXPMC_ORACLE_LIB") or os.path.join(HERE, "liboracle.so"))
        L.orc_gen_fd_nnz.restype = C.c_uint64
        L.orc_gen_fd_nnz.argtypes = [C.c_int, C.c_uint64]
        L.orc_gen_fd.argtypes = [C.c_int, C.c_uint64, C.c_double, _u64p, _u32p, _f64p, _f64p]
        L.orc_gen_ws.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, _u64p, _u32p,
                                 _f64p, _f64p]
        L.orc_gen_vector.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                     _f64p]
        L.orc_gen_row_sample.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u32p]
        self.L = L


_GEN = None


def _gen():
    global _GEN
    if _GEN is None:
        _GEN = _Gen()
    return _GEN.L


@dataclass
class RefCsr:
    """Same fields as the product's inputs.Csr (n, row_ptr, col, val, diag)."""
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    diag: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.n else 0


def _p(a, t):
    return a.ctypes.data_as(t)


def gen_fd(dim: int, side: int, scale: float = 1.0) -> RefCsr:
    L = _gen()
    n = side ** dim
    nnz = int(L.orc_gen_fd_nnz(dim, side))
    c = RefCsr(n, np.zeros(n + 1, np.uint64), np.zeros(nnz, np.uint32), np.zeros(nnz),
               np.zeros(n))
    if L.orc_gen_fd(dim, side, scale, _p(c.row_ptr, _u64p), _p(c.col, _u32p),
                    _p(c.val, _f64p), _p(c.diag, _f64p)) != 0:
        raise ValueError("fd: bad arguments")
    return c


def gen_ws(n: int, half_k: int, p: float, seed: int) -> RefCsr:
    L = _gen()
    nnz = 2 * n * half_k
    c = RefCsr(n, np.zeros(n + 1, np.uint64), np.zeros(nnz, np.uint32), np.zeros(nnz),
               np.zeros(n))
    if L.orc_gen_ws(n, half_k, p, seed, _p(c.row_ptr, _u64p), _p(c.col, _u32p),
                    _p(c.val, _f64p), _p(c.diag, _f64p)) != 0:
        raise ValueError("watts-strogatz: bad arguments")
    return c


def gen_vector(kind: int, n: int, seed: int, side: int = 0, sigma: float = 0.0) -> np.ndarray:
    out = np.zeros(n)
    if _gen().orc_gen_vector(kind, n, side, sigma, seed, _p(out, _f64p)) != 0:
        raise ValueError("vector: bad arguments")
    return out


def gen_row_sample(n: int, k: int, seed: int) -> np.ndarray:
    out = np.zeros(k, np.uint32)
    if _gen().orc_gen_row_sample(n, k, seed, _p(out, _u32p)) != 0:
        raise ValueError("row sample: bad arguments")
    return out


def n_rule(beta: float, d: np.ndarray) -> int:
    """N = max(32, next_pow2(ceil(beta * max|d|)))."""
    x = beta * float(np.max(np.abs(d))) if len(d) else 0.0
    k = max(1, math.ceil(x))
    return max(32, 1 << (k - 1).bit_length())


@dataclass
class RefConfig:
    idx: int
    name: str
    matrix: RefMatrix        # the reference's SparseSymmetric + SplitMatrix
    n: int
    nnz: int
    v: np.ndarray
    rows: np.ndarray | None  # None = every row
    beta: float
    n_steps: int
    walkers: int

    @property
    def nrows(self) -> int:
        return self.n if self.rows is None else len(self.rows)


def _d_of(m: RefMatrix) -> np.ndarray:
    d = np.zeros(m.n)
    m.ref.L.ref_split_export(m.h, None, _p(d, _f64p), None, None, None, None, None, None,
                             None, None)
    return d


def build_config(idx: int, scale: float = 1.0) -> RefConfig:
    """Config ``idx`` (1-based) exactly as paper_1904_12759_b200.build_config
    builds it, from the reference and the oracle only."""
    ref = Ref()
    if idx == 1:
        side = max(4, int(round(64 * math.sqrt(scale))))
        m = ref.matrix_from_csr(gen_fd(2, side, 1.0))
        v = gen_vector(0, m.n, 2)
        beta, W, rows, name = 1.0, 10_000, None, f"fd2d_{side}x{side}"
    elif idx == 2:
        n = max(1000, int(1e5 * scale))
        m = ref.generate(1, n, m0=5, seed=1)
        v = np.ones(n)
        beta, W, rows, name = 0.5 / m.lambda_max(100), 10_000, None, f"ba_n{n}_m5"
    elif idx == 3:
        n = max(1000, int(1e6 * scale))
        m = ref.matrix_from_csr(gen_ws(n, 5, 0.1, 1))
        v = np.ones(n)
        beta, W, rows, name = 0.05, 2_000, None, f"ws_n{n}_k10_p0.1"
    elif idx == 4:
        side = max(8, int(round(256 * scale ** (1 / 3))))
        h = 1.0 / (side + 1)
        m = ref.matrix_from_csr(gen_fd(3, side, 1.0 / (h * h)))
        v = gen_vector(2, m.n, 2, side=side, sigma=0.1)
        k = min(m.n, max(1, int(1e6 * scale)))
        rows = gen_row_sample(m.n, k, 4)
        beta, W, name = 1e-4, 10_000, f"fd3d_{side}^3"
    elif idx == 5:
        n = max(1000, int(1e7 * scale))
        m = ref.generate(1, n, m0=8, seed=1)
        v = gen_vector(1, n, 2)
        beta, W, rows, name = 0.02, 1_000, None, f"ba_n{n}_m8"
    else:
        raise ValueError("config index must be 1..5")
    N = n_rule(beta, _d_of(m))
    return RefConfig(idx, name, m, m.n, m.nnz, v, rows, beta, N, W)
