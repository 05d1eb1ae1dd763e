"""Synthetic inputs for BASELINE.json configs 1-5 (host C++ builders in
csrc/gen.cpp, called through the C ABI).

Config table (seeds: graph 1, v 2, paths 3, row sample 4):

  1  FD2D 64x64 Dirichlet (diag -4, off +1), v ~ U[0,1), t = 1, W = 1e4, all rows
  2  BA n=1e5 m0=5, v = 1, beta = 0.5 / lambda_max (stats, 100 power iters), W = 1e4
  3  WS n=1e6 k=10 p=0.1, v = 1, beta = 0.05, W = 2e3, all rows
  4  FD3D 256^3 scaled 1/h^2 (h = 1/257), v = bump(sigma 0.1) + U[0,1), t = 1e-4,
     W = 1e4, 1e6 rows sampled without replacement
  5  BA n=1e7 m0=8, v ~ U[-1,1), beta = 0.02, W = 1e3, all rows

N rule: N = max(32, next_pow2(ceil(beta * max_i |d_i|))).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from ._lib import check, f64p, lib, u32p, u64p


@dataclass
class Csr:
    """Mirrored, row-sorted adjacency + diagonal (the SparseSymmetric view)."""
    n: int
    row_ptr: np.ndarray  # uint64, n+1
    col: np.ndarray      # uint32
    val: np.ndarray      # float64
    diag: np.ndarray     # float64, n

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.n else 0


def _take(h) -> Csr:
    L = lib()
    n, nnz = C.c_uint64(), C.c_uint64()
    L.expmc_csr_sizes(h, C.byref(n), C.byref(nnz))
    c = Csr(n.value, np.zeros(n.value + 1, np.uint64), np.zeros(nnz.value, np.uint32),
            np.zeros(nnz.value), np.zeros(n.value))
    L.expmc_csr_export(h, c.row_ptr.ctypes.data_as(u64p), c.col.ctypes.data_as(u32p),
                       c.val.ctypes.data_as(f64p), c.diag.ctypes.data_as(f64p))
    L.expmc_csr_free(h)
    return c


def gen_fd(dim: int, side: int, scale: float = 1.0) -> Csr:
    h = C.c_void_p()
    check(lib().expmc_gen_fd(dim, side, scale, C.byref(h)), gen=True)
    return _take(h)


def gen_ba(n: int, m0: int, seed: int) -> Csr:
    h = C.c_void_p()
    check(lib().expmc_gen_ba(n, m0, seed, C.byref(h)), gen=True)
    return _take(h)


def gen_ws(n: int, half_k: int, p: float, seed: int) -> Csr:
    h = C.c_void_p()
    check(lib().expmc_gen_ws(n, half_k, p, seed, C.byref(h)), gen=True)
    return _take(h)


def gen_vector(kind: int, n: int, seed: int, side: int = 0, sigma: float = 0.0) -> np.ndarray:
    out = np.zeros(n)
    check(lib().expmc_gen_vector(kind, n, side, sigma, seed, out.ctypes.data_as(f64p)),
          gen=True)
    return out


def gen_row_sample(n: int, k: int, seed: int) -> np.ndarray:
    out = np.zeros(k, np.uint32)
    check(lib().expmc_gen_row_sample(n, k, seed, out.ctypes.data_as(u32p)), gen=True)
    return out


# ------------------------------------------- Matrix Market + CSR cache (f1, f3)
@dataclass
class MmEntries:
    """One parsed Matrix Market file before the fold / from_entries."""
    n: int
    general: bool
    pattern: bool
    last_line: int
    rows: np.ndarray   # uint32, 0-based, file order
    cols: np.ndarray
    weights: np.ndarray


def parse_matrix_market(path) -> MmEntries:
    """The parse half of load_matrix_market (matrix_market.cpp:51-131), on all
    host cores.  Errors raise ExpmcError("path:line: what")."""
    L = lib()
    h = C.c_void_p()
    check(L.expmc_mm_parse(os.fsencode(path), C.byref(h)), gen=True)
    try:
        n, ne, last = C.c_uint64(), C.c_uint64(), C.c_uint64()
        g, pt = C.c_int32(), C.c_int32()
        check(L.expmc_mm_info(h, C.byref(n), C.byref(ne), C.byref(g), C.byref(pt), C.byref(last)),
              gen=True)
        r, c, w = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(L.expmc_mm_view(h, C.byref(r), C.byref(c), C.byref(w)), gen=True)
        k = ne.value

        def arr(p, t, dt):
            if k == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(t)), (k,)).astype(dt, copy=True)

        return MmEntries(n.value, bool(g.value), bool(pt.value), last.value,
                         arr(r, C.c_uint32, np.uint32), arr(c, C.c_uint32, np.uint32),
                         arr(w, C.c_double, np.float64))
    finally:
        L.expmc_mm_free(h)


def load_matrix_market(path, device=0) -> Csr:
    """load_matrix_market (matrix_market.cpp:51-165) -> the SparseSymmetric
    adjacency (fold + from_entries on the GPU)."""
    h = C.c_void_p()
    check(lib().expmc_cuda_mm_load(os.fsencode(path), int(device), C.byref(h)))
    return _take(h)


def _csr_args(csr: Csr):
    rp = np.ascontiguousarray(csr.row_ptr, np.uint64)
    col = np.ascontiguousarray(csr.col, np.uint32)
    val = np.ascontiguousarray(csr.val, np.float64)
    diag = np.ascontiguousarray(csr.diag, np.float64)
    return (int(csr.n), rp.ctypes.data_as(u64p), col.ctypes.data_as(u32p),
            val.ctypes.data_as(f64p), diag.ctypes.data_as(f64p)), (rp, col, val, diag)


def write_matrix_market(csr: Csr, path) -> None:
    """write_matrix_market (matrix_market.cpp:167-194): lower triangle,
    1-based, ``pattern`` when every weight is 1, shortest round-trip reals."""
    args, _keep = _csr_args(csr)
    check(lib().expmc_mm_write(os.fsencode(path), *args), gen=True)


def save_csr(csr: Csr, path) -> None:
    """Binary CSR cache: header + arrays + checksum."""
    args, _keep = _csr_args(csr)
    check(lib().expmc_csr_save(os.fsencode(path), *args), gen=True)


def load_csr(path) -> Csr:
    """Read a binary CSR cache written by :func:`save_csr` (size, checksum and
    row_ptr verified)."""
    h = C.c_void_p()
    check(lib().expmc_csr_load(os.fsencode(path), C.byref(h)), gen=True)
    return _take(h)


def _cached(name: str, make) -> Csr:
    """Generated graph through the CSR cache in $EXPMC_CSR_CACHE (if set)."""
    d = os.environ.get("EXPMC_CSR_CACHE")
    if not d:
        return make()
    path = os.path.join(d, name + ".csr")
    if os.path.exists(path):
        try:
            return load_csr(path)
        except Exception:
            pass  # stale / corrupt: regenerate
    csr = make()
    os.makedirs(d, exist_ok=True)
    tmp = f"{path}.{os.getpid()}.tmp"
    save_csr(csr, tmp)
    os.replace(tmp, path)
    return csr


def csr_from_dense(a: np.ndarray) -> Csr:
    """Small symmetric dense matrix -> Csr (tests)."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    rp = [0]
    cols, vals = [], []
    for i in range(n):
        for j in range(n):
            if i != j and a[i, j] != 0.0:
                cols.append(j)
                vals.append(a[i, j])
        rp.append(len(cols))
    return Csr(n, np.array(rp, np.uint64), np.array(cols, np.uint32), np.array(vals, np.float64),
               np.diag(a).copy())


def n_rule(beta: float, d: np.ndarray) -> int:
    """N = max(32, next_pow2(ceil(beta * max|d|)))."""
    x = beta * float(np.max(np.abs(d))) if len(d) else 0.0
    k = max(1, math.ceil(x))
    return max(32, 1 << (k - 1).bit_length())


def split_d(csr: Csr) -> np.ndarray:
    """d = diag + rate on the host (only for the N rule; the GPU split is the
    product path)."""
    cs = np.concatenate([[0.0], np.cumsum(csr.val)])
    rp = csr.row_ptr.astype(np.int64)
    return csr.diag + (cs[rp[1:]] - cs[rp[:-1]])


@dataclass
class Config:
    idx: int
    name: str
    csr: Csr
    v: np.ndarray
    rows: np.ndarray | None   # None = every row
    beta: float
    n_steps: int
    walkers: int
    note: str = ""

    @property
    def nrows(self) -> int:
        return self.csr.n if self.rows is None else len(self.rows)


def build_config(idx: int, scale: float = 1.0, lambda_max=None) -> Config:
    """Inputs of BASELINE.json config ``idx`` (1-based).  ``scale`` < 1 shrinks
    n (tests / quick runs); 1.0 is the named configuration."""
    if idx == 1:
        side = max(4, int(round(64 * math.sqrt(scale))))
        csr = gen_fd(2, side, 1.0)
        v = gen_vector(0, csr.n, 2)
        beta, W, rows, name = 1.0, 10_000, None, f"fd2d_{side}x{side}"
    elif idx == 2:
        n = max(1000, int(1e5 * scale))
        csr = _cached(f"ba_n{n}_m5_s1", lambda: gen_ba(n, 5, 1))
        v = np.ones(n)
        if lambda_max is None:
            from .estimator import split as _split
            from .spectral import lambda_max as _lm
            lambda_max = _lm(_split(csr), 100)
        beta, W, rows, name = 0.5 / lambda_max, 10_000, None, f"ba_n{n}_m5"
    elif idx == 3:
        n = max(1000, int(1e6 * scale))
        csr = _cached(f"ws_n{n}_k5_p0.1_s1", lambda: gen_ws(n, 5, 0.1, 1))
        v = np.ones(n)
        beta, W, rows, name = 0.05, 2_000, None, f"ws_n{n}_k10_p0.1"
    elif idx == 4:
        side = max(8, int(round(256 * scale ** (1 / 3))))
        h = 1.0 / (side + 1)
        csr = gen_fd(3, side, 1.0 / (h * h))
        v = gen_vector(2, csr.n, 2, side=side, sigma=0.1)
        k = min(csr.n, max(1, int(1e6 * scale)))
        rows = gen_row_sample(csr.n, k, 4)
        beta, W, name = 1e-4, 10_000, f"fd3d_{side}^3"
    elif idx == 5:
        n = max(1000, int(1e7 * scale))
        csr = _cached(f"ba_n{n}_m8_s1", lambda: gen_ba(n, 8, 1))
        v = gen_vector(1, n, 2)
        beta, W, rows, name = 0.02, 1_000, None, f"ba_n{n}_m8"
    else:
        raise ValueError("config index must be 1..5")
    N = n_rule(beta, split_d(csr))
    return Config(idx, name, csr, v, rows, beta, N, W)
