"""Host-side mirror of the reference estimator API, over the C ABI.

Reference interface mirrored (names, argument meaning, errors):
  PathParams, Splitting, Estimate, VectorEstimate
      /root/reference/proj/include/expmc/estimator.hpp:11-52
  entry_estimate / vector_estimate / tc_estimate
      estimator.hpp:59-72, proj/src/estimator.cpp:169-318
  split(SparseSymmetric) -> SplitMatrix
      proj/include/expmc/sparse_matrix.hpp:105, proj/src/sparse_matrix.cpp:101-142

``std::invalid_argument`` maps to ``ValueError`` with the reference's
message; CUDA / runtime failures raise ``ExpmcError``.  ``workers`` is
accepted for signature compatibility and ignored (the GPU decides the
parallelism; results do not depend on it).
"""
from __future__ import annotations

import ctypes as C
import os
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import EstimateC, PathParamsC, check, f64p, lib, u8p, u32p, u64p


class Splitting(enum.IntEnum):
    """estimator.hpp:11"""
    Lie = 0
    Strang = 1


class Rng(enum.IntEnum):
    """Walker engine: PHILOX = production continuous-clock walker (K3/K4);
    PCG_COMPAT = path-by-path replay of the reference PCG32 streams (K2)."""
    PHILOX = 0
    PCG_COMPAT = 1


@dataclass
class PathParams:
    """estimator.hpp:16-33 (same defaults)."""
    beta: float = 1.0
    n_steps: int = 32
    samples: int = 1_000_000
    splitting: Splitting = Splitting.Strang
    seed: int = 0
    rng: Rng = Rng.PHILOX

    def dt(self) -> float:
        return self.beta / float(self.n_steps)

    @staticmethod
    def with_steps(beta, n_steps, samples, s, seed, rng=Rng.PHILOX) -> "PathParams":
        p = PathParams(beta, n_steps, samples, s, seed, rng)
        p.validate()
        return p

    @staticmethod
    def with_dt(beta, dt, samples, s, seed, rng=Rng.PHILOX) -> "PathParams":
        # estimator.cpp:151-159: llround(beta/dt), at least 1
        if not (beta > 0.0) or not (dt > 0.0):
            raise ValueError("beta and dt must be positive")
        q = beta / dt
        n = max(1, int(math.floor(q + 0.5)) if q >= 0 else int(math.ceil(q - 0.5)))
        return PathParams.with_steps(beta, n, samples, s, seed, rng)

    def validate(self) -> None:
        # estimator.cpp:161-167
        if not (self.beta > 0.0) or not math.isfinite(self.beta):
            raise ValueError("beta must be positive and finite")
        if self.n_steps == 0:
            raise ValueError("n_steps must be >= 1")
        if self.samples == 0:
            raise ValueError("samples must be >= 1")

    def _c(self) -> PathParamsC:
        if self.n_steps < 0 or self.samples < 0 or self.seed < 0:
            raise ValueError("n_steps, samples and seed must be non-negative")
        return PathParamsC(float(self.beta), int(self.n_steps), int(self.samples),
                           int(self.splitting), int(self.rng), int(self.seed) & (2**64 - 1))


@dataclass
class Estimate:
    """estimator.hpp:37-42"""
    value: float = 0.0
    std_error: float = 0.0
    samples_used: int = 0
    total_jumps: int = 0


@dataclass
class VectorEstimate:
    """estimator.hpp:46-52"""
    values: np.ndarray = field(default_factory=lambda: np.zeros(0))
    std_error_global: float = 0.0
    samples_used: int = 0
    total_jumps: int = 0
    v_sum: float = 0.0


@dataclass
class EntriesEstimate:
    """Batched entry_estimate over many rows ("full vector with W walkers
    per entry"): per-row value, standard error and jump count.  ``rows`` is
    None for the full vector (row k = entry k)."""
    rows: np.ndarray | None
    values: np.ndarray
    std_errors: np.ndarray
    jumps: np.ndarray
    samples_per_entry: int
    total_jumps: int  # sum of jumps (reduced on the device)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class SplitMatrix:
    """Device-resident SplitMatrix (sparse_matrix.hpp:66-91) on one GPU.

    Built by :func:`split` from the mirrored adjacency of a symmetric matrix;
    immutable afterwards.  ``export()`` copies the reference's fields back to
    host memory (for parity checks)."""

    def __init__(self, handle, csr_n):
        self._h = handle
        n, nnz, dbar, dmax = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_uint64()
        anu, dev = C.c_int32(), C.c_int32()
        check(lib().expmc_cuda_matrix_info(handle, C.byref(n), C.byref(nnz), C.byref(dbar),
                                           C.byref(dmax), C.byref(anu), C.byref(dev)))
        self.n, self.nnz = n.value, nnz.value
        self.dbar, self.dmax = dbar.value, dmax.value
        self.any_nonuniform = bool(anu.value)
        self.device = dev.value

    @classmethod
    def from_csr(cls, n, row_ptr, col, val, diag=None, device=0) -> "SplitMatrix":
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        col = np.ascontiguousarray(col, dtype=np.uint32)
        val = _f64(val)
        diag = None if diag is None else _f64(diag)
        if len(row_ptr) != n + 1:
            raise ValueError("row_ptr must have n + 1 entries")
        h = C.c_void_p()
        check(lib().expmc_cuda_create_from_csr(
            n, row_ptr.ctypes.data_as(u64p), col.ctypes.data_as(u32p),
            val.ctypes.data_as(f64p), None if diag is None else diag.ctypes.data_as(f64p),
            int(device), C.byref(h)))
        return cls(h, n)

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().expmc_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self) -> dict:
        n, nnz = self.n, self.nnz
        s = dict(diag=np.zeros(n), d=np.zeros(n), rate=np.zeros(n),
                 row_offset=np.zeros(n + 1, np.uint64), neighbor=np.zeros(nnz, np.uint32),
                 weight=np.zeros(nnz), cum=np.zeros(nnz), uniform_row=np.zeros(n, np.uint8))
        check(lib().expmc_cuda_split_export(
            self._h, s["diag"].ctypes.data_as(f64p), s["d"].ctypes.data_as(f64p),
            s["rate"].ctypes.data_as(f64p), s["row_offset"].ctypes.data_as(u64p),
            s["neighbor"].ctypes.data_as(u32p), s["weight"].ctypes.data_as(f64p),
            s["cum"].ctypes.data_as(f64p), s["uniform_row"].ctypes.data_as(u8p)))
        s["dbar"], s["dmax"] = self.dbar, self.dmax
        return s

    def alias_tables(self):
        thr = np.zeros(self.nnz, np.uint32)
        al = np.zeros(self.nnz, np.uint32)
        check(lib().expmc_cuda_alias_export(self._h, thr.ctypes.data_as(u32p),
                                            al.ctypes.data_as(u32p)))
        return thr, al

    REC = np.dtype([("off", "<u4"), ("degf", "<u4"), ("inv_rate", "<f4"), ("spare", "<u4"),
                    ("d", "<f8"), ("v", "<f8")])

    def records(self) -> np.ndarray:
        out = np.zeros(self.n, self.REC)
        check(lib().expmc_cuda_records_export(self._h, out.ctypes.data))
        return out


def from_entries(n: int, rows, cols, weights, device=0) -> SplitMatrix:
    """SparseSymmetric::from_entries + split() (sparse_matrix.cpp:18-85,
    :101-142) on the GPU: raw (row, col, weight) entries in either triangle
    and any order; the reference's validation messages and precedence."""
    r = np.ascontiguousarray(rows, dtype=np.uint32)
    c = np.ascontiguousarray(cols, dtype=np.uint32)
    w = _f64(weights)
    if not (len(r) == len(c) == len(w)):
        raise ValueError("rows, cols and weights must have the same length")
    h = C.c_void_p()
    check(lib().expmc_cuda_create_from_entries(int(n), r.ctypes.data_as(u32p),
                                               c.ctypes.data_as(u32p), w.ctypes.data_as(f64p),
                                               len(w), int(device), C.byref(h)))
    return SplitMatrix(h, n)


def from_matrix_market(path, device=0) -> SplitMatrix:
    """load_matrix_market + split() (matrix_market.cpp:51-165,
    sparse_matrix.cpp:101-142): host parse on all cores, general fold,
    from_entries and split on the GPU.  Parse errors raise ExpmcError
    ("path:line: what", the reference's runtime_error); from_entries errors
    raise ValueError."""
    h = C.c_void_p()
    check(lib().expmc_cuda_create_from_mm(os.fsencode(path), int(device), C.byref(h)))
    n = C.c_uint64()
    check(lib().expmc_cuda_matrix_info(h, C.byref(n), None, None, None, None, None))
    return SplitMatrix(h, n.value)


def split(csr, device=0) -> SplitMatrix:
    """split(SparseSymmetric) (sparse_matrix.cpp:101-142), on the GPU.
    ``csr`` has ``n, row_ptr, col, val, diag`` (see :class:`inputs.Csr`)."""
    return SplitMatrix.from_csr(csr.n, csr.row_ptr, csr.col, csr.val, csr.diag, device)


def entry_slots(walkers: int) -> int:
    """Lane slots per entry of the Philox walker (result contract)."""
    return int(lib().expmc_cuda_entry_slots(int(walkers)))


def entry_estimate(m: SplitMatrix, v, i: int, p: PathParams, workers: int = 1) -> Estimate:
    """estimator.cpp:169-206 — entry i of the splitting approximation."""
    v = _f64(v)
    if i < 0 or i >= 2**32:
        raise ValueError("entry index out of range")
    out = EstimateC()
    pc = p._c()
    check(lib().expmc_cuda_entry_estimate(m.handle, v.ctypes.data_as(f64p), len(v), int(i),
                                          C.byref(pc), C.byref(out)))
    return Estimate(out.value, out.std_error, out.samples_used, out.total_jumps)


def entries_estimate(m: SplitMatrix, v, rows, p: PathParams, out=None) -> EntriesEstimate:
    """Batched entry_estimate: rows=None means every row (full vector).
    ``out`` = optional preallocated (values f64, std_errors f64, jumps u64)
    host arrays (e.g. pinned) to write into."""
    v = _f64(v)
    pc = p._c()
    if rows is None:
        nrows = m.n
        rp = None
        rows_arr = None
    else:
        rows_arr = np.asarray(rows)
        if rows_arr.size and (rows_arr.min() < 0 or rows_arr.max() >= 2**32):
            raise ValueError("entry index out of range")
        rows_arr = np.ascontiguousarray(rows_arr, dtype=np.uint32)
        nrows = len(rows_arr)
        rp = rows_arr.ctypes.data_as(u32p)
    if out is None:
        val, se, jm = np.zeros(nrows), np.zeros(nrows), np.zeros(nrows, np.uint64)
    else:
        val, se, jm = out
        if not (len(val) >= nrows and len(se) >= nrows and len(jm) >= nrows
                and val.dtype == np.float64 and se.dtype == np.float64
                and jm.dtype in (np.uint64, np.int64) and val.flags.c_contiguous
                and se.flags.c_contiguous and jm.flags.c_contiguous):
            raise ValueError("out arrays must be contiguous f64/f64/u64 of length >= nrows")
    tot = C.c_uint64()
    check(lib().expmc_cuda_entries(m.handle, v.ctypes.data_as(f64p), len(v), rp, nrows,
                                   C.byref(pc), val.ctypes.data_as(f64p),
                                   se.ctypes.data_as(f64p), jm.ctypes.data_as(u64p),
                                   C.byref(tot)))
    return EntriesEstimate(rows_arr, val, se, jm, p.samples, tot.value)


def entries_estimate_multi(ms, v, rows, p: PathParams, out=None) -> EntriesEstimate:
    """Batched entry_estimate over several replicas (one per GPU, or several
    on one GPU): rows in len(ms) contiguous equal shards, all run
    concurrently (C ABI expmc_cuda_entries_multi).  Bitwise identical to
    :func:`entries_estimate` on one replica."""
    ms = list(ms)
    if not ms:
        raise ValueError("need at least one matrix")
    v = _f64(v)
    pc = p._c()
    n = ms[0].n
    if rows is None:
        nrows, rp, rows_arr = n, None, None
    else:
        rows_arr = np.asarray(rows)
        if rows_arr.size and (rows_arr.min() < 0 or rows_arr.max() >= 2**32):
            raise ValueError("entry index out of range")
        rows_arr = np.ascontiguousarray(rows_arr, dtype=np.uint32)
        nrows, rp = len(rows_arr), rows_arr.ctypes.data_as(u32p)
    if out is None:
        val, se, jm = np.zeros(nrows), np.zeros(nrows), np.zeros(nrows, np.uint64)
    else:
        val, se, jm = out
    hs = (C.c_void_p * len(ms))(*[m.handle for m in ms])
    tot = C.c_uint64()
    check(lib().expmc_cuda_entries_multi(hs, len(ms), v.ctypes.data_as(f64p), len(v), rp, nrows,
                                         C.byref(pc), val.ctypes.data_as(f64p),
                                         se.ctypes.data_as(f64p), jm.ctypes.data_as(u64p),
                                         C.byref(tot)))
    return EntriesEstimate(rows_arr, val, se, jm, p.samples, tot.value)


def set_v_cache(m: SplitMatrix, enable: bool = True) -> None:
    """Reuse the staged v across host entry calls with the same array (call
    :func:`invalidate_v` after changing it in place)."""
    check(lib().expmc_cuda_set_v_cache(m.handle, 1 if enable else 0))


def invalidate_v(m: SplitMatrix) -> None:
    check(lib().expmc_cuda_invalidate_v(m.handle))


def v_stagings(m: SplitMatrix) -> int:
    c = C.c_uint64()
    check(lib().expmc_cuda_v_stagings(m.handle, C.byref(c)))
    return int(c.value)


def vector_estimate(m: SplitMatrix, v, p: PathParams, workers: int = 1) -> VectorEstimate:
    """estimator.cpp:208-278 — Theorem 2 full-vector estimator (v >= 0)."""
    v = _f64(v)
    pc = p._c()
    vals = np.zeros(m.n)
    se, jm, vs = C.c_double(), C.c_uint64(), C.c_double()
    check(lib().expmc_cuda_vector_estimate(m.handle, v.ctypes.data_as(f64p), len(v),
                                           C.byref(pc), vals.ctypes.data_as(f64p),
                                           C.byref(se), C.byref(jm), C.byref(vs)))
    return VectorEstimate(vals, se.value, p.samples, jm.value, vs.value)


def vector_estimate_rows(m: SplitMatrix, v, p: PathParams, row_lo: int, row_hi: int):
    """One row shard of vector_estimate (walkers starting in [row_lo, row_hi)):
    (values / M contribution, Σf, Σf², jumps).  See shard.vector_estimate_sharded."""
    v = _f64(v)
    pc = p._c()
    vals = np.zeros(m.n)
    s1, s2, jm = C.c_double(), C.c_double(), C.c_uint64()
    check(lib().expmc_cuda_vector_estimate_rows(m.handle, v.ctypes.data_as(f64p), len(v),
                                                C.byref(pc), int(row_lo), int(row_hi),
                                                vals.ctypes.data_as(f64p), C.byref(s1),
                                                C.byref(s2), C.byref(jm)))
    return vals, s1.value, s2.value, int(jm.value)


def tc_estimate_rows(m: SplitMatrix, p: PathParams, row_lo: int, row_hi: int):
    """One row shard of tc_estimate: (Σf, Σf², jumps) of its walkers."""
    pc = p._c()
    s1, s2, jm = C.c_double(), C.c_double(), C.c_uint64()
    check(lib().expmc_cuda_tc_estimate_rows(m.handle, C.byref(pc), int(row_lo), int(row_hi),
                                            C.byref(s1), C.byref(s2), C.byref(jm)))
    return s1.value, s2.value, int(jm.value)


def finalize(total: float, total_sq: float, samples: int, jumps: int) -> Estimate:
    """estimator.cpp:76-89: mean, one-pass variance clamped at 0, SE."""
    mm = float(samples)
    value = total / mm
    se = 0.0
    if samples > 1:
        var = max(0.0, (total_sq - total * total / mm) / (mm - 1.0))
        se = math.sqrt(var / mm)
    return Estimate(value, se, int(samples), int(jumps))


def tc_estimate(m: SplitMatrix, p: PathParams, workers: int = 1) -> Estimate:
    """estimator.cpp:280-318 — total communicability (1, e^{βA} 1)."""
    pc = p._c()
    out = EstimateC()
    check(lib().expmc_cuda_tc_estimate(m.handle, C.byref(pc), C.byref(out)))
    return Estimate(out.value, out.std_error, out.samples_used, out.total_jumps)


def expmv(m: SplitMatrix, v, t: float, tol: float = 1e-15) -> np.ndarray:
    """Deterministic fp64 exp(tA)v on the GPU (K5; accuracy reference)."""
    v = _f64(v)
    out = np.zeros(m.n)
    check(lib().expmc_cuda_expmv(m.handle, v.ctypes.data_as(f64p), len(v), float(t),
                                 float(tol), out.ctypes.data_as(f64p)))
    return out


def splitting_product(m: SplitMatrix, v, p: PathParams, tol: float = 1e-15) -> np.ndarray:
    """Deterministic splitting product the estimators sample (K5)."""
    v = _f64(v)
    pc = p._c()
    out = np.zeros(m.n)
    check(lib().expmc_cuda_splitting_product(m.handle, v.ctypes.data_as(f64p), len(v),
                                             C.byref(pc), float(tol),
                                             out.ctypes.data_as(f64p)))
    return out


# ------------------------------------------------- device-resident entry API
def set_v_device(m: SplitMatrix, v_ptr: int, n: int, stream: int = 0) -> None:
    check(lib().expmc_cuda_set_v_device(m.handle, v_ptr, n, stream or None))


def entries_device(m: SplitMatrix, rows_ptr: int, nrows: int, p: PathParams, value_ptr: int,
                   se_ptr: int, jumps_ptr: int, stream: int = 0) -> None:
    """Async Philox entry walker on device buffers (raw device pointers)."""
    pc = p._c()
    check(lib().expmc_cuda_entries_device(m.handle, rows_ptr, nrows, C.byref(pc), value_ptr,
                                          se_ptr, jumps_ptr, stream or None))


def entries_device_range(m: SplitMatrix, row_lo: int, nrows: int, p: PathParams, value_ptr: int,
                         se_ptr: int, jumps_ptr: int, stream: int = 0) -> None:
    """entries_device over the contiguous rows [row_lo, row_lo + nrows): no row
    array on the device; same results bit for bit."""
    pc = p._c()
    check(lib().expmc_cuda_entries_device_range(m.handle, int(row_lo), int(nrows), C.byref(pc),
                                                value_ptr, se_ptr, jumps_ptr, stream or None))


def gather_ceiling_device(m: SplitMatrix, rows_ptr: int, nrows: int, chains_per_row: int,
                          chain_len: int, stream: int = 0) -> None:
    check(lib().expmc_cuda_gather_ceiling_device(m.handle, rows_ptr, nrows,
                                                 int(chains_per_row), int(chain_len),
                                                 stream or None))


def exp_law(count: int, seed: int = 0, bin_width: float = 0.05, nbins: int = 512, device=0):
    """Test hook: histogram + moments of `count` draws of the walkers' Exp(1)
    transform (neg_ln_u over Philox words)."""
    hist = np.zeros(int(nbins), np.uint64)
    mom = np.zeros(2)
    check(lib().expmc_cuda_exp_law(int(device), int(count), int(seed), float(bin_width),
                                   int(nbins), hist.ctypes.data_as(u64p),
                                   mom.ctypes.data_as(f64p)))
    return hist, mom


def last_k4_stats(m: SplitMatrix):
    """(jumpers, fixed_point) of the last vector / tc call on m: walks K4
    actually ran, and whether vector_estimate's per-end sums used the exact
    128-bit fixed point (1), the sort-based reduction (0) or none yet (-1)."""
    j, fx = C.c_uint64(), C.c_int()
    check(lib().expmc_cuda_last_k4_stats(m.handle, C.byref(j), C.byref(fx)))
    return int(j.value), int(fx.value)


def last_jumpers(m: SplitMatrix) -> int:
    """Walks K4 actually ran (walkers with >= 1 jump) in the last vector / tc call."""
    return last_k4_stats(m)[0]


def binomial_samples(trials: int, p: float, count: int, seed: int = 0,
                     device: int = 0) -> np.ndarray:
    """`count` draws of K4's device Binomial(trials, p) sampler (test hook)."""
    out = np.zeros(int(count), dtype=np.uint64)
    check(lib().expmc_cuda_binomial_samples(int(device), int(trials), float(p), int(count),
                                            int(seed), out.ctypes.data_as(u64p)))
    return out


def start_counts(m: SplitMatrix, v, samples: int, seed: int) -> np.ndarray:
    """K4's walkers per start row ~ Multinomial(samples, v / V) (v None: uniform),
    the draw vector_estimate / tc_estimate make for (samples, seed)."""
    out = np.zeros(m.n, dtype=np.uint64)
    if v is None:
        vp_, nv = None, 0
    else:
        v = _f64(v)
        vp_, nv = v.ctypes.data_as(f64p), len(v)
    check(lib().expmc_cuda_start_counts(m.handle, vp_, nv, int(samples), int(seed),
                                        out.ctypes.data_as(u64p)))
    return out


def launch_count() -> int:
    return int(lib().expmc_cuda_launch_count())
