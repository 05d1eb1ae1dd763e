"""TEST INFRASTRUCTURE ONLY — the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_1904_12759_b200``) never does and has no CPU fallback.

Two libraries, both built by ``make -C oracle`` (``__graft_entry__.build()``):

* ``liboracle.so`` — a plain-C restatement of the reference hot path
  (``oracle/expmc_oracle.c``; each function cites the reference file:line),
  the alias-table contract of the B200 build, and a CPU model of the Philox
  walker (``oracle/fast_model.c``).
* ``_ref/libexpmc_ref.so`` — the UNMODIFIED reference library compiled from
  ``/root/reference/proj/src`` (6 of 7 translation units; ``oracle.cpp``
  needs the absent Eigen3) plus the extern-"C" shim ``oracle/ref_shim.cpp``.

Parity pinning: tests/test_oracle.py checks the restatement against the
public pcg32 sequence, the SURVEY §8a golden values and the committed
fixtures under tests/golden/ (generated from ``_ref`` by
tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _load(path):
    if not os.path.exists(path):
        raise RuntimeError(f"oracle library missing: {path} (run `make -C oracle`)")
    return C.CDLL(path)


_MM_WRITE_CHILD = r"""
import array, ctypes as C, sys
L = C.CDLL(sys.argv[1])
L.ref_from_entries.restype = C.c_void_p
L.ref_from_entries.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]
L.ref_mm_write.argtypes = [C.c_void_p, C.c_char_p]
L.ref_last_error.restype = C.c_char_p
raw = open(sys.argv[2], "rb").read()
hdr = array.array("Q"); hdr.frombytes(raw[:16]); n, ne = hdr
o = 16
r = array.array("I"); r.frombytes(raw[o:o + 4 * ne]); o += 4 * ne
c = array.array("I"); c.frombytes(raw[o:o + 4 * ne]); o += 4 * ne
w = array.array("d"); w.frombytes(raw[o:o + 8 * ne])
buf = lambda a: (C.c_char * max(1, len(a) * a.itemsize)).from_buffer_copy(a.tobytes() or b"\0")
h = L.ref_from_entries(n, buf(r), buf(c), buf(w), ne)
if not h:
    sys.exit(L.ref_last_error().decode())
if L.ref_mm_write(h, sys.argv[3].encode()) != 0:
    sys.exit(L.ref_last_error().decode())
"""


# ----------------------------------------------------------------- C oracle
class Oracle:
    """ctypes view of liboracle.so."""

    def __init__(self):
        L = _load(os.environ.get("EXPMC_ORACLE_LIB") or os.path.join(HERE, "liboracle.so"))
        self.L = L
        L.orc_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p]
        L.orc_split.argtypes = [C.c_uint64, _u64p, _u32p, _f64p, _f64p, _f64p, _f64p, _f64p,
                                _f64p, _u8p, _f64p, _u64p]
        L.orc_entry_estimate.argtypes = [C.c_void_p, _f64p, C.c_uint32, C.c_double, C.c_uint64,
                                         C.c_uint64, C.c_int, C.c_uint64, _f64p, _f64p, _u64p]
        L.orc_vector_estimate.argtypes = [C.c_void_p, _f64p, C.c_double, C.c_uint64, C.c_uint64,
                                          C.c_int, C.c_uint64, _f64p, _f64p, _u64p, _f64p]
        L.orc_tc_estimate.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_uint64, C.c_int,
                                      C.c_uint64, _f64p, _f64p, _u64p]
        L.orc_advance_many.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_double,
                                       C.c_uint64, _u32p, _u64p]
        L.orc_exp_times.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, _f64p]
        L.orc_alias_build.argtypes = [C.c_uint64, _u64p, _f64p, _f64p, _u8p, _u32p, _u32p]
        L.fm_philox.argtypes = [_u32p, C.c_uint32, C.c_uint32, _u32p]
        L.fm_neg_ln_u.argtypes = [C.c_uint32]
        L.fm_neg_ln_u.restype = C.c_float
        L.fm_build_records.argtypes = [C.c_uint64, _u64p, _f64p, _f64p, _u8p, _f64p, C.c_void_p]
        L.fm_entries.argtypes = [C.c_void_p, _f64p, _u32p, _u32p, _u32p, _u32p, C.c_uint64,
                                 C.c_double, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64,
                                 C.c_uint32, _f64p, _f64p, _u64p]

    # RNG ------------------------------------------------------------------
    def rng_draws(self, seed, stream, op, count, arg=0):
        dt = {0: np.uint32, 1: np.uint64, 2: np.float64, 3: np.float64, 4: np.uint64}[op]
        out = np.zeros(count, dtype=dt)
        self.L.orc_rng_draws(seed, stream, op, arg, count, out.ctypes.data)
        return out

    def exp_times(self, seed, stream, rate, count):
        out = np.zeros(count)
        self.L.orc_exp_times(seed, stream, rate, count, _p(out, _f64p))
        return out

    # split ----------------------------------------------------------------
    def split(self, csr):
        """split() restated (sparse_matrix.cpp:101-142) -> dict of arrays."""
        n = csr.n
        nnz = int(csr.row_ptr[-1]) if n else 0
        out = dict(diag=np.zeros(n), d=np.zeros(n), rate=np.zeros(n), cum=np.zeros(nnz),
                   uniform_row=np.zeros(n, np.uint8))
        dbar = C.c_double()
        dmax = C.c_uint64()
        self.L.orc_split(n, _p(csr.row_ptr, _u64p), _p(csr.col, _u32p), _p(csr.val, _f64p),
                         _p(csr.diag, _f64p), _p(out["diag"], _f64p), _p(out["d"], _f64p),
                         _p(out["rate"], _f64p), _p(out["cum"], _f64p),
                         _p(out["uniform_row"], _u8p), C.byref(dbar), C.byref(dmax))
        out.update(row_offset=csr.row_ptr.copy(), neighbor=csr.col.copy(),
                   weight=csr.val.copy(), dbar=dbar.value, dmax=dmax.value)
        return out

    class _SplitView(C.Structure):
        _fields_ = [("n", C.c_uint64), ("nnz", C.c_uint64), ("diag", _f64p), ("d", _f64p),
                    ("rate", _f64p), ("row_offset", _u64p), ("neighbor", _u32p),
                    ("cum", _f64p), ("uniform_row", _u8p)]

    def _view(self, s):
        v = self._SplitView(len(s["d"]), len(s["neighbor"]), _p(s["diag"], _f64p),
                            _p(s["d"], _f64p), _p(s["rate"], _f64p),
                            _p(s["row_offset"], _u64p), _p(s["neighbor"], _u32p),
                            _p(s["cum"], _f64p), _p(s["uniform_row"], _u8p))
        return v

    def entry_estimate(self, s, v, i, beta, n_steps, samples, splitting=1, seed=0):
        v = np.ascontiguousarray(v, dtype=np.float64)
        val, se, j = C.c_double(), C.c_double(), C.c_uint64()
        self.L.orc_entry_estimate(C.byref(self._view(s)), _p(v, _f64p), i, beta, n_steps,
                                  samples, splitting, seed, C.byref(val), C.byref(se),
                                  C.byref(j))
        return val.value, se.value, j.value

    def vector_estimate(self, s, v, beta, n_steps, samples, splitting=1, seed=0):
        v = np.ascontiguousarray(v, dtype=np.float64)
        vals = np.zeros(len(v))
        se, j, vs = C.c_double(), C.c_uint64(), C.c_double()
        self.L.orc_vector_estimate(C.byref(self._view(s)), _p(v, _f64p), beta, n_steps,
                                   samples, splitting, seed, _p(vals, _f64p), C.byref(se),
                                   C.byref(j), C.byref(vs))
        return vals, se.value, j.value, vs.value

    def tc_estimate(self, s, beta, n_steps, samples, splitting=1, seed=0):
        val, se, j = C.c_double(), C.c_double(), C.c_uint64()
        self.L.orc_tc_estimate(C.byref(self._view(s)), beta, n_steps, samples, splitting,
                               seed, C.byref(val), C.byref(se), C.byref(j))
        return val.value, se.value, j.value

    def advance_many(self, s, seed, start, dt, count):
        end = np.zeros(count, np.uint32)
        jumps = np.zeros(count, np.uint64)
        self.L.orc_advance_many(C.byref(self._view(s)), seed, start, dt, count,
                                _p(end, _u32p), _p(jumps, _u64p))
        return end, jumps

    def alias_build(self, s):
        nnz = len(s["neighbor"])
        thr = np.zeros(nnz, np.uint32)
        al = np.zeros(nnz, np.uint32)
        self.L.orc_alias_build(len(s["d"]), _p(s["row_offset"], _u64p), _p(s["weight"], _f64p),
                               _p(s["rate"], _f64p), _p(s["uniform_row"], _u8p),
                               _p(thr, _u32p), _p(al, _u32p))
        return thr, al

    # CPU model of the Philox walker (K3) ----------------------------------
    def philox(self, ctr, key):
        c = np.asarray(ctr, dtype=np.uint32)
        out = np.zeros(4, np.uint32)
        self.L.fm_philox(_p(c, _u32p), int(key[0]), int(key[1]), _p(out, _u32p))
        return out

    def neg_ln_u(self, w):
        return self.L.fm_neg_ln_u(int(w))

    REC = np.dtype([("off", "<u4"), ("degf", "<u4"), ("inv_rate", "<f4"), ("spare", "<u4"),
                    ("d", "<f8"), ("v", "<f8")])

    def fast_entries(self, s, v, rows, beta, n_steps, samples, splitting, seed, slots,
                     alias=None):
        n = len(s["d"])
        v = np.ascontiguousarray(v, dtype=np.float64)
        rec = np.zeros(n, self.REC)
        self.L.fm_build_records(n, _p(s["row_offset"], _u64p), _p(s["rate"], _f64p),
                                _p(s["d"], _f64p), _p(s["uniform_row"], _u8p), _p(v, _f64p),
                                rec.ctypes.data)
        if alias is None:
            alias = self.alias_build(s)
        thr, al = alias
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        m = len(rows)
        val, se, j = np.zeros(m), np.zeros(m), np.zeros(m, np.uint64)
        self.L.fm_entries(rec.ctypes.data, _p(s["rate"], _f64p), _p(s["neighbor"], _u32p),
                          _p(thr, _u32p), _p(al, _u32p), _p(rows, _u32p), m, beta, n_steps,
                          samples, splitting, seed, slots, _p(val, _f64p), _p(se, _f64p),
                          _p(j, _u64p))
        return val, se, j


# ------------------------------------------------------- compiled reference
class RefError(ValueError):
    pass


class Ref:
    """ctypes view of oracle/_ref/libexpmc_ref.so (the unmodified reference)."""

    def __init__(self):
        L = _load(os.path.join(HERE, "_ref", "libexpmc_ref.so"))
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_from_entries.restype = C.c_void_p
        L.ref_from_entries.argtypes = [C.c_uint64, _u32p, _u32p, _f64p, C.c_uint64]
        L.ref_from_csr.restype = C.c_void_p
        L.ref_from_csr.argtypes = [C.c_uint64, _u64p, _u32p, _f64p, _f64p]
        L.ref_generate.restype = C.c_void_p
        L.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                   C.c_double, C.c_uint64]
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_mm_load.restype = C.c_void_p
        L.ref_mm_load.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.ref_mm_write.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_sizes.argtypes = [C.c_void_p, _u64p, _u64p]
        L.ref_split_export.argtypes = [C.c_void_p, _f64p, _f64p, _f64p, _u64p, _u32p, _f64p,
                                       _f64p, _u8p, _f64p, _u64p]
        L.ref_lambda_max.restype = C.c_double
        L.ref_lambda_max.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_entry_estimate.argtypes = [C.c_void_p, _f64p, C.c_uint64, C.c_uint64, C.c_double,
                                         C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint,
                                         _f64p, _f64p, _u64p]
        L.ref_entries.argtypes = [C.c_void_p, _f64p, C.c_uint64, _u64p, C.c_uint64, C.c_double,
                                  C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint,
                                  C.c_uint, _f64p, _f64p, _u64p]
        L.ref_vector_estimate.argtypes = [C.c_void_p, _f64p, C.c_uint64, C.c_double, C.c_uint64,
                                          C.c_uint64, C.c_int, C.c_uint64, C.c_uint, _f64p,
                                          _f64p, _u64p, _f64p]
        L.ref_tc_estimate.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_uint64, C.c_int,
                                      C.c_uint64, C.c_uint, _f64p, _f64p, _u64p]
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                    C.c_void_p]
        L.ref_exp_times.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, _f64p]
        L.ref_advance.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                  _u32p, _u64p]
        L.ref_rank.argtypes = [_f64p, C.c_uint64, _u32p]
        L.ref_isim.argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, C.c_double, _f64p]

    def rank(self, values):
        v = np.ascontiguousarray(values, np.float64)
        out = np.zeros(len(v), np.uint32)
        self._chk(self.L.ref_rank(_p(v, _f64p), len(v), _p(out, _u32p)))
        return out

    def isim(self, ox, oy, top_fraction):
        ox = np.ascontiguousarray(ox, np.uint32)
        oy = np.ascontiguousarray(oy, np.uint32)
        out = C.c_double()
        self._chk(self.L.ref_isim(_p(ox, _u32p), _p(oy, _u32p), len(ox), len(oy), top_fraction,
                                  C.byref(out)))
        return out.value

    def _chk(self, rc):
        if rc != 0:
            raise RefError(self.L.ref_last_error().decode())

    def matrix_from_csr(self, csr):
        h = self.L.ref_from_csr(csr.n, _p(csr.row_ptr, _u64p), _p(csr.col, _u32p),
                                _p(csr.val, _f64p), _p(csr.diag, _f64p))
        if not h:
            raise RefError(self.L.ref_last_error().decode())
        return RefMatrix(self, h)

    def matrix_from_entries(self, n, rows, cols, w):
        rows = np.ascontiguousarray(rows, np.uint32)
        cols = np.ascontiguousarray(cols, np.uint32)
        w = np.ascontiguousarray(w, np.float64)
        h = self.L.ref_from_entries(n, _p(rows, _u32p), _p(cols, _u32p), _p(w, _f64p), len(w))
        if not h:
            raise RefError(self.L.ref_last_error().decode())
        return RefMatrix(self, h)

    def mm_load(self, path):
        """load_matrix_market; raises RefError with .kind 1 (invalid_argument)
        or 2 (runtime_error)."""
        st = C.c_int()
        h = self.L.ref_mm_load(os.fsencode(path), C.byref(st))
        if not h:
            e = RefError(self.L.ref_last_error().decode())
            e.kind = st.value
            raise e
        return RefMatrix(self, h)

    def mm_write_entries(self, n, rows, cols, w, path):
        """write_matrix_market of from_entries(n, entries), run in a child
        interpreter without numpy: the reference's std::ofstream writer
        crashes inside a process that has numpy's C++ runtime loaded first
        (observed here), so the child loads only ctypes."""
        import subprocess
        import sys
        import tempfile

        with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as f:
            np.array([n, len(w)], np.uint64).tofile(f)
            np.ascontiguousarray(rows, np.uint32).tofile(f)
            np.ascontiguousarray(cols, np.uint32).tofile(f)
            np.ascontiguousarray(w, np.float64).tofile(f)
            tmp = f.name
        try:
            r = subprocess.run([sys.executable, "-c", _MM_WRITE_CHILD,
                                os.path.join(HERE, "_ref", "libexpmc_ref.so"), tmp,
                                os.fspath(path)], capture_output=True, text=True)
        finally:
            os.unlink(tmp)
        if r.returncode != 0:
            raise RefError(r.stderr.strip() or f"writer exited {r.returncode}")

    def generate(self, kind, n, k=1, ps=0.0, m0=2, p=0.0, seed=0):
        h = self.L.ref_generate(kind, n, k, ps, m0, p, seed)
        if not h:
            raise RefError(self.L.ref_last_error().decode())
        return RefMatrix(self, h)

    def rng_draws(self, seed, stream, op, count, arg=0):
        dt = {0: np.uint32, 1: np.uint64, 2: np.float64, 3: np.float64, 4: np.uint64}[op]
        out = np.zeros(count, dtype=dt)
        self.L.ref_rng_draws(seed, stream, op, arg, count, out.ctypes.data)
        return out

    def exp_times(self, seed, stream, rate, count):
        out = np.zeros(count)
        self._chk(self.L.ref_exp_times(seed, stream, rate, count, _p(out, _f64p)))
        return out


class RefMatrix:
    def __init__(self, ref, h):
        self.ref, self.h = ref, h
        n, nnz = C.c_uint64(), C.c_uint64()
        ref.L.ref_sizes(h, C.byref(n), C.byref(nnz))
        self.n, self.nnz = n.value, nnz.value

    def __del__(self):
        try:
            self.ref.L.ref_destroy(self.h)
        except Exception:
            pass

    def split(self):
        n, nnz = self.n, self.nnz
        s = dict(diag=np.zeros(n), d=np.zeros(n), rate=np.zeros(n),
                 row_offset=np.zeros(n + 1, np.uint64), neighbor=np.zeros(nnz, np.uint32),
                 weight=np.zeros(nnz), cum=np.zeros(nnz), uniform_row=np.zeros(n, np.uint8))
        dbar, dmax = C.c_double(), C.c_uint64()
        self.ref.L.ref_split_export(self.h, _p(s["diag"], _f64p), _p(s["d"], _f64p),
                                    _p(s["rate"], _f64p), _p(s["row_offset"], _u64p),
                                    _p(s["neighbor"], _u32p), _p(s["weight"], _f64p),
                                    _p(s["cum"], _f64p), _p(s["uniform_row"], _u8p),
                                    C.byref(dbar), C.byref(dmax))
        s["dbar"], s["dmax"] = dbar.value, dmax.value
        return s

    def lambda_max(self, iters):
        return self.ref.L.ref_lambda_max(self.h, iters)

    def entry_estimate(self, v, i, beta, n_steps, samples, splitting=1, seed=0, workers=1):
        v = np.ascontiguousarray(v, np.float64)
        val, se, j = C.c_double(), C.c_double(), C.c_uint64()
        self.ref._chk(self.ref.L.ref_entry_estimate(self.h, _p(v, _f64p), len(v), i, beta,
                                                    n_steps, samples, splitting, seed, workers,
                                                    C.byref(val), C.byref(se), C.byref(j)))
        return val.value, se.value, j.value

    def entries(self, v, rows, beta, n_steps, samples, splitting=1, seed=0, workers=1,
                threads=1):
        v = np.ascontiguousarray(v, np.float64)
        rows = np.ascontiguousarray(rows, np.uint64)
        m = len(rows)
        val, se, j = np.zeros(m), np.zeros(m), np.zeros(m, np.uint64)
        self.ref._chk(self.ref.L.ref_entries(self.h, _p(v, _f64p), len(v), _p(rows, _u64p), m,
                                             beta, n_steps, samples, splitting, seed, workers,
                                             threads, _p(val, _f64p), _p(se, _f64p),
                                             _p(j, _u64p)))
        return val, se, j

    def vector_estimate(self, v, beta, n_steps, samples, splitting=1, seed=0, workers=1):
        v = np.ascontiguousarray(v, np.float64)
        vals = np.zeros(self.n)
        se, j, vs = C.c_double(), C.c_uint64(), C.c_double()
        self.ref._chk(self.ref.L.ref_vector_estimate(self.h, _p(v, _f64p), len(v), beta,
                                                     n_steps, samples, splitting, seed, workers,
                                                     _p(vals, _f64p), C.byref(se), C.byref(j),
                                                     C.byref(vs)))
        return vals, se.value, j.value, vs.value

    def tc_estimate(self, beta, n_steps, samples, splitting=1, seed=0, workers=1):
        val, se, j = C.c_double(), C.c_double(), C.c_uint64()
        self.ref._chk(self.ref.L.ref_tc_estimate(self.h, beta, n_steps, samples, splitting,
                                                 seed, workers, C.byref(val), C.byref(se),
                                                 C.byref(j)))
        return val.value, se.value, j.value

    def advance_many(self, seed, start, dt, count):
        end = np.zeros(count, np.uint32)
        jumps = np.zeros(count, np.uint64)
        self.ref._chk(self.ref.L.ref_advance(self.h, seed, start, dt, count, _p(end, _u32p),
                                             _p(jumps, _u64p)))
        return end, jumps


def oracle():
    return Oracle()


def ref_available():
    return os.path.exists(os.path.join(HERE, "_ref", "libexpmc_ref.so"))


def ref():
    return Ref()
