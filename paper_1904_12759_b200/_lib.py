"""Loader for the in-tree product library ``libexpmc_b200.so`` (C ABI:
``include/expmc_b200.h``).  There is no fallback: if the library is missing
the import fails loudly."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# EXPMC_B200_LIB selects an alternative build of the same library (tuning
# variants under paper_1904_12759_b200/variants/); default is the in-tree .so.
LIB_PATH = os.environ.get("EXPMC_B200_LIB") or os.path.join(HERE, "libexpmc_b200.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p


class PathParamsC(C.Structure):
    """expmc_path_params."""
    _fields_ = [("beta", C.c_double), ("n_steps", C.c_uint64), ("samples", C.c_uint64),
                ("splitting", C.c_int32), ("rng", C.c_int32), ("seed", C.c_uint64)]


class EstimateC(C.Structure):
    """expmc_estimate."""
    _fields_ = [("value", C.c_double), ("std_error", C.c_double),
                ("samples_used", C.c_uint64), ("total_jumps", C.c_uint64)]


# (name, restype, argtypes) for every exported symbol of include/expmc_b200.h
SIGNATURES = [
    ("expmc_cuda_last_error", C.c_char_p, []),
    ("expmc_cuda_abi_version", C.c_int, []),
    ("expmc_cuda_create_from_csr", C.c_int,
     [C.c_uint64, u64p, u32p, f64p, f64p, C.c_int, C.POINTER(vp)]),
    ("expmc_cuda_rank", C.c_int, [f64p, C.c_uint64, C.c_int, u32p]),
    ("expmc_cuda_isim", C.c_int,
     [u32p, u32p, C.c_uint64, C.c_uint64, C.c_double, C.c_int, f64p]),
    ("expmc_cuda_create_from_entries", C.c_int,
     [C.c_uint64, u32p, u32p, f64p, C.c_uint64, C.c_int, C.POINTER(vp)]),
    ("expmc_cuda_create_from_split", C.c_int,
     [C.c_uint64, u64p, u32p, f64p, f64p, C.c_int, C.POINTER(vp)]),
    ("expmc_cuda_create_from_mm", C.c_int, [C.c_char_p, C.c_int, C.POINTER(vp)]),
    ("expmc_cuda_destroy", C.c_int, [vp]),
    ("expmc_cuda_matrix_info", C.c_int,
     [vp, u64p, u64p, f64p, u64p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("expmc_cuda_split_export", C.c_int, [vp, f64p, f64p, f64p, u64p, u32p, f64p, f64p, u8p]),
    ("expmc_cuda_alias_export", C.c_int, [vp, u32p, u32p]),
    ("expmc_cuda_records_export", C.c_int, [vp, vp]),
    ("expmc_cuda_entry_estimate", C.c_int,
     [vp, f64p, C.c_uint64, C.c_uint32, C.POINTER(PathParamsC), C.POINTER(EstimateC)]),
    ("expmc_cuda_entries", C.c_int,
     [vp, f64p, C.c_uint64, u32p, C.c_uint64, C.POINTER(PathParamsC), f64p, f64p, u64p, u64p]),
    ("expmc_cuda_entries_multi", C.c_int,
     [C.POINTER(vp), C.c_int, f64p, C.c_uint64, u32p, C.c_uint64, C.POINTER(PathParamsC), f64p,
      f64p, u64p, u64p]),
    ("expmc_cuda_exp_law", C.c_int,
     [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_uint32, u64p, f64p]),
    ("expmc_cuda_set_v_cache", C.c_int, [vp, C.c_int]),
    ("expmc_cuda_invalidate_v", C.c_int, [vp]),
    ("expmc_cuda_v_stagings", C.c_int, [vp, u64p]),
    ("expmc_cuda_vector_estimate", C.c_int,
     [vp, f64p, C.c_uint64, C.POINTER(PathParamsC), f64p, f64p, u64p, f64p]),
    ("expmc_cuda_tc_estimate", C.c_int, [vp, C.POINTER(PathParamsC), C.POINTER(EstimateC)]),
    ("expmc_cuda_vector_estimate_rows", C.c_int,
     [vp, f64p, C.c_uint64, C.POINTER(PathParamsC), C.c_uint64, C.c_uint64, f64p, f64p, f64p,
      u64p]),
    ("expmc_cuda_tc_estimate_rows", C.c_int,
     [vp, C.POINTER(PathParamsC), C.c_uint64, C.c_uint64, f64p, f64p, u64p]),
    ("expmc_cuda_set_v_device", C.c_int, [vp, vp, C.c_uint64, vp]),
    ("expmc_cuda_entries_device", C.c_int,
     [vp, vp, C.c_uint64, C.POINTER(PathParamsC), vp, vp, vp, vp]),
    ("expmc_cuda_entries_device_range", C.c_int,
     [vp, C.c_uint64, C.c_uint64, C.POINTER(PathParamsC), vp, vp, vp, vp]),
    ("expmc_cuda_gather_ceiling_device", C.c_int,
     [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, vp]),
    ("expmc_cuda_entry_slots", C.c_uint32, [C.c_uint64]),
    ("expmc_cuda_last_k4_stats", C.c_int, [vp, u64p, C.POINTER(C.c_int)]),
    ("expmc_cuda_binomial_samples", C.c_int,
     [C.c_int, C.c_uint64, C.c_double, C.c_uint64, C.c_uint64, u64p]),
    ("expmc_cuda_start_counts", C.c_int, [vp, f64p, C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
    ("expmc_cuda_launch_count", C.c_uint64, []),
    ("expmc_cuda_expmv", C.c_int, [vp, f64p, C.c_uint64, C.c_double, C.c_double, f64p]),
    ("expmc_cuda_lambda_max", C.c_int, [vp, C.c_uint64, f64p, f64p]),
    ("expmc_cuda_splitting_product", C.c_int,
     [vp, f64p, C.c_uint64, C.POINTER(PathParamsC), C.c_double, f64p]),
    ("expmc_gen_last_error", C.c_char_p, []),
    ("expmc_gen_fd", C.c_int, [C.c_int, C.c_uint64, C.c_double, C.POINTER(vp)]),
    ("expmc_gen_ba", C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(vp)]),
    ("expmc_gen_ws", C.c_int, [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.POINTER(vp)]),
    ("expmc_csr_sizes", C.c_int, [vp, u64p, u64p]),
    ("expmc_csr_export", C.c_int, [vp, u64p, u32p, f64p, f64p]),
    ("expmc_csr_view", C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    ("expmc_csr_free", None, [vp]),
    ("expmc_cuda_mm_load", C.c_int, [C.c_char_p, C.c_int, C.POINTER(vp)]),
    ("expmc_mm_parse", C.c_int, [C.c_char_p, C.POINTER(vp)]),
    ("expmc_mm_info", C.c_int,
     [vp, u64p, u64p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), u64p]),
    ("expmc_mm_view", C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    ("expmc_mm_free", None, [vp]),
    ("expmc_mm_write", C.c_int, [C.c_char_p, C.c_uint64, u64p, u32p, f64p, f64p]),
    ("expmc_csr_save", C.c_int, [C.c_char_p, C.c_uint64, u64p, u32p, f64p, f64p]),
    ("expmc_csr_load", C.c_int, [C.c_char_p, C.POINTER(vp)]),
    ("expmc_gen_vector", C.c_int,
     [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, f64p]),
    ("expmc_gen_row_sample", C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, u32p]),
]

_lib = None


def lib():
    """The loaded product library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_1904_12759_b200` or "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class ExpmcError(RuntimeError):
    """CUDA / runtime failure inside the library (reference: runtime_error)."""


def check(rc, gen=False):
    if rc == 0:
        return
    L = lib()
    msg = (L.expmc_gen_last_error() if gen else L.expmc_cuda_last_error()).decode()
    if rc == 1:  # EXPMC_INVALID_ARGUMENT  (reference: std::invalid_argument)
        raise ValueError(msg)
    raise ExpmcError(msg)
