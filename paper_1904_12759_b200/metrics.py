"""Ranking metrics on the GPU (§8f row f4): rank / isim of the reference
(/root/reference/proj/src/metrics.cpp:10-55), same semantics and messages.
normalized_tc (metrics.cpp:57-60) is trivial host arithmetic."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, f64p, lib, u32p


def rank(values, device: int = 0) -> np.ndarray:
    """Node ids by descending score, ties by ascending id (NaN rejected)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.zeros(len(v), np.uint32)
    check(lib().expmc_cuda_rank(v.ctypes.data_as(f64p), len(v), int(device),
                                out.ctypes.data_as(u32p)))
    return out


def isim(order_x, order_y, top_fraction: float, device: int = 0) -> float:
    """Intersection similarity of the top ceil(top_fraction * n) prefixes."""
    ox = np.ascontiguousarray(order_x, dtype=np.uint32)
    oy = np.ascontiguousarray(order_y, dtype=np.uint32)
    out = C.c_double()
    check(lib().expmc_cuda_isim(ox.ctypes.data_as(u32p), oy.ctypes.data_as(u32p), len(ox),
                                len(oy), float(top_fraction), int(device), C.byref(out)))
    return out.value


def normalized_tc(tc: float, n: int) -> float:
    if n < 1:
        raise ValueError("normalized_tc: n must be >= 1")
    return tc / float(n)
