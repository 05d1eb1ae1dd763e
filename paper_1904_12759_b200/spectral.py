"""stats() / resolve_beta() on the GPU.

Reference: ``stats`` (proj/src/sparse_matrix.cpp:176-217) estimates the
largest eigenvalue of A by power iteration on A shifted by its Gershgorin
lower bound; ``resolve_beta`` (proj/src/metrics.cpp:69-91) turns it into
the inverse temperature (config 2 uses beta = 0.5 / lambda_max).
"""
from __future__ import annotations

import ctypes as C
import enum

from ._lib import check, lib


def lambda_max(m, power_iters: int = 100):
    """Largest eigenvalue estimate of A after ``power_iters`` iterations."""
    lam, rel = C.c_double(), C.c_double()
    check(lib().expmc_cuda_lambda_max(m.handle, int(power_iters), C.byref(lam), C.byref(rel)))
    return lam.value


class BetaRule(enum.Enum):
    """metrics.hpp:31-41"""
    Fixed = 0
    InverseLambdaMax = 1
    InverseDmax = 2


def resolve_beta(rule: BetaRule, m=None, fixed_beta: float = 1.0, power_iters: int = 100,
                 lam=None) -> float:
    """metrics.cpp:69-91 with the same error messages."""
    if rule == BetaRule.Fixed:
        if not (fixed_beta > 0.0):
            raise ValueError("BetaRule: fixed beta must be positive")
        return fixed_beta
    if rule == BetaRule.InverseLambdaMax:
        if lam is None:
            if m is None:
                raise ValueError("resolve_beta: lambda_max has not been estimated")
            lam = lambda_max(m, power_iters)
        if not (lam > 0.0):
            raise ValueError("resolve_beta: lambda_max must be positive")
        return 1.0 / lam
    if m is None or m.dmax == 0:
        raise ValueError("resolve_beta: graph has no edges, d_max = 0")
    return 1.0 / float(m.dmax)
