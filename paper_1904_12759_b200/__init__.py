"""paper_1904_12759_b200 — B200-native Monte Carlo exp(tA)v hot path.

The reference's estimator API (arXiv 1904.12759 C++ artifact,
/root/reference/proj/include/expmc/estimator.hpp) over a C ABI
(include/expmc_b200.h) implemented by hand-written sm_100a kernels in
``csrc/``.  There is no CPU fallback: every estimate runs on the GPU.
"""
from ._lib import ExpmcError, lib
from .estimator import (EntriesEstimate, binomial_samples, last_jumpers, last_k4_stats, start_counts, tc_estimate_rows,
                        vector_estimate_rows, finalize, Estimate, PathParams, Rng, SplitMatrix, Splitting,
                        VectorEstimate, entries_device, entries_device_range, entries_estimate, entries_estimate_multi, entry_estimate,
                        invalidate_v, set_v_cache, v_stagings, exp_law,
                        entry_slots, expmv, from_entries, from_matrix_market, gather_ceiling_device, launch_count, set_v_device,
                        split, splitting_product, tc_estimate, vector_estimate)
from .inputs import (Csr, MmEntries, build_config, csr_from_dense, gen_ba, gen_fd, gen_row_sample,
                     gen_vector, gen_ws, load_csr, load_matrix_market, n_rule, parse_matrix_market,
                     save_csr, write_matrix_market)
from .spectral import BetaRule, lambda_max, resolve_beta

__all__ = [
    "ExpmcError", "lib", "binomial_samples", "last_jumpers", "last_k4_stats", "start_counts", "tc_estimate_rows",
    "vector_estimate_rows", "finalize", "EntriesEstimate", "Estimate", "PathParams", "Rng", "SplitMatrix",
    "Splitting", "VectorEstimate", "entries_device", "entries_device_range", "entries_estimate", "entries_estimate_multi",
    "entry_estimate", "invalidate_v", "set_v_cache", "v_stagings", "exp_law",
    "entry_slots", "expmv", "gather_ceiling_device", "launch_count", "set_v_device", "split",
    "splitting_product", "tc_estimate", "vector_estimate", "Csr", "build_config",
    "csr_from_dense", "gen_ba", "gen_fd", "gen_row_sample", "gen_vector", "gen_ws", "n_rule",
    "BetaRule", "lambda_max", "resolve_beta", "from_matrix_market", "MmEntries", "load_csr",
    "load_matrix_market", "parse_matrix_market", "save_csr", "write_matrix_market",
]
