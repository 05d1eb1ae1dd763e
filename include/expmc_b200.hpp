// expmc_b200.hpp — C++ host mirror of the reference estimator API over the
// C ABI (expmc_b200.h).  Header-only; link against libexpmc_b200.so.
//
// Mirrors, name for name (reference: /root/reference/proj/include/expmc/):
//   Splitting, PathParams{beta, n_steps, samples, splitting, seed}
//       estimator.hpp:11-33
//   Estimate, VectorEstimate                      estimator.hpp:37-52
//   entry_estimate / vector_estimate / tc_estimate estimator.hpp:59-72
//   split(SparseSymmetric) -> SplitMatrix          sparse_matrix.hpp:105
// Argument errors throw std::invalid_argument with the reference's
// messages; CUDA failures throw std::runtime_error.  `workers` is accepted
// and ignored (results do not depend on it).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "expmc_b200.h"

namespace expmc::b200 {

using NodeId = std::uint32_t;

enum class Splitting { Lie = EXPMC_LIE, Strang = EXPMC_STRANG };
enum class Rng { Philox = EXPMC_RNG_PHILOX, PcgCompat = EXPMC_RNG_PCG_COMPAT };

struct PathParams {
    double beta = 1.0;
    std::size_t n_steps = 32;
    std::size_t samples = 1'000'000;
    Splitting splitting = Splitting::Strang;
    std::uint64_t seed = 0;
    Rng rng = Rng::Philox;

    double dt() const { return beta / static_cast<double>(n_steps); }
    expmc_path_params c() const {
        return {beta, n_steps, samples, static_cast<int32_t>(splitting),
                static_cast<int32_t>(rng), seed};
    }
};

struct Estimate {
    double value = 0.0;
    double std_error = 0.0;
    std::size_t samples_used = 0;
    std::uint64_t total_jumps = 0;
};

struct VectorEstimate {
    std::vector<double> values;
    double std_error_global = 0.0;
    std::size_t samples_used = 0;
    std::uint64_t total_jumps = 0;
    double v_sum = 0.0;
};

struct EntriesEstimate {
    std::vector<double> values, std_errors;
    std::vector<std::uint64_t> jumps;
    std::uint64_t total_jumps = 0;
};

inline void check(int rc) {
    if (rc == EXPMC_OK) return;
    const std::string msg = expmc_cuda_last_error();
    if (rc == EXPMC_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// Device-resident SplitMatrix on one GPU (RAII over expmc_matrix*).
class SplitMatrix {
public:
    SplitMatrix() = default;
    // From the mirrored, row-sorted adjacency of a symmetric matrix
    // (SparseSymmetric's CSR) plus its diagonal; split() runs on the device.
    SplitMatrix(std::size_t n, std::span<const std::uint64_t> row_ptr,
                std::span<const std::uint32_t> col, std::span<const double> val,
                std::span<const double> diag = {}, int device = 0) {
        if (row_ptr.size() != n + 1) throw std::invalid_argument("row_ptr must have n + 1 entries");
        check(expmc_cuda_create_from_csr(n, row_ptr.data(), col.data(), val.data(),
                                         diag.empty() ? nullptr : diag.data(), device, &h_));
    }
    SplitMatrix(SplitMatrix&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    SplitMatrix& operator=(SplitMatrix&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    SplitMatrix(const SplitMatrix&) = delete;
    SplitMatrix& operator=(const SplitMatrix&) = delete;
    ~SplitMatrix() {
        if (h_) expmc_cuda_destroy(h_);
    }

    expmc_matrix* handle() const { return h_; }
    std::size_t n() const { return info().n; }
    std::size_t nnz() const { return info().nnz; }
    double dbar() const { return info().dbar; }
    std::size_t dmax() const { return info().dmax; }

private:
    struct Info {
        std::uint64_t n, nnz, dmax;
        double dbar;
    };
    Info info() const {
        Info i{};
        check(expmc_cuda_matrix_info(h_, &i.n, &i.nnz, &i.dbar, &i.dmax, nullptr, nullptr));
        return i;
    }
    expmc_matrix* h_ = nullptr;
};

inline Estimate entry_estimate(const SplitMatrix& m, std::span<const double> v, NodeId i,
                               const PathParams& p, unsigned /*workers*/ = 1) {
    const expmc_path_params c = p.c();
    expmc_estimate e{};
    check(expmc_cuda_entry_estimate(m.handle(), v.data(), v.size(), i, &c, &e));
    return {e.value, e.std_error, e.samples_used, e.total_jumps};
}

// Batched entry_estimate over `rows` (empty span = every row).
inline EntriesEstimate entries_estimate(const SplitMatrix& m, std::span<const double> v,
                                        std::span<const NodeId> rows, const PathParams& p) {
    const expmc_path_params c = p.c();
    const std::size_t k = rows.empty() ? m.n() : rows.size();
    EntriesEstimate out{std::vector<double>(k), std::vector<double>(k),
                        std::vector<std::uint64_t>(k)};
    check(expmc_cuda_entries(m.handle(), v.data(), v.size(), rows.empty() ? nullptr : rows.data(),
                             k, &c, out.values.data(), out.std_errors.data(), out.jumps.data(),
                             &out.total_jumps));
    return out;
}

// Batched entry_estimate over several replicas of one matrix — the
// reference's `workers` parallelism mapped to devices: `shards[k]` (one per
// GPU, or several on one GPU) estimates the k-th contiguous block of rows,
// all concurrently.  Bitwise identical to the single-replica call.
inline EntriesEstimate entries_estimate(std::span<const SplitMatrix* const> shards,
                                        std::span<const double> v,
                                        std::span<const NodeId> rows, const PathParams& p) {
    if (shards.empty()) throw std::invalid_argument("need at least one matrix handle");
    const expmc_path_params c = p.c();
    const std::size_t k = rows.empty() ? shards[0]->n() : rows.size();
    std::vector<expmc_matrix*> hs;
    for (const SplitMatrix* s : shards) hs.push_back(s ? s->handle() : nullptr);
    EntriesEstimate out{std::vector<double>(k), std::vector<double>(k),
                        std::vector<std::uint64_t>(k)};
    check(expmc_cuda_entries_multi(hs.data(), (int)hs.size(), v.data(), v.size(),
                                   rows.empty() ? nullptr : rows.data(), k, &c,
                                   out.values.data(), out.std_errors.data(), out.jumps.data(),
                                   &out.total_jumps));
    return out;
}

// One replica per device 0..ndev-1 of the same symmetric CSR (the
// `workers` -> GPUs mapping of entries_estimate above).
inline std::vector<SplitMatrix> replicas(int ndev, std::size_t n,
                                         std::span<const std::uint64_t> row_ptr,
                                         std::span<const std::uint32_t> col,
                                         std::span<const double> val,
                                         std::span<const double> diag = {}) {
    std::vector<SplitMatrix> r;
    for (int d = 0; d < ndev; ++d) r.emplace_back(n, row_ptr, col, val, diag, d);
    return r;
}

inline VectorEstimate vector_estimate(const SplitMatrix& m, std::span<const double> v,
                                      const PathParams& p, unsigned /*workers*/ = 1) {
    const expmc_path_params c = p.c();
    VectorEstimate e;
    e.values.resize(m.n());
    check(expmc_cuda_vector_estimate(m.handle(), v.data(), v.size(), &c, e.values.data(),
                                     &e.std_error_global, &e.total_jumps, &e.v_sum));
    e.samples_used = p.samples;
    return e;
}

inline Estimate tc_estimate(const SplitMatrix& m, const PathParams& p, unsigned /*workers*/ = 1) {
    const expmc_path_params c = p.c();
    expmc_estimate e{};
    check(expmc_cuda_tc_estimate(m.handle(), &c, &e));
    return {e.value, e.std_error, e.samples_used, e.total_jumps};
}

}  // namespace expmc::b200
