// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile).  Only tests/, the smoke
// check and bench.py's reference / cpu_baseline legs load the resulting
// oracle/_ref/libexpmc_ref.so.  Every function forwards to the reference's
// own public API:
//   SparseSymmetric::from_entries   proj/src/sparse_matrix.cpp:18-85
//   split                           proj/src/sparse_matrix.cpp:101-142
//   stats                           proj/src/sparse_matrix.cpp:176-217
//   generate                        proj/src/generators.cpp:154-164
//   entry_estimate                  proj/src/estimator.cpp:169-206
//   vector_estimate                 proj/src/estimator.cpp:208-278
//   tc_estimate                     proj/src/estimator.cpp:280-318
//   load/write_matrix_market        proj/src/matrix_market.cpp:51-207
//   RngStream / exp_time / advance  proj/include/expmc/rng.hpp:14-63,
//                                   proj/src/sampler.cpp:10-49
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "expmc/estimator.hpp"
#include "expmc/generators.hpp"
#include "expmc/matrix_market.hpp"
#include "expmc/metrics.hpp"
#include "expmc/rng.hpp"
#include "expmc/sampler.hpp"
#include "expmc/sparse_matrix.hpp"

using namespace expmc;

namespace {
thread_local std::string g_err;

struct RefMatrix {
    SparseSymmetric sym;
    SplitMatrix split;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

PathParams make_params(double beta, std::uint64_t n_steps, std::uint64_t samples,
                       int splitting, std::uint64_t seed) {
    PathParams p;
    p.beta = beta;
    p.n_steps = n_steps;
    p.samples = samples;
    p.splitting = splitting == 0 ? Splitting::Lie : Splitting::Strang;
    p.seed = seed;
    return p;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Build from a (possibly two-triangle) entry list via the reference's own
// validating constructor, then split().  Returns NULL on error.
void* ref_from_entries(std::uint64_t n, const std::uint32_t* rows,
                       const std::uint32_t* cols, const double* w,
                       std::uint64_t ne) {
    RefMatrix* out = nullptr;
    int rc = guarded([&] {
        std::vector<Entry> e(ne);
        for (std::uint64_t k = 0; k < ne; ++k) e[k] = {rows[k], cols[k], w[k]};
        auto* m = new RefMatrix;
        m->sym = SparseSymmetric::from_entries(n, std::move(e));
        m->split = split(m->sym);
        out = m;
    });
    return rc == 0 ? out : nullptr;
}

// Upper-triangle + diagonal entries taken from a symmetric two-direction CSR.
void* ref_from_csr(std::uint64_t n, const std::uint64_t* row_ptr,
                   const std::uint32_t* col, const double* val,
                   const double* diag) {
    std::vector<std::uint32_t> r, c;
    std::vector<double> w;
    for (std::uint64_t i = 0; i < n; ++i) {
        if (diag && diag[i] != 0.0) {
            r.push_back((std::uint32_t)i);
            c.push_back((std::uint32_t)i);
            w.push_back(diag[i]);
        }
        for (std::uint64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            if (col[k] > i) {
                r.push_back((std::uint32_t)i);
                c.push_back(col[k]);
                w.push_back(val[k]);
            }
        }
    }
    return ref_from_entries(n, r.data(), c.data(), w.data(), r.size());
}

// kind: 0 SmallWorld, 1 ScaleFree, 2 ErdosRenyi (generators.hpp:9).
void* ref_generate(int kind, std::uint64_t n, std::uint64_t k, double ps,
                   std::uint64_t m0, double p, std::uint64_t seed) {
    RefMatrix* out = nullptr;
    int rc = guarded([&] {
        GenSpec s;
        s.kind = kind == 0 ? GraphKind::SmallWorld
                           : (kind == 1 ? GraphKind::ScaleFree : GraphKind::ErdosRenyi);
        s.n = n;
        s.k = k;
        s.ps = ps;
        s.m0 = m0;
        s.p = p;
        s.seed = seed;
        auto* m = new RefMatrix;
        m->sym = generate(s);
        m->split = split(m->sym);
        out = m;
    });
    return rc == 0 ? out : nullptr;
}

// load_matrix_market + split; *status: 0 ok, 1 invalid_argument, 2 other.
void* ref_mm_load(const char* path, int* status) {
    RefMatrix* out = nullptr;
    *status = guarded([&] {
        auto* m = new RefMatrix;
        try {
            m->sym = load_matrix_market(path);
            m->split = split(m->sym);
        } catch (...) {
            delete m;
            throw;
        }
        out = m;
    });
    return out;
}

int ref_mm_write(void* h, const char* path) {
    return guarded([&] { write_matrix_market(static_cast<RefMatrix*>(h)->sym, path); });
}

void ref_destroy(void* h) { delete static_cast<RefMatrix*>(h); }

void ref_sizes(void* h, std::uint64_t* n, std::uint64_t* nnz) {
    auto* m = static_cast<RefMatrix*>(h);
    *n = m->split.n;
    *nnz = m->split.neighbor.size();
}

// Export the SplitMatrix (sparse_matrix.hpp:66-91) field by field.  Any
// output pointer may be NULL.
void ref_split_export(void* h, double* diag, double* d, double* rate,
                      std::uint64_t* row_offset, std::uint32_t* neighbor,
                      double* weight, double* cum, std::uint8_t* uniform_row,
                      double* dbar, std::uint64_t* dmax) {
    const SplitMatrix& s = static_cast<RefMatrix*>(h)->split;
    const std::size_t n = s.n, nnz = s.neighbor.size();
    if (diag) std::memcpy(diag, s.diag.data(), n * 8);
    if (d) std::memcpy(d, s.d.data(), n * 8);
    if (rate) std::memcpy(rate, s.rate.data(), n * 8);
    if (row_offset)
        for (std::size_t i = 0; i <= n; ++i) row_offset[i] = s.row_offset[i];
    if (neighbor) std::memcpy(neighbor, s.neighbor.data(), nnz * 4);
    if (weight) std::memcpy(weight, s.weight.data(), nnz * 8);
    if (cum) std::memcpy(cum, s.cum.data(), nnz * 8);
    if (uniform_row) std::memcpy(uniform_row, s.uniform_row.data(), n);
    if (dbar) *dbar = s.dbar;
    if (dmax) *dmax = s.dmax;
}

double ref_lambda_max(void* h, std::uint64_t iters) {
    auto st = stats(static_cast<RefMatrix*>(h)->split, iters);
    return st.lambda_max.value_or(0.0);
}

int ref_entry_estimate(void* h, const double* v, std::uint64_t nv,
                       std::uint64_t i, double beta, std::uint64_t n_steps,
                       std::uint64_t samples, int splitting, std::uint64_t seed,
                       unsigned workers, double* value, double* se,
                       std::uint64_t* jumps) {
    return guarded([&] {
        const auto& m = static_cast<RefMatrix*>(h)->split;
        Estimate e = entry_estimate(m, std::span<const double>(v, nv),
                                    (NodeId)i,
                                    make_params(beta, n_steps, samples, splitting, seed),
                                    workers);
        *value = e.value;
        *se = e.std_error;
        *jumps = e.total_jumps;
    });
}

// Many rows.  nthreads <= 1: sequential calls with `workers` threads each
// (the reference "as-is" mode).  nthreads > 1: row-parallel, nthreads
// threads each calling entry_estimate(..., workers=1) on rows taken from a
// shared counter (legal: SplitMatrix is immutable, sparse_matrix.hpp:63-65).
int ref_entries(void* h, const double* v, std::uint64_t nv,
                const std::uint64_t* rows, std::uint64_t nrows, double beta,
                std::uint64_t n_steps, std::uint64_t samples, int splitting,
                std::uint64_t seed, unsigned workers, unsigned nthreads,
                double* value, double* se, std::uint64_t* jumps) {
    return guarded([&] {
        const auto& m = static_cast<RefMatrix*>(h)->split;
        const PathParams p = make_params(beta, n_steps, samples, splitting, seed);
        const std::span<const double> vs(v, nv);
        if (nthreads <= 1) {
            for (std::uint64_t r = 0; r < nrows; ++r) {
                Estimate e = entry_estimate(m, vs, (NodeId)rows[r], p, workers);
                value[r] = e.value;
                se[r] = e.std_error;
                jumps[r] = e.total_jumps;
            }
            return;
        }
        std::atomic<std::uint64_t> next{0};
        std::vector<std::string> errs(nthreads);
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nthreads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (;;) {
                        const std::uint64_t r = next.fetch_add(1);
                        if (r >= nrows) break;
                        Estimate e = entry_estimate(m, vs, (NodeId)rows[r], p, 1);
                        value[r] = e.value;
                        se[r] = e.std_error;
                        jumps[r] = e.total_jumps;
                    }
                } catch (const std::exception& ex) {
                    errs[t] = ex.what();
                    next.store(nrows);
                }
            });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::invalid_argument(e);
    });
}

int ref_vector_estimate(void* h, const double* v, std::uint64_t nv, double beta,
                        std::uint64_t n_steps, std::uint64_t samples,
                        int splitting, std::uint64_t seed, unsigned workers,
                        double* values, double* se_global,
                        std::uint64_t* jumps, double* v_sum) {
    return guarded([&] {
        const auto& m = static_cast<RefMatrix*>(h)->split;
        VectorEstimate e = vector_estimate(
            m, std::span<const double>(v, nv),
            make_params(beta, n_steps, samples, splitting, seed), workers);
        std::memcpy(values, e.values.data(), e.values.size() * 8);
        *se_global = e.std_error_global;
        *jumps = e.total_jumps;
        *v_sum = e.v_sum;
    });
}

int ref_tc_estimate(void* h, double beta, std::uint64_t n_steps,
                    std::uint64_t samples, int splitting, std::uint64_t seed,
                    unsigned workers, double* value, double* se,
                    std::uint64_t* jumps) {
    return guarded([&] {
        const auto& m = static_cast<RefMatrix*>(h)->split;
        Estimate e = tc_estimate(
            m, make_params(beta, n_steps, samples, splitting, seed), workers);
        *value = e.value;
        *se = e.std_error;
        *jumps = e.total_jumps;
    });
}

// --- ranking metrics (metrics.cpp:10-55) ---------------------------------
int ref_rank(const double* values, std::uint64_t n, std::uint32_t* order) {
    return guarded([&] {
        RankedVector r = rank(std::span<const double>(values, n));
        std::memcpy(order, r.order.data(), n * 4);
    });
}

int ref_isim(const std::uint32_t* ox, const std::uint32_t* oy, std::uint64_t nx,
             std::uint64_t ny, double top_fraction, double* out) {
    return guarded([&] {
        RankedVector x, y;
        x.order.assign(ox, ox + nx);
        y.order.assign(oy, oy + ny);
        x.scores.assign(nx, 0.0);
        y.scores.assign(ny, 0.0);
        *out = isim(x, y, top_fraction);
    });
}

// --- RNG / sampler known-answer helpers (rng.hpp, sampler.cpp) ------------
// op: 0 next_u32, 1 next_u64, 2 uniform, 3 uniform_pos, 4 uniform_index(arg)
void ref_rng_draws(std::uint64_t seed, std::uint64_t stream, int op,
                   std::uint64_t arg, std::uint64_t count, void* out) {
    RngStream rng(seed, stream);
    for (std::uint64_t k = 0; k < count; ++k) {
        switch (op) {
            case 0: static_cast<std::uint32_t*>(out)[k] = rng.next_u32(); break;
            case 1: static_cast<std::uint64_t*>(out)[k] = rng.next_u64(); break;
            case 2: static_cast<double*>(out)[k] = rng.uniform(); break;
            case 3: static_cast<double*>(out)[k] = rng.uniform_pos(); break;
            default:
                static_cast<std::uint64_t*>(out)[k] = rng.uniform_index(arg);
                break;
        }
    }
}

int ref_exp_times(std::uint64_t seed, std::uint64_t stream, double rate,
                  std::uint64_t count, double* out) {
    return guarded([&] {
        RngStream rng(seed, stream);
        for (std::uint64_t k = 0; k < count; ++k) out[k] = exp_time(rng, rate);
    });
}

// One advance() per stream id l in [0, count) from `start`.
int ref_advance(void* h, std::uint64_t seed, std::uint64_t start, double dt,
                std::uint64_t count, std::uint32_t* end_state,
                std::uint64_t* jumps) {
    return guarded([&] {
        const auto& m = static_cast<RefMatrix*>(h)->split;
        for (std::uint64_t l = 0; l < count; ++l) {
            RngStream rng(seed, l);
            auto r = advance(rng, m, (NodeId)start, dt);
            end_state[l] = r.end_state;
            jumps[l] = r.jumps;
        }
    });
}

}  // extern "C"
