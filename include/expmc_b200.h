/*
 * expmc_b200 — C ABI of the B200-native Monte Carlo exp(tA)v hot path.
 *
 * Drop-in boundary for the reference C++ API (namespace expmc,
 * /root/reference/proj/include/expmc/estimator.hpp:59-72 and
 * sparse_matrix.hpp:105).  Plain pointers and sizes only; no CUDA or torch
 * types.  Every function returns an expmc_status; on failure
 * expmc_cuda_last_error() (thread-local) holds the message, which for
 * argument errors is the reference's own std::invalid_argument text.
 *
 * Conventions (mirroring the reference):
 *   - NodeId is uint32_t (sparse_matrix.hpp:11).
 *   - The matrix is immutable after creation and may be shared by callers
 *     (sparse_matrix.hpp:63-65); a handle is bound to one CUDA device and
 *     should be used by one host thread at a time.
 *   - Host-buffer calls are synchronous and blocking, like the reference.
 *   - *_device calls take device pointers on the handle's device and a
 *     cudaStream_t passed as void* (NULL = the legacy default stream); they
 *     are asynchronous on that stream.
 */
#ifndef EXPMC_B200_H_
#define EXPMC_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    EXPMC_OK = 0,
    EXPMC_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    EXPMC_RUNTIME_ERROR = 2,    /* reference: std::runtime_error     */
    EXPMC_CUDA_ERROR = 3        /* CUDA failure (maps to runtime_error) */
} expmc_status;

/* Splitting (estimator.hpp:11). */
enum { EXPMC_LIE = 0, EXPMC_STRANG = 1 };

/* Walker engine.  PHILOX is the production path (K3/K4: continuous clock,
 * counter-based RNG keyed by (seed, row, walker)).  PCG_COMPAT (K2) replays
 * the reference's PCG32 streams path by path for parity checks. */
enum { EXPMC_RNG_PHILOX = 0, EXPMC_RNG_PCG_COMPAT = 1 };

/* PathParams (estimator.hpp:16-33): dt = beta / n_steps. */
typedef struct {
    double beta;
    uint64_t n_steps;
    uint64_t samples;  /* M: walkers per entry (entry) or in total (vector, tc) */
    int32_t splitting; /* EXPMC_LIE or EXPMC_STRANG */
    int32_t rng;       /* EXPMC_RNG_PHILOX or EXPMC_RNG_PCG_COMPAT */
    uint64_t seed;
} expmc_path_params;

/* Estimate (estimator.hpp:37-42). */
typedef struct {
    double value;
    double std_error;
    uint64_t samples_used;
    uint64_t total_jumps;
} expmc_estimate;

typedef struct expmc_matrix expmc_matrix; /* device-resident SplitMatrix */

const char* expmc_cuda_last_error(void);
int expmc_cuda_abi_version(void); /* 1 */

/* ------------------------------------------------------------ matrices */
/* From the mirrored adjacency of a SparseSymmetric (sparse_matrix.hpp:25-61):
 * rows sorted by column, both directions stored, off-diagonal weights > 0,
 * diagonal separately (diag may be NULL = zero).  Validated on the device
 * with from_entries' checks (sparse_matrix.cpp:20-51), then split() runs on
 * the device (K1, bit-exact with sparse_matrix.cpp:101-142). */
int expmc_cuda_create_from_csr(uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                               const double* val, const double* diag, int device,
                               expmc_matrix** out);
/* From a raw entry list, exactly SparseSymmetric::from_entries
 * (sparse_matrix.cpp:18-85) on the device: entries may come in either
 * triangle and any order; validated with the reference's messages and
 * precedence (first offending entry in input order, then the first duplicate
 * after canonical sorting), sorted, mirrored, then split on the device. */
int expmc_cuda_create_from_entries(uint64_t n, const uint32_t* rows, const uint32_t* cols,
                                   const double* weights, uint64_t n_entries, int device,
                                   expmc_matrix** out);
/* From an existing reference SplitMatrix (sparse_matrix.hpp:66-91): its
 * row_offset / neighbor / weight / diag fields.  rate, cum, d, uniform_row,
 * dbar and dmax are re-derived on the device bit-exactly. */
int expmc_cuda_create_from_split(uint64_t n, const uint64_t* row_offset,
                                 const uint32_t* neighbor, const double* weight,
                                 const double* diag, int device, expmc_matrix** out);
/* From a Matrix Market coordinate file, exactly load_matrix_market
 * (matrix_market.cpp:51-165): header rules and "path:line: what" messages
 * as EXPMC_RUNTIME_ERROR; the body is parsed on all host cores, the
 * general-symmetry fold and from_entries run on the device (from_entries'
 * own messages as EXPMC_INVALID_ARGUMENT), then split() on the device. */
int expmc_cuda_create_from_mm(const char* path, int device, expmc_matrix** out);
int expmc_cuda_destroy(expmc_matrix* m);

int expmc_cuda_matrix_info(const expmc_matrix* m, uint64_t* n, uint64_t* nnz, double* dbar,
                           uint64_t* dmax, int32_t* any_nonuniform, int32_t* device);
/* Copy the device SplitMatrix back (any pointer may be NULL). */
int expmc_cuda_split_export(const expmc_matrix* m, double* diag, double* d, double* rate,
                            uint64_t* row_offset, uint32_t* neighbor, double* weight,
                            double* cum, uint8_t* uniform_row);
/* Walker alias tables (nnz each): keep column k of a row when a u32 coin is
 * < thr[k], else jump to column alias[k].  Uniform rows hold thr = ~0. */
int expmc_cuda_alias_export(const expmc_matrix* m, uint32_t* thr, uint32_t* alias);
/* Packed 32-byte row records {u32 off, u32 deg|nonuniform<<31, f32 1/rate,
 * u32 0, f64 d, f64 v}, n * 32 bytes. */
int expmc_cuda_records_export(const expmc_matrix* m, void* out);

/* ---------------------------------------------------------- estimators */
/* entry_estimate (estimator.cpp:169-206): one entry i of
 * the splitting approximation to exp(beta A) v. */
int expmc_cuda_entry_estimate(expmc_matrix* m, const double* v, uint64_t nv, uint32_t i,
                              const expmc_path_params* p, expmc_estimate* out);
/* Batched entry_estimate over rows[0..nrows) (rows == NULL: every row,
 * nrows must equal n): the "full vector with W walkers per entry".
 * total_jumps (may be NULL) receives the sum of jumps[] (reduced on the
 * device for the Philox walker). */
int expmc_cuda_entries(expmc_matrix* m, const double* v, uint64_t nv, const uint32_t* rows,
                       uint64_t nrows, const expmc_path_params* p, double* value,
                       double* std_error, uint64_t* jumps, uint64_t* total_jumps);
/* The batched entry estimator over several replicas of one matrix (the
 * reference's `workers` knob, estimator.hpp:59-61 / estimator.cpp:50-68,
 * mapped to devices): rows split into nh contiguous equal shards, shard k
 * on handles[k] (one per GPU, or several on one GPU), all driven
 * concurrently; each shard's slice lands directly in value / std_error /
 * jumps.  Bitwise identical to expmc_cuda_entries on one handle for any nh. */
int expmc_cuda_entries_multi(expmc_matrix* const* handles, int nh, const double* v, uint64_t nv,
                             const uint32_t* rows, uint64_t nrows, const expmc_path_params* p,
                             double* value, double* std_error, uint64_t* jumps,
                             uint64_t* total_jumps);
/* Staged-v reuse for repeated host entry calls with the same v (the
 * reference passes v on every call, estimator.hpp:59-60, and recomputes its
 * O(n) node factors each time, estimator.cpp:177-178).  With the cache
 * enabled, a call whose v pointer and length equal the last staged ones
 * skips the H2D copy, the finiteness scan and the repack of v into the
 * walk layout; the caller must call expmc_cuda_invalidate_v after changing
 * v in place.  Off by default (every call stages v).  v_stagings counts the
 * stagings performed (measurement / tests). */
int expmc_cuda_set_v_cache(expmc_matrix* m, int enable);
int expmc_cuda_invalidate_v(expmc_matrix* m);
int expmc_cuda_v_stagings(const expmc_matrix* m, uint64_t* count);
/* Test hook: `count` Exp(1) draws of the walkers' transform (neg_ln_u over
 * Philox words), histogram in nbins bins of bin_width (last bin = the rest)
 * and moments {sum E, sum E^2}; the law check of sampler.cpp:10-16's
 * exp_time (tests/test_gpu_rng_law.py). */
int expmc_cuda_exp_law(int device, uint64_t count, uint64_t seed, double bin_width,
                       uint32_t nbins, uint64_t* hist, double* moments);
/* vector_estimate (estimator.cpp:208-278), Theorem 2; values has n entries. */
int expmc_cuda_vector_estimate(expmc_matrix* m, const double* v, uint64_t nv,
                               const expmc_path_params* p, double* values,
                               double* std_error_global, uint64_t* total_jumps,
                               double* v_sum);
/* tc_estimate (estimator.cpp:280-318). */
int expmc_cuda_tc_estimate(expmc_matrix* m, const expmc_path_params* p, expmc_estimate* out);
/* One shard of vector_estimate / tc_estimate (multi-GPU): only
 * the walkers whose start lies in rows [row_lo, row_hi) — the same walkers,
 * with the same randomness, that the unsharded call runs there (Philox
 * engine only).  values (n entries, may be NULL for the scalar functional) is
 * this shard's per-end contribution divided by M; sum / sum_sq / total_jumps
 * are its raw tallies.  Over a partition of the rows the shard values add up
 * to vector_estimate's values and the tallies give its std_error_global via
 * finalize (estimator.cpp:76-89); only the fp summation order differs. */
int expmc_cuda_vector_estimate_rows(expmc_matrix* m, const double* v, uint64_t nv,
                                    const expmc_path_params* p, uint64_t row_lo,
                                    uint64_t row_hi, double* values, double* sum,
                                    double* sum_sq, uint64_t* total_jumps);
int expmc_cuda_tc_estimate_rows(expmc_matrix* m, const expmc_path_params* p, uint64_t row_lo,
                                uint64_t row_hi, double* sum, double* sum_sq,
                                uint64_t* total_jumps);

/* -------------------------------------------- device-resident variants */
/* Stage v (device pointer, n doubles) for subsequent *_device calls:
 * checks finiteness (same message as check_vector) and packs v into the
 * row records.  Synchronises the stream to report errors. */
int expmc_cuda_set_v_device(expmc_matrix* m, const double* v_dev, uint64_t nv, void* stream);
/* Philox entry walker (K3) over device rows -> device outputs, async.
 * Rows are NOT range-checked here (the caller's host layer does that). */
int expmc_cuda_entries_device(expmc_matrix* m, const uint32_t* rows_dev, uint64_t nrows,
                              const expmc_path_params* p, double* value_dev,
                              double* std_error_dev, uint64_t* jumps_dev, void* stream);
/* Same over the contiguous rows [row_lo, row_lo + nrows) (range-checked): no
 * row array — the walker derives a task's row from its index.  Bitwise the
 * same results as the listed form. */
int expmc_cuda_entries_device_range(expmc_matrix* m, uint64_t row_lo, uint64_t nrows,
                                    const expmc_path_params* p, double* value_dev,
                                    double* std_error_dev, uint64_t* jumps_dev, void* stream);
/* K6 gather ceiling: chains_per_row chains of chain_len jumps from every
 * listed row (memory-only walker, same access pattern as K3), async. */
int expmc_cuda_gather_ceiling_device(expmc_matrix* m, const uint32_t* rows_dev, uint64_t nrows,
                                     uint32_t chains_per_row, uint32_t chain_len, void* stream);
/* Lane slots T per entry used by the Philox entry walker for W walkers
 * (W < 2^29): the entry's walkers are split into T/32 contiguous parts; the
 * k-th jumper of a part is summed in lane k mod 32, lanes by a fixed xor
 * tree, parts in order — part of the result contract (oracle/fast_model.c
 * replays it). */
uint32_t expmc_cuda_entry_slots(uint64_t walkers);
/* Number of kernels this library has launched in this process. */
uint64_t expmc_cuda_launch_count(void);

/* K4 facts about the last vector / tc estimate on this handle: jumpers
 * (walkers with at least one jump, i.e. walks actually run) and the per-end
 * reduction used by vector_estimate (1: exact 128-bit fixed point, 0:
 * sort-based, -1: none yet).  Either pointer may be NULL. */
int expmc_cuda_last_k4_stats(const expmc_matrix* m, uint64_t* jumpers, int* fixed_point);

/* ------------------------------------------- K4 sampler diagnostics (tests) */
/* `count` draws of the device Binomial(trials, p) sampler used by the
 * Theorem-2 walkers (inversion / BTRS), Philox-keyed by seed, into out[]. */
int expmc_cuda_binomial_samples(int device, uint64_t trials, double p, uint64_t count,
                                uint64_t seed, uint64_t* out);
/* The K4 start counts: walkers per start row ~ Multinomial(samples, v / V)
 * (v == NULL: uniform over rows), as vector_estimate / tc_estimate draw them
 * for (samples, seed).  counts[] has n entries and sums to samples. */
int expmc_cuda_start_counts(expmc_matrix* m, const double* v, uint64_t nv, uint64_t samples,
                            uint64_t seed, uint64_t* counts);

/* ------------------------------------------------------- accuracy (K5) */
/* Deterministic fp64 y = exp(t A) v by scaled Taylor series (tol relative). */
int expmc_cuda_expmv(expmc_matrix* m, const double* v, uint64_t nv, double t, double tol,
                     double* out);
/* stats() power iteration (sparse_matrix.cpp:176-217) on the device:
 * largest eigenvalue of A via the Gershgorin-shifted power method. */
int expmc_cuda_lambda_max(expmc_matrix* m, uint64_t power_iters, double* lambda_max,
                          double* rel_change);
/* Deterministic splitting product the estimators sample:
 *   Strang (e^{dt D/2} e^{-dt L} e^{dt D/2})^N v,  Lie (e^{-dt L} e^{dt D})^N v. */
int expmc_cuda_splitting_product(expmc_matrix* m, const double* v, uint64_t nv,
                                 const expmc_path_params* p, double tol, double* out);

/* ------------------------------------------------ ranking metrics (f4) */
/* rank() (metrics.cpp:10-25): order[] = node ids by descending score, ties
 * by ascending id; "rank: NaN score" on NaN. */
int expmc_cuda_rank(const double* scores, uint64_t n, int device, uint32_t* order);
/* isim() (metrics.cpp:27-55) of two rankings' top ceil(top_fraction * n)
 * prefixes; same checks and messages as the reference. */
int expmc_cuda_isim(const uint32_t* order_x, const uint32_t* order_y, uint64_t nx, uint64_t ny,
                    double top_fraction, int device, double* out);

/* ----------------------------------------- synthetic inputs (host, C++) */
/* Host CSR builders for the benchmark configurations.  The returned object
 * owns a mirrored, row-sorted CSR (the SparseSymmetric adjacency) plus the
 * diagonal. */
typedef struct expmc_csr expmc_csr;
const char* expmc_gen_last_error(void); /* message of the last failed expmc_gen_* */
/* 2-D 5-point / 3-D 7-point Dirichlet FD stencil scaled by s:
 * diag -2*dim*s, neighbours +s. */
int expmc_gen_fd(int dim, uint64_t side, double s, expmc_csr** out);
/* Barabasi-Albert exactly as generate({ScaleFree, n, m0, seed})
 * (generators.cpp:58-103). */
int expmc_gen_ba(uint64_t n, uint64_t m0, uint64_t seed, expmc_csr** out);
/* Watts-Strogatz: ring with k/2 neighbours per side, each edge rewired with
 * probability p (no self loops, no duplicates), PCG32 stream (seed, 0). */
int expmc_gen_ws(uint64_t n, uint64_t half_k, double p, uint64_t seed, expmc_csr** out);
int expmc_csr_sizes(const expmc_csr* c, uint64_t* n, uint64_t* nnz);
int expmc_csr_export(const expmc_csr* c, uint64_t* row_ptr, uint32_t* col, double* val,
                     double* diag);
/* Zero-copy views (valid until expmc_csr_free). */
int expmc_csr_view(const expmc_csr* c, const uint64_t** row_ptr, const uint32_t** col,
                   const double** val, const double** diag);
void expmc_csr_free(expmc_csr* c);

/* ------------------------------------ Matrix Market + CSR cache (f1, f3) */
/* load_matrix_market (matrix_market.cpp:51-165) into a host CSR (the
 * SparseSymmetric adjacency); fold + from_entries on `device`.  Errors as
 * expmc_cuda_create_from_mm, message in expmc_cuda_last_error(). */
int expmc_cuda_mm_load(const char* path, int device, expmc_csr** out);
/* The parse alone (matrix_market.cpp:51-131, host, all cores): entries in
 * file order, 0-based, before the general fold / from_entries.  Message in
 * expmc_gen_last_error(). */
typedef struct expmc_mm expmc_mm;
int expmc_mm_parse(const char* path, expmc_mm** out);
int expmc_mm_info(const expmc_mm* m, uint64_t* n, uint64_t* n_entries, int32_t* general,
                  int32_t* pattern, uint64_t* last_line);
int expmc_mm_view(const expmc_mm* m, const uint32_t** rows, const uint32_t** cols,
                  const double** weights);
void expmc_mm_free(expmc_mm* m);
/* write_matrix_market (matrix_market.cpp:167-194) of a mirrored CSR + diag
 * (diag may be NULL): lower triangle, 1-based, shortest round-trip weights,
 * `pattern` when every stored weight is 1. */
int expmc_mm_write(const char* path, uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                   const double* val, const double* diag);
/* Binary CSR cache: 64-byte header ("EXPMCCSR", version 1, n, nnz,
 * checksum) + row_ptr u64[n+1] + col u32[nnz] (8-byte padded) + val f64[nnz]
 * + diag f64[n].  Load verifies size, checksum and row_ptr. */
int expmc_csr_save(const char* path, uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                   const double* val, const double* diag);
int expmc_csr_load(const char* path, expmc_csr** out);
/* Seeded vectors / row samples with PCG32 RngStream(seed, 0):
 *   kind 0: U[0,1)  1: U[-1,1)  2: 3-D Gaussian bump (sigma) + U[0,1) on a
 *   side^3 grid (row-major, cube [0,1]^3, centre 0.5) */
int expmc_gen_vector(int kind, uint64_t n, uint64_t side, double sigma, uint64_t seed,
                     double* out);
/* k distinct rows of [0, n), uniform without replacement (partial
 * Fisher-Yates, RngStream(seed, 0)), returned sorted ascending. */
int expmc_gen_row_sample(uint64_t n, uint64_t k, uint64_t seed, uint32_t* out);

#ifdef __cplusplus
}
#endif

#endif /* EXPMC_B200_H_ */
