// Internal declarations shared by the .cu translation units and the host
// driver (api.cu).  Not part of the public C ABI (include/expmc_b200.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace expmc_b200 {

// Device-resident SplitMatrix (proj/include/expmc/sparse_matrix.hpp:66-91)
// plus the B200 walk layout.  All pointers are device pointers.
struct DevSplit {
    uint64_t n = 0, nnz = 0;
    // SplitMatrix fields, same meaning and bits as the reference
    double* diag = nullptr;
    double* d = nullptr;
    double* rate = nullptr;
    uint64_t* row_offset = nullptr;
    uint32_t* neighbor = nullptr;
    double* weight = nullptr;
    double* cum = nullptr;
    uint8_t* uniform_row = nullptr;
    double dbar = 0.0;
    uint64_t dmax = 0;
    bool any_nonuniform = false;
    double mean_rate = 0.0;      // launch heuristics only (K3 occupancy choice)
    double dabs_max = 0.0;       // max |d_i| (+inf if some d is not finite): K3's exp range bound
    // walk layout
    RowRec* rec = nullptr;       // n packed 32-B row records
    uint32_t* alias_thr = nullptr; // nnz (only if any_nonuniform)
    uint32_t* alias_idx = nullptr; // nnz (only if any_nonuniform)
    Edge* adj = nullptr;           // nnz fat adjacency slots (32 B each)
};

// Parameters of the fast walkers (K3/K4).  Built once on the host from
// PathParams; the CPU model oracle/fast_model.c consumes the same numbers.
struct FastParams {
    double beta;   // horizon β
    double dt;     // β / N
    double inv_dt; // N / β
    double n_grid; // (double) N
    double n_grid1; // (double) (N + 1)
    uint32_t N;
    int strang;
    uint64_t W;    // walkers per entry (K3) or total walkers (K4)
    uint32_t k0, k1; // Philox key = seed
    // Philox round keys (k0 + r W0, k1 + r W1), precomputed on the host so the
    // rounds read them as constant-bank operands instead of registers.
    PhiloxKeys rk;
    unsigned long long* stats = nullptr;  // ENTRY_STATS builds only
    uint32_t row0 = 0;  // K3 with rows == nullptr: the launch covers rows [row0, row0 + nrows)
    int exp_safe = 0;   // K3: every exponent Δt (S - corr) is within ±690 (set per launch
                        // from max |d|): exp_det without range clamps, same bits
};

// split_pack.cu
void launch_validate_csr(uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                         const double* val, unsigned long long* err, cudaStream_t s);
void launch_split_pack(uint64_t n, const uint64_t* row_ptr, const double* weight,
                       const double* diag, double* d, double* rate, double* cum,
                       uint8_t* uniform_row, RowRec* rec, unsigned long long* dmax,
                       unsigned int* any_nonuniform, cudaStream_t s);
void launch_rate_sum(uint64_t n, const double* rate, const double* d, double* out,
                     unsigned long long* dabs_max, cudaStream_t s);
void launch_alias_build(uint64_t n, const uint64_t* row_ptr, const double* weight,
                        const double* rate, const uint8_t* uniform_row, uint32_t* thr,
                        uint32_t* alias, double* p, uint32_t* small, uint32_t* large,
                        cudaStream_t s);
void launch_pack_v(uint64_t n, const double* v, RowRec* rec, cudaStream_t s);
void launch_build_adj(uint64_t nnz, const uint32_t* neighbor, const RowRec* rec, Edge* adj,
                      cudaStream_t s);
void launch_pack_v_adj(uint64_t nnz, const uint32_t* neighbor, const double* v, Edge* adj,
                       cudaStream_t s);
void launch_node_factors(uint64_t n, const double* d, double scale, double* f,
                         cudaStream_t s);

// walk_compat.cu (K2)
void launch_entry_compat(const DevSplit& m, const double* v, const uint32_t* rows,
                         uint64_t nrows, double dt, uint64_t n_steps, uint64_t samples,
                         const double* before, const double* after, uint64_t seed,
                         double* value, double* se, uint64_t* jumps, cudaStream_t s);
unsigned scatter_compat_grid();
void launch_scatter_compat(const DevSplit& m, int start_mode, const double* vcum, double v_sum,
                           double dt, uint64_t n_steps, uint64_t samples, const double* before,
                           const double* after, uint64_t seed, uint64_t l0, uint64_t lend,
                           uint32_t* out_end, double* out_f, double* part_sum, double* part_sq,
                           unsigned long long* part_j, cudaStream_t s);

// from_entries.cu (§8f f1)
void from_entries_device(uint64_t n, const uint32_t* r, const uint32_t* c, const double* w,
                         uint64_t ne, uint64_t* row_ptr, uint32_t** col_out, double** val_out,
                         double* diag, uint64_t* nnz_out, unsigned long long* err_host,
                         unsigned long long* dup_key, cudaStream_t s);
void fold_general_device(const uint32_t* r, const uint32_t* c, const double* w, uint64_t ne,
                         uint32_t** r_out, uint32_t** c_out, double** w_out, uint64_t* m,
                         unsigned long long* err_host, unsigned long long* err_key,
                         cudaStream_t s);

// metrics.cu (§8f f4)
bool rank_device(const double* scores_host, uint64_t n, uint32_t* order_host, cudaStream_t s);
double isim_device(const uint32_t* ox_host, const uint32_t* oy_host, uint64_t n, uint64_t k,
                   cudaStream_t s);

// scatter_sort.cu
size_t scatter_sort_temp_bytes(uint64_t batch, uint64_t n);
// sort + per-run sums; launches 3 kernels (sort counted as one)
void scatter_sort_accumulate(uint32_t* end, double* f, uint32_t* end_sorted, double* f_sorted,
                             uint64_t count, uint64_t n, void* temp, size_t temp_bytes,
                             double* values, cudaStream_t s);

// walk_entry.cu (K3), walk_fast.cu (K6)
int entry_fast_wpr(uint64_t W);
size_t entry_fast_scratch_bytes(uint64_t nrows, uint64_t W);
// returns the number of kernels launched
int launch_entry_fast(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                      const FastParams& p, double* value, double* se, uint64_t* jumps,
                      void* scratch, cudaStream_t s);
void launch_exp_law(uint64_t count, uint64_t seed, double width, uint32_t nbins,
                    unsigned long long* hist, unsigned long long* mom, cudaStream_t s);
void launch_gather_ceiling(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                           uint32_t chains_per_row, uint32_t chain_len, uint32_t salt,
                           unsigned long long* sink, cudaStream_t s);

// walk_vec.cu (K4: vector / tc by grouped starts)
unsigned vec_rows_grid();
// walk kernels: blocks for a batch of `count` jumpers (one tally part each)
unsigned vec_walk_blocks(uint64_t count);
// returns the number of kernels launched (root + tree levels)
int launch_start_counts(uint64_t n, uint64_t M, const double* cum, const PhiloxKeys& K,
                        uint64_t* cnt, cudaStream_t s);
void launch_vec_rows(const DevSplit& m, const uint64_t* cnt, const FastParams& p, double v_sum,
                     uint64_t lo, uint64_t hi, double* values, uint64_t* jcount, double2* rowc, double* part_s1,
                     double* part_s2, cudaStream_t s);
size_t scan_u64_temp_bytes(uint64_t count);
void launch_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, void* temp,
                     size_t temp_bytes, cudaStream_t s);
void launch_expand_rows(const uint64_t* off, uint64_t n, uint64_t q0, uint64_t q1,
                        uint32_t* row_of, cudaStream_t s);
void launch_vec_walk(const DevSplit& m, const double2* rowc, const uint32_t* row_of,
                     const FastParams& p, double v_sum, uint64_t q0, uint64_t q1,
                     uint32_t* out_end, double* out_f, unsigned long long* acc,
                     double scale_hi, double* part_s1, double* part_s2,
                     unsigned long long* part_j, cudaStream_t s);
void launch_fixed_to_values(const unsigned long long* acc, uint64_t n, double inv_scale,
                            double* values, cudaStream_t s);
// large-W entry path (samples >= 2^29)
void launch_entry_big_rows(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                           const FastParams& p, uint64_t* jcount, double2* rowc, double* Kr,
                           double* s1, double* s2, unsigned long long* jumps, cudaStream_t s);
void launch_entry_big_walk(const DevSplit& m, const uint32_t* rows, const double2* rowc,
                           const double* Kr, const uint32_t* row_of, const uint64_t* off,
                           const FastParams& p, uint64_t q0, uint64_t q1, double* dev1,
                           double* dev2, unsigned long long* jumps, cudaStream_t s);
void launch_entry_big_finalize(uint64_t nrows, uint64_t W, const double* Kr, const double* s1,
                               const double* s2, const unsigned long long* jumps, double* value,
                               double* se, uint64_t* out_jumps, cudaStream_t s);
// per-run sums of already sorted keys (scatter_sort.cu): out[key] += Σ run
size_t run_sums_temp_bytes(uint64_t count);
void run_sums_sorted(const uint32_t* keys, const double* vals, uint64_t count, void* temp,
                     size_t temp_bytes, double* out, cudaStream_t s);
void launch_binomial_debug(uint64_t n, double p, uint64_t count, const PhiloxKeys& K,
                           uint64_t* out, cudaStream_t s);

// reduce.cu
void launch_final_reduce(const double* part_a, const double* part_b,
                         const unsigned long long* part_c, unsigned nparts, double* out_a,
                         double* out_b, unsigned long long* out_c, cudaStream_t s);
// same, added to the running totals out_* (deterministic: launch order)
void launch_final_reduce_acc(const double* part_a, const double* part_b,
                             const unsigned long long* part_c, unsigned nparts, double* out_a,
                             double* out_b, unsigned long long* out_c, cudaStream_t s);
void launch_scale(uint64_t n, double* x, double alpha, cudaStream_t s);
void launch_count_nonfinite(uint64_t n, const double* x, unsigned int* flag, cudaStream_t s);
void launch_sum_u64(uint64_t n, const uint64_t* x, unsigned long long* out, cudaStream_t s);

// expmv.cu (K5)
void launch_spmv(const DevSplit& m, int mode, double shift, const double* x, double* y,
                 cudaStream_t s);
void launch_axpy(uint64_t n, double a, const double* x, double* y, cudaStream_t s);
void launch_scale_diag(uint64_t n, const double* d, double scale, double* x, cudaStream_t s);
void launch_norm_inf(uint64_t n, const double* x, double* part, unsigned nparts, cudaStream_t s);
unsigned norm_parts();
void launch_dot2(uint64_t n, const double* x, const double* y, double* pa, double* pb,
                 unsigned long long* pc, unsigned nparts, cudaStream_t s);

}  // namespace expmc_b200
