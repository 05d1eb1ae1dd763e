// K2 walk_compat: path-by-path replay of the reference estimators on the GPU.
//
// Every walker l owns PCG32 stream (seed, l) exactly like the reference
// (proj/src/estimator.cpp:188, :242, :299) and performs the reference's
// per-segment algorithm: fresh exponential clock per Δt segment
// (proj/src/sampler.cpp:36-49), jump by degree scaling or by upper_bound over
// the cumulative row weights (:18-34), before/after node factors
// (proj/src/estimator.cpp:26-39).  Outcomes (end state, jumps, weight) match
// the CPU reference walker for walker; only the order in which the per-entry
// sums are added differs (fixed tree here, sequential there).
//
// This is the parity kernel.  The production kernel is walk_fast.cu (K3).
#include "kernels.cuh"

namespace expmc_b200 {

namespace {

struct SoA {
    const double* rate;
    const uint64_t* row_offset;
    const uint32_t* neighbor;
    const double* cum;
    const uint8_t* uniform_row;
};

__device__ __forceinline__ double exp_time(Pcg32& rng, double rate) {
    // sampler.cpp:10-16; rate 0 -> +inf without consuming the stream
    if (rate == 0.0) return __longlong_as_double(0x7ff0000000000000LL);
    return __ddiv_rn(-log(rng.uniform_pos()), rate);
}

__device__ __forceinline__ uint32_t jump(Pcg32& rng, const SoA& m, uint32_t i) {
    // sampler.cpp:18-34
    const uint64_t lo = m.row_offset[i];
    const uint64_t deg = m.row_offset[i + 1] - lo;
    if (m.uniform_row[i]) return m.neighbor[lo + rng.uniform_index(deg)];
    const double target = __dmul_rn(rng.uniform(), m.rate[i]);
    uint64_t a = 0, b = deg;
    while (a < b) {  // std::upper_bound
        const uint64_t mid = a + (b - a) / 2;
        if (target < m.cum[lo + mid]) b = mid; else a = mid + 1;
    }
    if (a == deg) --a;
    return m.neighbor[lo + a];
}

__device__ __forceinline__ double run_path(Pcg32& rng, const SoA& m, uint32_t start,
                                           double dt, uint64_t n_steps,
                                           const double* before, const double* after,
                                           uint32_t& end, uint64_t& jumps) {
    // estimator.cpp:26-39 with advance() (sampler.cpp:36-49) inlined
    double w = 1.0;
    uint32_t s = start;
    for (uint64_t k = 0; k < n_steps; ++k) {
        if (before) w = __dmul_rn(w, before[s]);
        double tau = exp_time(rng, m.rate[s]);
        while (tau < dt) {
            s = jump(rng, m, s);
            ++jumps;
            tau = __dadd_rn(tau, exp_time(rng, m.rate[s]));
        }
        if (after) w = __dmul_rn(w, after[s]);
    }
    end = s;
    return w;
}

template <int BS>
__device__ __forceinline__ void block_sum3(double& a, double& b, unsigned long long& c,
                                           double* sa, double* sb, unsigned long long* sc) {
    // fixed-shape tree: deterministic for a given block size
    const int t = threadIdx.x;
    sa[t] = a;
    sb[t] = b;
    sc[t] = c;
    __syncthreads();
#pragma unroll
    for (int o = BS / 2; o > 0; o >>= 1) {
        if (t < o) {
            sa[t] = __dadd_rn(sa[t], sa[t + o]);
            sb[t] = __dadd_rn(sb[t], sb[t + o]);
            sc[t] += sc[t + o];
        }
        __syncthreads();
    }
    a = sa[0];
    b = sb[0];
    c = sc[0];
}

constexpr int kCompatBS = 128;

// Entry estimator (Theorem 1), one block per requested row.
__global__ void __launch_bounds__(kCompatBS)
entry_compat_kernel(SoA m, const double* __restrict__ v, const uint32_t* __restrict__ rows,
                    uint64_t nrows, double dt, uint64_t n_steps, uint64_t samples,
                    const double* __restrict__ before, const double* __restrict__ after,
                    uint64_t seed, double* __restrict__ out_value, double* __restrict__ out_se,
                    uint64_t* __restrict__ out_jumps) {
    __shared__ double sa[kCompatBS], sb[kCompatBS];
    __shared__ unsigned long long sc[kCompatBS];
    for (uint64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
        const uint32_t i = rows[r];
        double sum = 0.0, sum_sq = 0.0;
        unsigned long long jumps = 0;
        for (uint64_t l = threadIdx.x; l < samples; l += kCompatBS) {
            Pcg32 rng(seed, l);
            uint32_t end;
            uint64_t j = 0;
            const double w = run_path(rng, m, i, dt, n_steps, before, after, end, j);
            const double f = __dmul_rn(w, v[end]);
            sum = __dadd_rn(sum, f);
            sum_sq = __dadd_rn(sum_sq, __dmul_rn(f, f));
            jumps += j;
        }
        block_sum3<kCompatBS>(sum, sum_sq, jumps, sa, sb, sc);
        if (threadIdx.x == 0) {
            // finalize: estimator.cpp:76-89
            const double mm = (double)samples;
            out_value[r] = __ddiv_rn(sum, mm);
            double se = 0.0;
            if (samples > 1) {
                double var = __ddiv_rn(__dsub_rn(sum_sq, __ddiv_rn(__dmul_rn(sum, sum), mm)),
                                       __dsub_rn(mm, 1.0));
                var = var > 0.0 ? var : 0.0;
                se = sqrt(__ddiv_rn(var, mm));
            }
            out_se[r] = se;
            out_jumps[r] = jumps;
        }
        __syncthreads();
    }
}

// Vector / TC estimators (Theorem 2): grid-stride over walkers.
//   start_mode 0: uniform index (tc, or vector with constant v)
//   start_mode 1: categorical v / V through the host-built cumulative table
//                 (StartSampler, estimator.cpp:92-128)
__global__ void __launch_bounds__(kCompatBS)
scatter_compat_kernel(SoA m, uint64_t n, int start_mode, const double* __restrict__ vcum,
                      double v_sum, double dt, uint64_t n_steps, uint64_t samples,
                      const double* __restrict__ before, const double* __restrict__ after,
                      uint64_t seed, uint64_t l0, uint64_t lend, uint32_t* __restrict__ out_end,
                      double* __restrict__ out_f, double* __restrict__ part_sum,
                      double* __restrict__ part_sq, unsigned long long* __restrict__ part_j) {
    __shared__ double sa[kCompatBS], sb[kCompatBS];
    __shared__ unsigned long long sc[kCompatBS];
    double sum = 0.0, sum_sq = 0.0;
    unsigned long long jumps = 0;
    const uint64_t stride = (uint64_t)gridDim.x * kCompatBS;
    for (uint64_t l = l0 + blockIdx.x * (uint64_t)kCompatBS + threadIdx.x; l < lend; l += stride) {
        Pcg32 rng(seed, l);
        uint32_t start;
        if (start_mode == 0) {
            start = (uint32_t)rng.uniform_index(n);
        } else {
            const double target = __dmul_rn(rng.uniform(), v_sum);
            uint64_t a = 0, b = n;
            while (a < b) {
                const uint64_t mid = a + (b - a) / 2;
                if (target < vcum[mid]) b = mid; else a = mid + 1;
            }
            if (a == n) --a;
            start = (uint32_t)a;
        }
        uint32_t end;
        uint64_t j = 0;
        const double w = run_path(rng, m, start, dt, n_steps, before, after, end, j);
        const double f = __dmul_rn(v_sum, w);
        sum = __dadd_rn(sum, f);
        sum_sq = __dadd_rn(sum_sq, __dmul_rn(f, f));
        jumps += j;
        if (out_end) {  // (end, f) record for the deterministic per-end reduction
            out_end[l - l0] = end;
            out_f[l - l0] = f;
        }
    }
    block_sum3<kCompatBS>(sum, sum_sq, jumps, sa, sb, sc);
    if (threadIdx.x == 0) {
        part_sum[blockIdx.x] = sum;
        part_sq[blockIdx.x] = sum_sq;
        part_j[blockIdx.x] = jumps;
    }
}

}  // namespace

void launch_entry_compat(const DevSplit& m, const double* v, const uint32_t* rows,
                         uint64_t nrows, double dt, uint64_t n_steps, uint64_t samples,
                         const double* before, const double* after, uint64_t seed,
                         double* value, double* se, uint64_t* jumps, cudaStream_t s) {
    if (nrows == 0) return;
    SoA a{m.rate, m.row_offset, m.neighbor, m.cum, m.uniform_row};
    const uint64_t grid = nrows < 1184 * 16 ? nrows : 1184 * 16;
    entry_compat_kernel<<<(unsigned)grid, kCompatBS, 0, s>>>(a, v, rows, nrows, dt, n_steps,
                                                             samples, before, after, seed,
                                                             value, se, jumps);
}

unsigned scatter_compat_grid() { return 148 * 8; }

void launch_scatter_compat(const DevSplit& m, int start_mode, const double* vcum, double v_sum,
                           double dt, uint64_t n_steps, uint64_t samples, const double* before,
                           const double* after, uint64_t seed, uint64_t l0, uint64_t lend,
                           uint32_t* out_end, double* out_f, double* part_sum, double* part_sq,
                           unsigned long long* part_j, cudaStream_t s) {
    SoA a{m.rate, m.row_offset, m.neighbor, m.cum, m.uniform_row};
    scatter_compat_kernel<<<scatter_compat_grid(), kCompatBS, 0, s>>>(
        a, m.n, start_mode, vcum, v_sum, dt, n_steps, samples, before, after, seed, l0, lend,
        out_end, out_f, part_sum, part_sq, part_j);
}

}  // namespace expmc_b200
