// Deterministic final reductions over per-block partials (fixed shape:
// one 256-thread block, thread t sums parts t, t+256, ... in order, then a
// fixed tree), plus small elementwise helpers.
#include "kernels.cuh"

namespace expmc_b200 {

namespace {

__global__ void __launch_bounds__(256)
final_reduce_kernel(const double* __restrict__ a, const double* __restrict__ b,
                    const unsigned long long* __restrict__ c, unsigned nparts,
                    double* __restrict__ oa, double* __restrict__ ob,
                    unsigned long long* __restrict__ oc, bool accumulate) {
    __shared__ double sa[256], sb[256];
    __shared__ unsigned long long sc[256];
    double x = 0.0, y = 0.0;
    unsigned long long z = 0;
    for (unsigned k = threadIdx.x; k < nparts; k += 256) {
        x = __dadd_rn(x, a[k]);
        y = __dadd_rn(y, b[k]);
        z += c[k];
    }
    sa[threadIdx.x] = x;
    sb[threadIdx.x] = y;
    sc[threadIdx.x] = z;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sa[threadIdx.x] = __dadd_rn(sa[threadIdx.x], sa[threadIdx.x + o]);
            sb[threadIdx.x] = __dadd_rn(sb[threadIdx.x], sb[threadIdx.x + o]);
            sc[threadIdx.x] += sc[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {  // accumulate: running totals added in launch order
        *oa = accumulate ? __dadd_rn(*oa, sa[0]) : sa[0];
        *ob = accumulate ? __dadd_rn(*ob, sb[0]) : sb[0];
        *oc = accumulate ? *oc + sc[0] : sc[0];
    }
}

__global__ void scale_kernel(uint64_t n, double* __restrict__ x, double alpha) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = __dmul_rn(x[i], alpha);
}

__global__ void nonfinite_kernel(uint64_t n, const double* __restrict__ x,
                                 unsigned int* __restrict__ flag) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool bad = i < n && !isfinite(x[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace

// *out += sum of x[0..n) (integer: exact and order-independent)
__global__ void sum_u64_kernel(const uint64_t* __restrict__ x, uint64_t n,
                               unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x)
        acc += x[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

void launch_sum_u64(uint64_t n, const uint64_t* x, unsigned long long* out, cudaStream_t s) {
    if (!n) return;
    const uint64_t want = (n + 255) / 256;
    const unsigned grid = (unsigned)(want < 148 * 8 ? want : 148 * 8);
    sum_u64_kernel<<<grid, 256, 0, s>>>(x, n, out);
}

void launch_count_nonfinite(uint64_t n, const double* x, unsigned int* flag, cudaStream_t s) {
    if (n == 0) return;
    nonfinite_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, x, flag);
}

void launch_final_reduce(const double* part_a, const double* part_b,
                         const unsigned long long* part_c, unsigned nparts, double* out_a,
                         double* out_b, unsigned long long* out_c, cudaStream_t s) {
    final_reduce_kernel<<<1, 256, 0, s>>>(part_a, part_b, part_c, nparts, out_a, out_b, out_c,
                                          false);
}

void launch_final_reduce_acc(const double* part_a, const double* part_b,
                             const unsigned long long* part_c, unsigned nparts, double* out_a,
                             double* out_b, unsigned long long* out_c, cudaStream_t s) {
    final_reduce_kernel<<<1, 256, 0, s>>>(part_a, part_b, part_c, nparts, out_a, out_b, out_c,
                                          true);
}

void launch_scale(uint64_t n, double* x, double alpha, cudaStream_t s) {
    if (n == 0) return;
    scale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, x, alpha);
}

}  // namespace expmc_b200
