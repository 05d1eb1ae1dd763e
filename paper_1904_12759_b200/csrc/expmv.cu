// K5: deterministic fp64 sparse building blocks for the accuracy leg
// (SURVEY §8c iii): y = A x through the splitting (apply_matrix,
// proj/src/sparse_matrix.cpp:163-174 in the reference listing) or y = -L x,
// used by the host driver's scaled Taylor exp(tA)v and the splitting
// product (e^{ΔtD/2} e^{-ΔtL} e^{ΔtD/2})^N v.  One warp per row, fixed
// in-row order + xor tree: deterministic.
#include "kernels.cuh"

namespace expmc_b200 {

namespace {

// mode 0: y = A x + shift x   (A = diag + off-diagonal weights)
// mode 1: y = -L x + shift x  (-L = -rate on the diagonal + weights)
__global__ void __launch_bounds__(256)
spmv_kernel(uint64_t n, const uint64_t* __restrict__ row_offset,
            const uint32_t* __restrict__ nbr, const double* __restrict__ w,
            const double* __restrict__ diag, const double* __restrict__ rate, int mode,
            double shift, const double* __restrict__ x, double* __restrict__ y) {
    const uint64_t row = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const uint64_t lo = row_offset[row], hi = row_offset[row + 1];
    double acc = 0.0;
    for (uint64_t k = lo + lane; k < hi; k += 32)
        acc = __fma_rn(__ldg(w + k), __ldg(x + __ldg(nbr + k)), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) {
        const double dii = mode == 0 ? diag[row] : -rate[row];
        y[row] = __fma_rn(__dadd_rn(dii, shift), x[row], acc);
    }
}

__global__ void axpy_kernel(uint64_t n, double a, const double* __restrict__ x,
                            double* __restrict__ y) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) y[i] = __fma_rn(a, x[i], y[i]);
}

__global__ void scale_diag_kernel(uint64_t n, const double* __restrict__ d, double scale,
                                  double* __restrict__ x) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = __dmul_rn(x[i], exp(__dmul_rn(scale, d[i])));
}

__global__ void __launch_bounds__(256)
norm_inf_kernel(uint64_t n, const double* __restrict__ x, double* __restrict__ part) {
    __shared__ double s[256];
    double m = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(x[i]));
    s[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

// per-block partials of (x . y, y . y); fixed grid -> deterministic
__global__ void __launch_bounds__(256)
dot2_kernel(uint64_t n, const double* __restrict__ x, const double* __restrict__ y,
            double* __restrict__ pa, double* __restrict__ pb, unsigned long long* __restrict__ pc) {
    __shared__ double sa[256], sb[256];
    double a = 0.0, b = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        a = __fma_rn(x[i], y[i], a);
        b = __fma_rn(y[i], y[i], b);
    }
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sa[threadIdx.x] = __dadd_rn(sa[threadIdx.x], sa[threadIdx.x + o]);
            sb[threadIdx.x] = __dadd_rn(sb[threadIdx.x], sb[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pa[blockIdx.x] = sa[0];
        pb[blockIdx.x] = sb[0];
        pc[blockIdx.x] = 0;
    }
}

}  // namespace

void launch_dot2(uint64_t n, const double* x, const double* y, double* pa, double* pb,
                 unsigned long long* pc, unsigned nparts, cudaStream_t s) {
    dot2_kernel<<<nparts, 256, 0, s>>>(n, x, y, pa, pb, pc);
}

void launch_spmv(const DevSplit& m, int mode, double shift, const double* x, double* y,
                 cudaStream_t s) {
    if (m.n == 0) return;
    const uint64_t threads = m.n * 32;
    spmv_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
        m.n, m.row_offset, m.neighbor, m.weight, m.diag, m.rate, mode, shift, x, y);
}

void launch_axpy(uint64_t n, double a, const double* x, double* y, cudaStream_t s) {
    if (n == 0) return;
    axpy_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, a, x, y);
}

void launch_scale_diag(uint64_t n, const double* d, double scale, double* x, cudaStream_t s) {
    if (n == 0) return;
    scale_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, d, scale, x);
}

unsigned norm_parts() { return 148 * 2; }

void launch_norm_inf(uint64_t n, const double* x, double* part, unsigned nparts,
                     cudaStream_t s) {
    norm_inf_kernel<<<nparts, 256, 0, s>>>(n, x, part);
}

}  // namespace expmc_b200
