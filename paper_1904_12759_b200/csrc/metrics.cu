// §8f row f4: rank / isim on the device (reference: proj/src/metrics.cpp).
//
// rank (metrics.cpp:10-25): descending scores, ties by ascending index,
// NaN rejected.  Scores map to 64-bit keys whose ascending order is the
// descending order of the scores (-0.0 folded onto +0.0, which compare
// equal in the reference); a stable radix sort of (key, index) keeps
// ascending indices inside ties.  Integer work: identical to std::sort's
// result (the comparator is a strict total order on (score, index)).
//
// isim (metrics.cpp:27-55): with 0-based positions, node e is in both top-i
// prefixes iff max(posX[e], posY[e]) < i, so common(i) is a prefix sum of
// the histogram of m(e) = max(posX[e], posY[e]) over e in X's top K, and
// isim = (1/K) sum_{i=1..K} (i - common(i)) / i — every term exact as in the
// reference; the sum is a fixed-shape reduction (deterministic).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "kernels.cuh"

namespace expmc_b200 {

namespace {

inline unsigned blocks(uint64_t x) { return (unsigned)((x + 255) / 256); }

__global__ void rank_keys_kernel(const double* __restrict__ s, uint64_t n,
                                 unsigned long long* __restrict__ key,
                                 uint32_t* __restrict__ idx, unsigned int* __restrict__ nan_flag) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x = s[i];
    if (x != x) atomicOr(nan_flag, 1u);
    if (x == 0.0) x = 0.0;  // -0.0 == +0.0 in the reference comparator
    unsigned long long u = (unsigned long long)__double_as_longlong(x);
    u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);  // ascending in x
    key[i] = ~u;                                       // descending in x
    idx[i] = (uint32_t)i;
}

__global__ void scatter_pos_kernel(const uint32_t* __restrict__ order, uint64_t n,
                                   uint32_t* __restrict__ pos) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) pos[order[i]] = (uint32_t)i;
}

__global__ void hist_kernel(const uint32_t* __restrict__ ox, const uint32_t* __restrict__ posy,
                            uint64_t k, unsigned int* __restrict__ hist) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= k) return;
    const uint64_t py = posy[ox[i]];
    const uint64_t m = i > py ? i : py;
    if (m < k) atomicAdd(hist + m, 1u);
}

// partials of sum_{i=1..k} (i - common(i)) / i, common(i) = cum[i-1]
__global__ void __launch_bounds__(256)
isim_terms_kernel(const unsigned long long* __restrict__ cum, uint64_t k,
                  double* __restrict__ part_a, double* __restrict__ part_b,
                  unsigned long long* __restrict__ part_c) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1; i <= k;
         i += (uint64_t)gridDim.x * blockDim.x)
        acc = __dadd_rn(acc, __ddiv_rn((double)(i - cum[i - 1]), (double)i));
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part_a[blockIdx.x] = sh[0];
        part_b[blockIdx.x] = 0.0;
        part_c[blockIdx.x] = 0;
    }
}

__global__ void u32_to_u64_kernel(const unsigned int* __restrict__ a, uint64_t n,
                                  unsigned long long* __restrict__ b) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}

struct Scratch {
    void* p[8] = {};
    ~Scratch() {
        for (void* q : p) cudaFree(q);
    }
};

}  // namespace

// returns false if a NaN score was found (order not written)
bool rank_device(const double* scores_host, uint64_t n, uint32_t* order_host, cudaStream_t s) {
    if (n == 0) return true;
    Scratch sc;
    double* sd;
    unsigned long long *k1, *k2;
    uint32_t *i1, *i2;
    unsigned int* flag;
    cudaMalloc(&sd, n * 8); sc.p[0] = sd;
    cudaMalloc(&k1, n * 8); sc.p[1] = k1;
    cudaMalloc(&k2, n * 8); sc.p[2] = k2;
    cudaMalloc(&i1, n * 4); sc.p[3] = i1;
    cudaMalloc(&i2, n * 4); sc.p[4] = i2;
    cudaMalloc(&flag, 4); sc.p[5] = flag;
    cudaMemsetAsync(flag, 0, 4, s);
    cudaMemcpyAsync(sd, scores_host, n * 8, cudaMemcpyHostToDevice, s);
    rank_keys_kernel<<<blocks(n), 256, 0, s>>>(sd, n, k1, i1, flag);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k2, i1, i2, (int)n, 0, 64, s);
    void* tmp;
    cudaMalloc(&tmp, tb); sc.p[6] = tmp;
    cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k2, i1, i2, (int)n, 0, 64, s);
    unsigned int bad = 0;
    cudaMemcpyAsync(&bad, flag, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(order_host, i2, n * 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return bad == 0;
}

double isim_device(const uint32_t* ox_host, const uint32_t* oy_host, uint64_t n, uint64_t k,
                   cudaStream_t s) {
    Scratch sc;
    uint32_t *ox, *oy, *posy;
    unsigned int* hist;
    unsigned long long *h64, *cum;
    cudaMalloc(&ox, n * 4); sc.p[0] = ox;
    cudaMalloc(&oy, n * 4); sc.p[1] = oy;
    cudaMalloc(&posy, n * 4); sc.p[2] = posy;
    cudaMalloc(&hist, k * 4); sc.p[3] = hist;
    cudaMalloc(&h64, k * 8); sc.p[4] = h64;
    cudaMalloc(&cum, k * 8); sc.p[5] = cum;
    cudaMemcpyAsync(ox, ox_host, n * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(oy, oy_host, n * 4, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(hist, 0, k * 4, s);
    scatter_pos_kernel<<<blocks(n), 256, 0, s>>>(oy, n, posy);
    hist_kernel<<<blocks(k), 256, 0, s>>>(ox, posy, k, hist);
    u32_to_u64_kernel<<<blocks(k), 256, 0, s>>>(hist, k, h64);
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, h64, cum, (int)k, s);
    void* tmp;
    cudaMalloc(&tmp, tb); sc.p[6] = tmp;
    cub::DeviceScan::InclusiveSum(tmp, tb, h64, cum, (int)k, s);
    const unsigned parts = 148 * 2;
    double* pa;
    cudaMalloc(&pa, parts * 24 + 64); sc.p[7] = pa;
    double* pb = pa + parts;
    unsigned long long* pc = reinterpret_cast<unsigned long long*>(pa + 2 * parts);
    isim_terms_kernel<<<parts, 256, 0, s>>>(cum, k, pa, pb, pc);
    double* tot = pa + 3 * parts;
    launch_final_reduce(pa, pb, pc, parts, tot, tot + 1,
                        reinterpret_cast<unsigned long long*>(tot + 2), s);
    double sum = 0.0;
    cudaMemcpyAsync(&sum, tot, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return sum / (double)k;
}

}  // namespace expmc_b200
