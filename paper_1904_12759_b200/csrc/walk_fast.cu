// K6 gather_ceiling: the same-pattern random-gather roofline of the entry
// walker (K4, the Theorem-2 estimators, lives in walk_vec.cu).
#include "kernels.cuh"

namespace expmc_b200 {

namespace {

constexpr uint32_t kChainsPerThread = 16;

// K6: memory-only walker with the K3 access pattern (neighbour id gather ->
// landing record gather) and a cheap integer hash instead of Philox / log /
// exp.  chains_per_row chains of chain_len jumps start at every listed row;
// consecutive lanes walk chains of the same row, as in K3.  Its jumps/s is
// the same-pattern random-gather ceiling for the roofline.
__global__ void __launch_bounds__(128)
gather_ceiling_kernel(const RowRec* __restrict__ rec, const Edge* __restrict__ adj,
                      const uint32_t* __restrict__ rows, uint64_t nrows,
                      uint32_t chains_per_row, uint32_t chain_len, uint32_t salt,
                      unsigned long long* __restrict__ sink) {
    const uint64_t total = nrows * (uint64_t)chains_per_row;
    // block-owned chain ranges (many small blocks, balanced by the hardware
    // block scheduler — the same work distribution as the K3/K4 walkers)
    const uint64_t base = blockIdx.x * (uint64_t)blockDim.x * kChainsPerThread;
    const uint64_t end = base + (uint64_t)blockDim.x * kChainsPerThread < total
                             ? base + (uint64_t)blockDim.x * kChainsPerThread : total;
    unsigned long long acc = 0;
    for (uint64_t c = base + threadIdx.x; c < end; c += blockDim.x) {
        uint32_t cur = rows[c / chains_per_row];
        const RowRec r = load_rec(rec, cur);  // start record, as K3
        uint32_t off = r.off, degf = r.deg_flags;
        uint32_t h = (uint32_t)c * 0x9E3779B9u ^ salt;
        double dsum = r.d;
        for (uint32_t k = 0; k < chain_len; ++k) {
            h ^= h << 13; h ^= h >> 17; h ^= h << 5;
            const uint32_t deg = degf & kDegMask;
            if (deg == 0) break;
            // one sector per jump, with the walkers' load policy (ld256_gather)
#ifdef K6_PLAIN_LD
            const Edge e = load_edge(adj, off + __umulhi(h, deg));
            cur = e.j; off = e.off; degf = e.deg_flags; dsum += e.d;
#else
            unsigned long long ea, eb, ec, ed;
            ld256_gather(adj + (off + __umulhi(h, deg)), ea, eb, ec, ed);
            cur = (uint32_t)ea; off = (uint32_t)(ea >> 32); degf = (uint32_t)eb;
            dsum += __longlong_as_double((long long)ec);
            (void)ed;
#endif
        }
        acc += cur + (dsum == 0.5 ? 1 : 0);
    }
    if (acc == 0x7fffffffffffffffull) *sink = acc;  // keep the loads live
}

// Law check of the walkers' Exp(1) transform (test hook): 4 count Philox
// words (counters (k, 0, 0, 'LAWS')) through neg_ln_u, histogrammed in bins
// of `width` (the last bin collects the rest) with the raw sum and sum of
// squares (integer atomics: exact, order-independent).
__global__ void exp_law_kernel(uint64_t blocks, PhiloxKeys K, double width, uint32_t nbins,
                               unsigned long long* __restrict__ hist,
                               unsigned long long* __restrict__ mom) {
    extern __shared__ unsigned int sh[];  // per-block histogram (u32: < 2^32 per block)
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) sh[b] = 0u;
    __syncthreads();
    unsigned long long s1 = 0, s2 = 0;  // sums of E and E^2 in 2^-30 units
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < blocks;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const U4 w = philox4x32_10(U4{(uint32_t)k, (uint32_t)(k >> 32), 0u, 0x4c415753u}, K);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float E = neg_ln_u(ws[q]);
            uint32_t b = (uint32_t)((double)E / width);
            b = b < nbins - 1 ? b : nbins - 1;
            atomicAdd(sh + b, 1u);
            s1 += (unsigned long long)((double)E * 1073741824.0);
            s2 += (unsigned long long)((double)E * (double)E * 1073741824.0);
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x)
        if (sh[b]) atomicAdd(hist + b, (unsigned long long)sh[b]);
    atomicAdd(mom, s1);
    atomicAdd(mom + 1, s2);
}

}  // namespace

void launch_exp_law(uint64_t count, uint64_t seed, double width, uint32_t nbins,
                    unsigned long long* hist, unsigned long long* mom, cudaStream_t s) {
    const uint64_t blocks = count / 4;
    const PhiloxKeys K = philox_keys((uint32_t)seed, (uint32_t)(seed >> 32));
    exp_law_kernel<<<148 * 8, 256, nbins * sizeof(unsigned int), s>>>(blocks, K, width, nbins,
                                                                    hist, mom);
}

void launch_gather_ceiling(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                           uint32_t chains_per_row, uint32_t chain_len, uint32_t salt,
                           unsigned long long* sink, cudaStream_t s) {
    if (nrows == 0 || chains_per_row == 0) return;
    const uint64_t total = nrows * (uint64_t)chains_per_row;
    const uint64_t blocks = (total + 128ull * kChainsPerThread - 1) / (128ull * kChainsPerThread);
    gather_ceiling_kernel<<<(unsigned)blocks, 128, 0, s>>>(m.rec, m.adj, rows, nrows,
                                                          chains_per_row, chain_len, salt, sink);
}

}  // namespace expmc_b200
