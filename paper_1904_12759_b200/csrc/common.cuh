// Shared device-side definitions for the B200 Monte Carlo exp(tA)v hot path.
//
// Reference behaviour restated here (never copied):
//   PCG32 XSH-RR stream          proj/include/expmc/rng.hpp:14-63
//   exp_time / jump / advance    proj/src/sampler.cpp:10-49
//   SplitMatrix layout           proj/include/expmc/sparse_matrix.hpp:66-91
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace expmc_b200 {

// ----------------------------------------------------------------- layout
// One 32-byte row record (one L2 sector): everything a walker needs when it
// lands on a row.  Built by split_pack (K1); `v` is refreshed per call by
// pack_v so the terminal score costs no extra gather.
struct __align__(32) RowRec {
    uint32_t off;       // CSR offset of the row in neighbor[]
    uint32_t deg_flags; // bits 0..30 degree, bit 31 = non-uniform row
    float inv_rate;     // (float)(1.0 / rate), +inf for isolated rows
    uint32_t spare;
    double d;           // D_ii = A_ii + rate_i
    double v;           // v_i for the current call
};
static_assert(sizeof(RowRec) == 32, "RowRec must be one sector");

constexpr uint32_t kNonUniform = 0x80000000u;
constexpr uint32_t kDegMask = 0x7fffffffu;

// ------------------------------------------------------------------ PCG32
// Bit-exact replay of RngStream (rng.hpp:14-63) for the parity kernels.
struct Pcg32 {
    uint64_t state, inc;
    __device__ __forceinline__ Pcg32(uint64_t seed, uint64_t stream)
        : state(0u), inc((stream << 1u) | 1u) {
        next_u32();
        state += seed;
        next_u32();
    }
    __device__ __forceinline__ uint32_t next_u32() {
        const uint64_t old = state;
        state = old * 6364136223846793005ULL + inc;
        const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
        const uint32_t rot = (uint32_t)(old >> 59u);
        return __funnelshift_r(xs, xs, rot);  // rotate right
    }
    __device__ __forceinline__ uint64_t next_u64() {
        const uint64_t hi = next_u32();
        return (hi << 32) | next_u32();
    }
    __device__ __forceinline__ double uniform() {
        return __dmul_rn((double)(next_u64() >> 11), 0x1.0p-53);
    }
    __device__ __forceinline__ double uniform_pos() {
        return __dmul_rn((double)((next_u64() >> 11) + 1), 0x1.0p-53);
    }
    __device__ __forceinline__ uint64_t uniform_index(uint64_t n) {
        const uint64_t k = (uint64_t)__dmul_rn(uniform(), (double)n);
        return k < n ? k : n - 1;
    }
};

// ---------------------------------------------------------- Philox4x32-10
// Counter-based generator (Salmon et al., SC'11).  Keyed by the user seed;
// the counter encodes (sojourn step, walker, row, estimator tag) so every
// walker's stream is a pure function of (seed, row, walker) — independent of
// the launch configuration and of how rows are sharded over GPUs.
struct U4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

constexpr uint32_t kTagEntry = 0x454e5452u;  // 'ENTR'
constexpr uint32_t kTagScatter = 0x56454354u; // 'VECT' (vector / tc)

// -ln(u) for u = ((w >> 9) + 0.5) * 2^-23 in (0, 1), fp32, using only
// IEEE-exact operations (fma, div) so the CPU model in oracle/fast_model.c
// reproduces it bit for bit.  ln(m) = 2 atanh(s), s = (m-1)/(m+1),
// m in [sqrt(1/2), sqrt(2)); |s| <= 0.1716, series to s^9 (rel. err < 3e-9).
__device__ __forceinline__ float neg_ln_u(uint32_t w) {
    const float u = __fmul_rn(__uint2float_rn(w >> 9) + 0.5f, 0x1.0p-23f);
    int e;
    uint32_t bits = __float_as_uint(u);
    e = (int)((bits >> 23) & 0xffu) - 127;
    float m = __uint_as_float((bits & 0x007fffffu) | 0x3f800000u);  // [1,2)
    if (m > 1.41421356f) {
        m = __fmul_rn(m, 0.5f);
        e += 1;
    }
    const float s = __fdiv_rn(__fsub_rn(m, 1.0f), __fadd_rn(m, 1.0f));
    const float z = __fmul_rn(s, s);
    float p = __fmaf_rn(z, 0.11111111f, 0.14285715f);
    p = __fmaf_rn(z, p, 0.2f);
    p = __fmaf_rn(z, p, 0.33333334f);
    p = __fmaf_rn(z, p, 1.0f);
    const float lnm = __fmul_rn(__fmul_rn(2.0f, s), p);
    const float ln_u = __fmaf_rn((float)e, 0.693147182f, lnm);
    return -ln_u;
}

// floor(x * n / 2^64) for a 64-bit uniform x: unbiased to n / 2^64.
__device__ __forceinline__ uint32_t pick_index(uint32_t hi, uint32_t lo,
                                               uint32_t n) {
    const uint64_t x = ((uint64_t)hi << 32) | lo;
    return (uint32_t)__umul64hi(x, (uint64_t)n);
}

}  // namespace expmc_b200
