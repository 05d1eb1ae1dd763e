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

// One 32-byte "fat" adjacency slot per directed edge (row i, column k):
// everything a walker needs after jumping from i through column k — the
// landing row j with its offset / degree / 1/rate / d and the current
// call's v_j (refreshed by pack_v).  A jump on a uniform row is then ONE
// dependent sector gather instead of neighbour-id -> row-record, and a
// finished walker already holds its terminal score.  Weighted rows read
// their alias entry (thr, alias arrays) first.  Costs nnz * 32 B of HBM
// (5.1 GB for the largest configuration), which the 180 GB part affords.
struct __align__(32) Edge {
    uint32_t j;         // landing row
    uint32_t off;       // its CSR offset
    uint32_t deg_flags; // its degree | non-uniform flag
    float inv_rate;     // its (float)(1/rate)
    double d;           // its D_jj
    double v;           // v_j of the current call
};
static_assert(sizeof(Edge) == 32, "Edge must be one sector");

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

// Same function with a precomputed key schedule (kernel parameter / constant
// bank): identical output, no per-thread registers for the 20 round keys.
struct PhiloxKeys {
    uint32_t k0[10], k1[10];
};

inline PhiloxKeys philox_keys(uint32_t k0, uint32_t k1) {
    PhiloxKeys r;
    for (int i = 0; i < 10; ++i) {
        r.k0[i] = k0;
        r.k1[i] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return r;
}

__device__ __forceinline__ U4 philox4x32_10(U4 c, const PhiloxKeys& K) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ K.k0[r], lo1, hi0 ^ c.w ^ K.k1[r], lo0};
    }
    return c;
}

constexpr uint32_t kTagEntry = 0x454e5452u;  // 'ENTR'
constexpr uint32_t kTagScatter = 0x56454354u; // 'VECT' (vector / tc)

// -ln(u) for u = ((w >> 9) + 0.5) * 2^-23 in (0, 1), fp32, using only
// IEEE-exact operations (mul, sub, fma) so the CPU model in
// oracle/fast_model.c reproduces it bit for bit.  u = 2^e m with
// m in [sqrt(1/2), sqrt(2)); ln(m) = f q(f), f = m - 1 (exact), q a degree-8
// Chebyshev fit of log1p(f)/f on [sqrt(1/2)-1, sqrt(2)-1] (rel. err 2.7e-8).
__device__ __forceinline__ float neg_ln_u(uint32_t w) {
    const float u = __fmul_rn(__uint2float_rn(w >> 9) + 0.5f, 0x1.0p-23f);
    const uint32_t bits = __float_as_uint(u);
    int e = (int)((bits >> 23) & 0xffu) - 127;
    float m = __uint_as_float((bits & 0x007fffffu) | 0x3f800000u);  // [1,2)
    if (m > 1.41421356f) {
        m = __fmul_rn(m, 0.5f);
        e += 1;
    }
    const float f = __fsub_rn(m, 1.0f);
    float q = 0.08743945509195328f;
    q = __fmaf_rn(q, f, -0.14377330243587494f);
    q = __fmaf_rn(q, f, 0.14949095249176025f);
    q = __fmaf_rn(q, f, -0.16560696065425873f);
    q = __fmaf_rn(q, f, 0.19956977665424347f);
    q = __fmaf_rn(q, f, -0.2500215470790863f);
    q = __fmaf_rn(q, f, 0.3333418369293213f);
    q = __fmaf_rn(q, f, -0.49999988079071045f);
    q = __fmaf_rn(q, f, 1.0f);
    const float ln_u = __fmaf_rn((float)e, 0.693147182f, __fmul_rn(f, q));
    return -ln_u;
}

// e^x in fp64 from IEEE-exact operations only (rint, fma, mul), so the CPU
// model (oracle/fast_model.c fm_exp) reproduces it bit for bit: Cody-Waite
// reduction x = n ln2 + r, |r| <= ln2/2, degree-13 Taylor for e^r, exact
// scaling by 2^n.  Max error ~1 ulp on [-745, 709.78]; +inf above, 0 below.
// Coefficients as immediates (UMOV pairs).  Measured: 2% faster on K3 than
// reading them from the constant bank (-DEXP_DET_CONST, kept as a variant).
#ifndef EXP_DET_CONST
#define EXPC(k) (exp_det_lit(k))
__device__ __forceinline__ constexpr double exp_det_lit(int k) {
    return k == 0 ? 1.4426950408889634 : k == 1 ? 6.93147180369123816490e-01
         : k == 2 ? 1.90821492927058770002e-10 : k == 3 ? 1.6059043836821614599e-10
         : k == 4 ? 2.0876756987868098979e-09 : k == 5 ? 2.5052108385441718775e-08
         : k == 6 ? 2.7557319223985890653e-07 : k == 7 ? 2.7557319223985890653e-06
         : k == 8 ? 2.4801587301587301566e-05 : k == 9 ? 1.9841269841269841253e-04
         : k == 10 ? 1.3888888888888889419e-03 : k == 11 ? 8.3333333333333332177e-03
         : k == 12 ? 4.1666666666666664354e-02 : k == 13 ? 1.6666666666666665741e-01
         : k == 14 ? 709.782712893384 : -745.1332191019412;
}
#else
#define EXPC(k) (c_exp_det[k])
#endif
__constant__ double c_exp_det[16] = {
    1.4426950408889634,         // log2(e)
    6.93147180369123816490e-01, // ln2 hi
    1.90821492927058770002e-10, // ln2 lo
    1.6059043836821614599e-10,  // 1/13!
    2.0876756987868098979e-09, 2.5052108385441718775e-08, 2.7557319223985890653e-07,
    2.7557319223985890653e-06, 2.4801587301587301566e-05, 1.9841269841269841253e-04,
    1.3888888888888889419e-03, 8.3333333333333332177e-03, 4.1666666666666664354e-02,
    1.6666666666666665741e-01, 709.782712893384, -745.1332191019412};

__device__ __forceinline__ double exp_det(double x) {
    // branch-free range handling: clamp (NaN passes through: the compares
    // are false), then scale by 2^k as 2^k1 * 2^k2 (k1 = k >> 1), which is
    // exact up to the final rounding for every k in [-1076, 1024]: the same
    // value as one correctly rounded q * 2^k, including overflow to +inf
    // (x >= ln(DBL_MAX)) and underflow to subnormals / 0
    x = x > 710.0 ? 710.0 : x;
    x = x < -746.0 ? -746.0 : x;
    const double n = rint(__dmul_rn(x, EXPC(0)));
    double r = __fma_rn(-n, EXPC(1), x);
    r = __fma_rn(-n, EXPC(2), r);
    double q = EXPC(3);
#pragma unroll
    for (int k = 4; k < 14; ++k) q = __fma_rn(q, r, EXPC(k));
    q = __fma_rn(q, r, 0.5);
    q = __fma_rn(q, r, 1.0);
    q = __fma_rn(q, r, 1.0);
    const int k = __double2int_rn(n);
    const int k1 = k >> 1;
    return __dmul_rn(__dmul_rn(q, __longlong_as_double((long long)(k1 + 1023) << 52)),
                     __longlong_as_double((long long)(k - k1 + 1023) << 52));
}

// floor(x * n / 2^64) for a 64-bit uniform x: unbiased to n / 2^64.
__device__ __forceinline__ uint32_t pick_index(uint32_t hi, uint32_t lo,
                                               uint32_t n) {
    const uint64_t x = ((uint64_t)hi << 32) | lo;
    return (uint32_t)__umul64hi(x, (uint64_t)n);
}

// One 32-byte row record through the read-only path (2 x 16-B loads of
// the same sector).
__device__ __forceinline__ void ld256(const void* p, unsigned long long& a, unsigned long long& b,
                                      unsigned long long& c, unsigned long long& d);

__device__ __forceinline__ RowRec load_rec(const RowRec* __restrict__ rec, uint32_t j) {
    unsigned long long a, b, c, d;
    ld256(rec + j, a, b, c, d);
    RowRec r;
    r.off = (uint32_t)a;
    r.deg_flags = (uint32_t)(a >> 32);
    r.inv_rate = __uint_as_float((uint32_t)b);
    r.spare = (uint32_t)(b >> 32);
    r.d = __longlong_as_double((long long)c);
    r.v = __longlong_as_double((long long)d);
    return r;
}

// One sector, one instruction: sm_100's 256-bit global load (SASS
// LDG.E.ENL2.256) — a single L1 wavefront per gathered sector instead of
// two 128-bit requests.
__device__ __forceinline__ void ld256(const void* p, unsigned long long& a, unsigned long long& b,
                                      unsigned long long& c, unsigned long long& d) {
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
}

__device__ __forceinline__ Edge load_edge(const Edge* __restrict__ adj, uint32_t k) {
    unsigned long long a, b, c, d;
    ld256(adj + k, a, b, c, d);
    Edge e;
    e.j = (uint32_t)a;
    e.off = (uint32_t)(a >> 32);
    e.deg_flags = (uint32_t)b;
    e.inv_rate = __uint_as_float((uint32_t)(b >> 32));
    e.d = __longlong_as_double((long long)c);
    e.v = __longlong_as_double((long long)d);
    return e;
}

// Jump from the row (off, degf) through the fat adjacency: 64-bit pick
// (hi, lo) of the column, alias correction with `coin` on weighted rows.
__device__ __forceinline__ Edge jump_edge(uint32_t hi, uint32_t lo, uint32_t coin, uint32_t off,
                                          uint32_t degf, const Edge* __restrict__ adj,
                                          const uint32_t* __restrict__ thr,
                                          const uint32_t* __restrict__ alias) {
    uint32_t k = pick_index(hi, lo, degf & kDegMask);
    if ((degf & kNonUniform) && coin >= __ldg(thr + off + k)) k = __ldg(alias + off + k);
    return load_edge(adj, off + k);
}

// Landing row of a jump from the row (off, degf): uniform rows by degree
// scaling (sampler.cpp:25-27) with a 64-bit draw (hi, lo), weighted rows by
// the Walker alias table with the independent 32-bit coin.
__device__ __forceinline__ uint32_t choose_next(uint32_t hi, uint32_t lo, uint32_t coin,
                                                uint32_t off, uint32_t degf,
                                                const uint32_t* __restrict__ nbr,
                                                const uint32_t* __restrict__ thr,
                                                const uint32_t* __restrict__ alias) {
    uint32_t k = pick_index(hi, lo, degf & kDegMask);
    if (degf & kNonUniform) {
        if (coin >= __ldg(thr + off + k)) k = __ldg(alias + off + k);
    }
    return __ldg(nbr + off + k);
}

}  // namespace expmc_b200
