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

// -ln(u) ~ Exp(1) from one 32-bit Philox word, fp32, IEEE-exact operations
// only (so oracle/fast_model.c fm_neg_ln_u reproduces it bit for bit).
// u = x 2^-32 with x = w | 1: the midpoint of one of 2^31 equal bins of
// (0, 1), so P(E > y) matches e^-y to within 2^-31 everywhere, up to the
// largest draw 32 ln 2 = 22.18 (the reference draws a 53-bit uniform,
// rng.hpp:47-49, sampler.cpp:10-16; tests/test_gpu_rng_law.py bounds the
// difference).  x = 2^e m exactly up to fp32 rounding of x (24 bits); with
// m folded into [sqrt(1/2), sqrt(2)), -ln u = (32 - e) ln 2 - ln m, ln m =
// f q(f), f = m - 1 (exact), q a degree-8 Chebyshev fit of log1p(f)/f (rel.
// err 2.7e-8).  Near u = 1 (e = 32) the ln 2 term vanishes exactly.
// Absolute error <= 1.5e-7 max(1, E).  (A 64-entry table variant with a
// degree-3 log1p measured 1.2 ms slower on config 5: the L1 lookups compete
// with the gathers, profiles/r02/README.md.)
__device__ __forceinline__ float neg_ln_u(uint32_t w) {
    const uint32_t bits = __float_as_uint(__uint2float_rn(w | 1u));
    int e32 = 159 - (int)(bits >> 23);  // 32 - e
    float m = __uint_as_float((bits & 0x007fffffu) | 0x3f800000u);  // [1,2)
    if (m > 1.41421356f) {
        m = __fmul_rn(m, 0.5f);
        e32 -= 1;
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
    const float E = __fmaf_rn(__int2float_rn(e32), 0.693147182f, -__fmul_rn(f, q));
    return E > 0.0f ? E : 0.0f;
}

// e^x in fp64 from IEEE-exact operations only (rint, fma, mul, add), so the
// CPU model (oracle/fast_model.c fm_exp) reproduces it bit for bit.
// Table-driven: x = (32k + j) ln2/32 + r, |r| <= ln2/64; e^x = 2^k 2^(j/32)
// e^r with 2^(j/32) as a double-double {hi, lo} (32 entries, 512 B, L1
// resident) and e^r - 1 = r(1 + r/2 + ... + r^5/720) (truncation 3e-18):
// y = hi + fma(hi, e^r - 1, lo), ~0.5 ulp.  Six dependent DFMAs instead of
// a degree-13 chain.  Range handling is branch-free: x is clamped (NaN
// passes through: the compares are false) and 2^k applied as 2^k1 * 2^k2,
// exact up to the final rounding, so overflow gives +inf and underflow
// rounds to subnormals / 0 like a single correctly rounded scaling.
__device__ const double2 kExpTab[32] = {
    {0x1.0000000000000p+0, 0x0.0p+0},
    {0x1.059b0d3158574p+0, 0x1.d73e2a475b465p-55},
    {0x1.0b5586cf9890fp+0, 0x1.8a62e4adc610bp-54},
    {0x1.11301d0125b51p+0, -0x1.6c51039449b3ap-54},
    {0x1.172b83c7d517bp+0, -0x1.19041b9d78a76p-55},
    {0x1.1d4873168b9aap+0, 0x1.e016e00a2643cp-54},
    {0x1.2387a6e756238p+0, 0x1.9b07eb6c70573p-54},
    {0x1.29e9df51fdee1p+0, 0x1.612e8afad1255p-55},
    {0x1.306fe0a31b715p+0, 0x1.6f46ad23182e4p-55},
    {0x1.371a7373aa9cbp+0, -0x1.63aeabf42eae2p-54},
    {0x1.3dea64c123422p+0, 0x1.ada0911f09ebcp-55},
    {0x1.44e086061892dp+0, 0x1.89b7a04ef80d0p-59},
    {0x1.4bfdad5362a27p+0, 0x1.d4397afec42e2p-56},
    {0x1.5342b569d4f82p+0, -0x1.07abe1db13cadp-55},
    {0x1.5ab07dd485429p+0, 0x1.6324c054647adp-54},
    {0x1.6247eb03a5585p+0, -0x1.383c17e40b497p-54},
    {0x1.6a09e667f3bcdp+0, -0x1.bdd3413b26456p-54},
    {0x1.71f75e8ec5f74p+0, -0x1.16e4786887a99p-55},
    {0x1.7a11473eb0187p+0, -0x1.41577ee04992fp-55},
    {0x1.82589994cce13p+0, -0x1.d4c1dd41532d8p-54},
    {0x1.8ace5422aa0dbp+0, 0x1.6e9f156864b27p-54},
    {0x1.93737b0cdc5e5p+0, -0x1.75fc781b57ebcp-57},
    {0x1.9c49182a3f090p+0, 0x1.c7c46b071f2bep-56},
    {0x1.a5503b23e255dp+0, -0x1.d2f6edb8d41e1p-54},
    {0x1.ae89f995ad3adp+0, 0x1.7a1cd345dcc81p-54},
    {0x1.b7f76f2fb5e47p+0, -0x1.5584f7e54ac3bp-56},
    {0x1.c199bdd85529cp+0, 0x1.11065895048ddp-55},
    {0x1.cb720dcef9069p+0, 0x1.503cbd1e949dbp-56},
    {0x1.d5818dcfba487p+0, 0x1.2ed02d75b3707p-55},
    {0x1.dfc97337b9b5fp+0, -0x1.1a5cd4f184b5cp-54},
    {0x1.ea4afa2a490dap+0, -0x1.e9c23179c2893p-54},
    {0x1.f50765b6e4540p+0, 0x1.9d3e12dd8a18bp-54}};

// `tab`: kExpTab or a shared-memory copy of it (same values, same result).
__device__ __forceinline__ double exp_det_tab(double x, const double2* __restrict__ tab, bool tab_global) {
    x = x > 710.0 ? 710.0 : x;
    x = x < -746.0 ? -746.0 : x;
    // n = rint(x 32/ln2) by the 1.5 2^52 shifter (round-to-nearest-even, as
    // rint; |x 32/ln2| < 2^15): the integer sits in the low word, no
    // FRND / F2I on the slow pipes
    const double sh = __dadd_rn(__dmul_rn(x, 0x1.71547652b82fep+5), 0x1.8p52);  // 32 / ln2
    const double n = __dsub_rn(sh, 0x1.8p52);
    double r = __fma_rn(-n, 0x1.62e42fee00000p-6, x);  // ln2/32, hi part (exact n*hi)
    r = __fma_rn(-n, 0x1.a39ef35793c76p-38, r);         // ln2/32, lo part
    double p = 1.0 / 720.0;
    p = __fma_rn(p, r, 1.0 / 120.0);
    p = __fma_rn(p, r, 1.0 / 24.0);
    p = __fma_rn(p, r, 1.0 / 6.0);
    p = __fma_rn(p, r, 0.5);
    p = __fma_rn(p, r, 1.0);
    p = __dmul_rn(p, r);  // e^r - 1
    const int ni = (int)__double2loint(sh);
    const double2 t = tab_global ? __ldg(&tab[ni & 31]) : tab[ni & 31];
    const double y = __dadd_rn(t.x, __fma_rn(t.x, p, t.y));
    const int k = ni >> 5;
    const int k1 = k >> 1;
    return __dmul_rn(__dmul_rn(y, __longlong_as_double((long long)(k1 + 1023) << 52)),
                     __longlong_as_double((long long)(k - k1 + 1023) << 52));
}

__device__ __forceinline__ double exp_det(double x) { return exp_det_tab(x, kExpTab, true); }

// exp_det for |x| <= 690, from a shared-memory table: the range clamps are
// no-ops there and 2^k is a normal number (|k| <= 996), so the scaling is one
// exact multiplication instead of two — the same bits as exp_det, eleven
// instructions fewer.  The caller guarantees the range (K3: from max |d|).
__device__ __forceinline__ double exp_det_inrange(double x, const double2* __restrict__ tab) {
    const double sh = __dadd_rn(__dmul_rn(x, 0x1.71547652b82fep+5), 0x1.8p52);  // 32 / ln2
    const double n = __dsub_rn(sh, 0x1.8p52);
    double r = __fma_rn(-n, 0x1.62e42fee00000p-6, x);
    r = __fma_rn(-n, 0x1.a39ef35793c76p-38, r);
    double p = 1.0 / 720.0;
    p = __fma_rn(p, r, 1.0 / 120.0);
    p = __fma_rn(p, r, 1.0 / 24.0);
    p = __fma_rn(p, r, 1.0 / 6.0);
    p = __fma_rn(p, r, 0.5);
    p = __fma_rn(p, r, 1.0);
    p = __dmul_rn(p, r);  // e^r - 1
    const int ni = (int)__double2loint(sh);
    const double2 t = tab[ni & 31];
    const double y = __dadd_rn(t.x, __fma_rn(t.x, p, t.y));
    return __dmul_rn(y, __longlong_as_double((long long)((ni >> 5) + 1023) << 52));
}

// floor(x * n / 2^64) for a 64-bit uniform x: unbiased to n / 2^64.
__device__ __forceinline__ uint32_t pick_index(uint32_t hi, uint32_t lo,
                                               uint32_t n) {
    // = umul64hi(hi:lo, n): the high word of lo n carries into hi n
    return (uint32_t)(((uint64_t)hi * n + __umulhi(lo, n)) >> 32);
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

// The walkers' random Edge gathers: same load with an L1 policy
// (ENTRY_LD_HINT 1: L1::no_allocate, 2: L1::evict_first, 0: none).  The
// gathered sectors are never reused from L1, and without an allocation per
// gather the number of gathers in flight is no longer capped by the L1 lines
// left beside the shared-memory carveout: config 4 at 8 blocks/SM (28 KB of
// L1) 4.59 s -> 2.72 s, config 5 45.1 -> 44.1 ms (profiles/r02/README.md).
#ifndef ENTRY_LD_HINT
#define ENTRY_LD_HINT 1
#endif
__device__ __forceinline__ void ld256_gather(const void* p, unsigned long long& a,
                                             unsigned long long& b, unsigned long long& c,
                                             unsigned long long& d) {
#if ENTRY_LD_HINT == 1
    asm("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
#elif ENTRY_LD_HINT == 2
    asm("ld.global.nc.L1::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
#else
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
#endif
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
