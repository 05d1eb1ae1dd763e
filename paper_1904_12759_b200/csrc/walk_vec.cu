// K4 — Theorem-2 estimators (vector_estimate, proj/src/estimator.cpp:208-278;
// tc_estimate, :280-318) by grouped starts.
//
// The reference draws M i.i.d. walkers, each with its own start
// (StartSampler, estimator.cpp:92-128: v / V by upper_bound on the
// cumulative table, or uniform), and sums f = V w over them.  Both outputs —
// values[j] = (1/M) Σ_{end = j} f and the tallies Σf, Σf², Σjumps — are
// symmetric functions of the multiset of walkers, so the walkers may be
// generated in any order with the same joint law.  This file generates
// them grouped by start row:
//
//   1. start counts (c_0..c_{n-1}) ~ Multinomial(M, v / V), drawn down a
//      binary tree over the row range: a node [lo, hi) holding c walkers
//      sends Binomial(c, V[lo,mid) / V[lo,hi)) of them left.  Masses are
//      differences of the reference's own cumulative table, so the leaf
//      probabilities telescope to exactly the (cum[i] - cum[i-1]) / V the
//      reference's upper_bound samples;
//   2. per row, the never-jumpers n0 = c_i - Binomial(c_i, 1 - e^{-λ_i}) (λ_i = rate_i β:
//      a walker stays put iff its first holding time exceeds β) score the
//      deterministic f0 = V e^{β d_i} at their own row — added to values[i]
//      directly, no scatter;
//   3. the c_i - n0 jumpers, numbered q = 0, 1, ... in start-row order, start
//      with a first holding time R / rate_i, R ~ Exp(1) truncated to [0, λ_i)
//      (memorylessness), and continue as the continuous-clock walkers of K3;
//      consecutive lanes walk jumpers of the same row, so the first gathers
//      share L1 lines.  Their (end, f) records go through the deterministic
//      sort-based per-end reduction (scatter_sort.cu).
//
// Every draw is keyed by position (tree node, row, global jumper index),
// never by thread, and every floating-point sum has a fixed order, so
// results are bitwise reproducible.
#include <cub/device/device_scan.cuh>

#include "kernels.cuh"

namespace expmc_b200 {

namespace {

constexpr uint32_t kTagTree = 0x4d554c54u;   // 'MULT' multinomial tree
constexpr uint32_t kTagStay = 0x53544159u;   // 'STAY' never-jumper binomial
constexpr uint32_t kTagDebug = 0x44454247u;  // 'DEBG' binomial test hook
constexpr uint32_t kTagBig = 0x454c5247u;    // 'ELRG' large-W entry jumpers
constexpr uint32_t kTagBigStay = 0x45535459u; // 'ESTY' large-W never-jumper split
constexpr int kRowsThreads = 256;
constexpr uint32_t kPer = 64;  // jumpers per thread in the walk kernels
constexpr unsigned kRowsBlocks = 148 * 8;

__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {
    return __dmul_rn((double)((((uint64_t)hi << 32) | lo) >> 11), 0x1.0p-53);
}

// Stirling remainder fc(k) = ln k! - (k + 1/2) ln(k + 1) + (k + 1) - ln √(2π).
__device__ __forceinline__ double stirling_tail(double k) {
    if (k <= 9.0) {
        // exact values for small k (ln k! by lgamma of an integer is exact to ~1 ulp)
        return lgamma(k + 1.0) - (k + 0.5) * log(k + 1.0) + (k + 1.0) -
               0.91893853320467274178;
    }
    const double kp1 = k + 1.0, kp1sq = kp1 * kp1;
    return (1.0 / 12.0 - (1.0 / 360.0 - 1.0 / 1260.0 / kp1sq) / kp1sq) / kp1;
}

// Binomial(n, p) from the Philox stream (iteration r, id0, id1, tag), one
// Philox block per iteration.  n * min(p, 1-p) < 10: inversion (sequential
// pmf search, expected n p + 1 steps); otherwise Hörmann's BTRS
// (transformed rejection with squeeze, W. Hörmann, "The generation of
// binomial random variates", J. Stat. Comput. Simul. 46, 1993), exact
// acceptance test on the Stirling-expanded log pmf ratio.
__device__ uint64_t binomial(uint64_t n, double p, uint32_t id0, uint32_t id1, uint32_t tag,
                             const PhiloxKeys& K) {
    if (n == 0 || !(p > 0.0)) return 0;
    if (p >= 1.0) return n;
    const bool flip = p > 0.5;
    const double pp = flip ? 1.0 - p : p;
    const double nd = (double)n;
    uint64_t x = 0;
    if (nd * pp < 10.0) {
        const double q = 1.0 - pp, s = pp / q, a = (nd + 1.0) * s;
        const double r0 = exp(nd * log1p(-pp));
        for (uint32_t it = 0;; ++it) {
            const U4 w = philox4x32_10(U4{it, id0, id1, tag}, K);
            double u = u53(w.x, w.y), r = r0;
            uint64_t k = 0;
            bool ok = true;
            while (u > r) {
                u -= r;
                ++k;
                if (k > n || k > 2000) { ok = false; break; }  // rounding tail: redraw
                r *= a / (double)k - s;
            }
            if (ok) { x = k; break; }
        }
    } else {
        const double spq = sqrt(nd * pp * (1.0 - pp));
        const double b = 1.15 + 2.53 * spq;
        const double a = -0.0873 + 0.0248 * b + 0.01 * pp;
        const double c = nd * pp + 0.5;
        const double vr = 0.92 - 4.2 / b;
        const double r = pp / (1.0 - pp);
        const double alpha = (2.83 + 5.1 / b) * spq;
        const double m = floor((nd + 1.0) * pp);
        const double fm = stirling_tail(m) + stirling_tail(nd - m);
        for (uint32_t it = 0;; ++it) {
            const U4 w = philox4x32_10(U4{it, id0, id1, tag}, K);
            const double U = u53(w.x, w.y) - 0.5;
            const double V = u53(w.z, w.w);
            const double us = 0.5 - fabs(U);
            const double kf = floor((2.0 * a / us + b) * U + c);
            if (kf < 0.0 || kf > nd) continue;
            if (us >= 0.07 && V <= vr) { x = (uint64_t)kf; break; }
            const double lv = log(V * alpha / (a / (us * us) + b));
            const double h = (m + 0.5) * log((m + 1.0) / (r * (nd - m + 1.0))) +
                             (nd + 1.0) * log1p((kf - m) / (nd - kf + 1.0)) +
                             (kf + 0.5) * log(r * (nd - kf + 1.0) / (kf + 1.0)) + fm -
                             stirling_tail(kf) - stirling_tail(nd - kf);
            if (lv <= h) { x = (uint64_t)kf; break; }
        }
    }
    return flip ? n - x : x;
}

__global__ void set_root_kernel(uint64_t* cnt, uint64_t M) { cnt[0] = M; }

// One level of the multinomial tree.  Node k of level L covers rows
// [k << (D-L), (k+1) << (D-L)) ∩ [0, n); its count lives at cnt[lo] and its
// right child's at cnt[mid] (zero until written here).
__global__ void tree_level_kernel(uint64_t* __restrict__ cnt, uint64_t n, int D, int L,
                                  const double* __restrict__ cum, PhiloxKeys K) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= (1ull << L)) return;
    const uint64_t span = 1ull << (D - L);
    const uint64_t lo = k * span, mid = lo + span / 2;
    if (mid >= n) return;  // no right child: the left keeps everything
    const uint64_t c = cnt[lo];
    if (c == 0) return;
    const uint64_t hi = lo + span < n ? lo + span : n;
    double pl;
    if (cum) {
        const double base = lo ? cum[lo - 1] : 0.0;
        const double left = __dsub_rn(cum[mid - 1], base);
        const double all = __dsub_rn(cum[hi - 1], base);
        pl = all > 0.0 ? left / all : 0.5;
    } else {
        pl = (double)(mid - lo) / (double)(hi - lo);
    }
    const uint64_t x = binomial(c, pl, (uint32_t)k, (uint32_t)L, kTagTree, K);
    cnt[lo] = x;
    cnt[mid] = c - x;
}

// Per row: never-jumpers and their score, jumper count.  Fixed grid and
// fixed in-block tree, so the partial tallies are deterministic.  Every row
// gets its jumper count (the global jumper numbering), only rows in
// [lo, hi) (the shard) score their never-jumpers.
__global__ void __launch_bounds__(kRowsThreads)
vec_rows_kernel(const uint64_t* __restrict__ cnt, const double* __restrict__ rate,
                const double* __restrict__ d, uint64_t n, FastParams p, double v_sum,
                uint64_t lo, uint64_t hi, double* __restrict__ values, uint64_t* __restrict__ jcount,
                double2* __restrict__ rowc, double* __restrict__ part_s1,
                double* __restrict__ part_s2) {
    __shared__ double sh1[kRowsThreads / 32], sh2[kRowsThreads / 32];
    double s1 = 0.0, s2 = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = cnt[i];
        uint64_t n0 = 0;
        double tot = 0.0;
        if (c) {
            const double lam = __dmul_rn(rate[i], p.beta);
            // jumpers ~ Binomial(c, 1 - e^{-λ}), the jump probability from
            // expm1 (no cancellation for small λ)
            const double pj = -expm1(-lam);
            n0 = c - binomial(c, pj, (uint32_t)i, (uint32_t)(i >> 32), kTagStay, p.rk);
            if (n0 < c)  // jumper constants: 1 - e^{-λ}, grid units per unit of R
                rowc[i] = make_double2(pj, __ddiv_rn(p.inv_dt, rate[i]));
            if (n0 && i >= lo && i < hi) {
                // the never-jumper's weight, formed exactly as a walker that
                // finishes at its start would form it (vec_walk_kernel)
                const double di = d[i];
                const double S = __dmul_rn(di, p.n_grid1);
                const double corr = p.strang ? __dadd_rn(__dmul_rn(0.5, di), __dmul_rn(0.5, di))
                                             : di;
                const double f0 = __dmul_rn(v_sum, exp(__dmul_rn(p.dt, __dsub_rn(S, corr))));
                tot = __dmul_rn((double)n0, f0);
                s1 = __dadd_rn(s1, tot);
                s2 = __fma_rn(tot, f0, s2);
            }
        }
        if (values) values[i] = tot;
        jcount[i] = c - n0;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
        s2 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, o));
    }
    if (lane == 0) { sh1[warp] = s1; sh2[warp] = s2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kRowsThreads / 32; ++k) {
            s1 = __dadd_rn(s1, sh1[k]);
            s2 = __dadd_rn(s2, sh2[k]);
        }
        part_s1[blockIdx.x] = s1;
        part_s2[blockIdx.x] = s2;
    }
}

struct U128 {
    unsigned long long lo, hi;
};

__device__ __forceinline__ void add128(U128& a, U128 b) {
    const unsigned long long lo = a.lo + b.lo;
    a.hi += b.hi + (lo < a.lo ? 1ull : 0ull);
    a.lo = lo;
}

// |x| 2^s as an unsigned 128-bit integer (x 2^(s-64) = y: hi = floor(y),
// lo = frac(y) 2^64; power-of-2 scalings and the split are exact), then two's
// complement for x < 0.
__device__ __forceinline__ U128 to_fixed(double x, double scale_hi) {
    const double y = __dmul_rn(fabs(x), scale_hi);
    const double yh = floor(y);
    U128 r{(unsigned long long)__dmul_rn(__dsub_rn(y, yh), 0x1.0p64), (unsigned long long)yh};
    if (x < 0.0) {
        r.lo = ~r.lo + 1ull;
        r.hi = ~r.hi + (r.lo == 0ull ? 1ull : 0ull);
    }
    return r;
}

__device__ __forceinline__ void flush128(unsigned long long* __restrict__ acc, uint64_t r, U128 a) {
    if ((a.lo | a.hi) == 0ull) return;
    const unsigned long long old = atomicAdd(acc + 2 * r, a.lo);
    const unsigned long long hi = a.hi + (old + a.lo < old ? 1ull : 0ull);
    if (hi) atomicAdd(acc + 2 * r + 1, hi);
}

// Order-independent exact per-end accumulation (vector_estimate, the
// `local_values[out.end] += f` of estimator.cpp:250).  f >= 0 is added as
// the 128-bit integer X = f 2^s (two 64-bit atomics with carry); integer
// addition is exact and commutative, so the per-end totals do not depend on
// the order in which walkers finish.  The host picks s so that M f_max 2^s <
// 2^127 and f_min 2^s >= 2^53 (no bit of any f is lost); otherwise it uses
// the sort-based reduction (scatter_sort.cu).
__device__ __forceinline__ void fixed_add(unsigned long long* __restrict__ acc, uint32_t j,
                                          double f, double scale_hi) {
    // (warp-level pre-aggregation of equal ends with __match_any_sync was
    // measured: +12 registers in the walk, 15-25% slower on configs 1-4)
    flush128(acc, j, to_fixed(f, scale_hi));  // f >= 0
}

// values[j] += (hi 2^64 + lo) 2^-s
__global__ void fixed_to_values_kernel(const unsigned long long* __restrict__ acc, uint64_t n,
                                       double inv_scale, double* __restrict__ values) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long lo = acc[2 * j], hi = acc[2 * j + 1];
        if (lo | hi) {
            const double x = __fma_rn(__ull2double_rn(hi), 0x1.0p64, __ull2double_rn(lo));
            values[j] = __dadd_rn(values[j], __dmul_rn(x, inv_scale));
        }
    }
}

// row_of[q - q0] = the start row of jumper q, for q in [q0, q1).  Each warp
// owns chunks of 1024 consecutive jumpers: one binary search over the
// offsets finds the row of the chunk's first jumper, then the warp walks
// the rows forward writing each row's slice (coalesced).  Balanced for many
// small rows and for a few rows with billions of jumpers alike.
__global__ void expand_rows_kernel(const uint64_t* __restrict__ off, uint64_t n, uint64_t q0,
                                   uint64_t q1, uint32_t* __restrict__ row_of) {
    constexpr uint64_t kSpan = 1024;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nchunks = (q1 - q0 + kSpan - 1) / kSpan;
    for (uint64_t c = warp; c < nchunks; c += warps) {
        const uint64_t c0 = q0 + c * kSpan;
        const uint64_t c1 = c0 + kSpan < q1 ? c0 + kSpan : q1;
        uint64_t r = 0;
        if (lane == 0) {  // last r with off[r] <= c0 (upper_bound - 1)
            uint64_t a = 0, b = n + 1;
            while (a < b) {
                const uint64_t mid = a + (b - a) / 2;
                if (off[mid] <= c0) a = mid + 1; else b = mid;
            }
            r = a - 1;
        }
        r = __shfl_sync(0xffffffffu, r, 0);
        uint64_t pos = c0;
        while (pos < c1) {
            uint64_t end = off[r + 1];
            end = end < c1 ? end : c1;
            for (uint64_t q = pos + lane; q < end; q += 32) row_of[q - q0] = (uint32_t)r;
            pos = end > pos ? end : pos;
            ++r;
        }
    }
}

// Jumper walks q in [q0, q1), one lane per walker, static grid-stride
// assignment (consecutive lanes: consecutive jumpers, mostly of one row).
// Jumper q (global index: jumpers numbered in start-row order, a pure
// function of the seed) draws its j-th jump from Philox (j, q_lo, 0,
// 'VECT' ^ q_hi) — y,w: 64-bit neighbour pick, z: alias coin — and x gives
// the holding time at the state it lands on (j >= 1) or, for j = 0, the
// truncated first holding time R at the start.  Lie weights sit on the state each
// segment leaves from (estimator.cpp:228-231).
__global__ void __launch_bounds__(128)
vec_walk_kernel(const RowRec* __restrict__ rec, const Edge* __restrict__ adj,
                const uint32_t* __restrict__ thr, const uint32_t* __restrict__ alias,
                const double2* __restrict__ rowc, const uint32_t* __restrict__ row_of,
                FastParams p, double v_sum, uint64_t q0,
                uint64_t q1, uint32_t* __restrict__ out_end, double* __restrict__ out_f,
                unsigned long long* __restrict__ acc, double scale_hi,
                double* __restrict__ part_s1, double* __restrict__ part_s2,
                unsigned long long* __restrict__ part_j) {
    __shared__ double sh1[4], sh2[4];
    __shared__ unsigned long long shj[4];
    // block b owns jumpers [q0 + b T kPer, q0 + (b+1) T kPer): many small
    // blocks, so the hardware block scheduler balances the SMs (a static
    // grid-stride left SMs idle at the tail)
    const uint64_t stride = blockDim.x;
    const uint64_t qb0 = q0 + blockIdx.x * (uint64_t)blockDim.x * kPer;
    const uint64_t qend = qb0 + (uint64_t)blockDim.x * kPer < q1 ? qb0 + (uint64_t)blockDim.x * kPer : q1;
    uint64_t q = qb0 + threadIdx.x;
    q1 = qend;
    double s1 = 0.0, s2 = 0.0;
    unsigned long long jt = 0;
    bool active = false;
    uint32_t i = 0, off = 0, degf = 0, step = 0, jc = 0, klo = 0, tagv = 0;
    uint32_t wy = 0, ww = 0, wz = 0;  // Philox words of the walker's next jump
    double t = 0.0, S = 0.0, g = 0.0, corr0 = 0.0;
    // start row of the lane's next jumper, loaded one walker ahead
    uint32_t inext = q < q1 ? __ldg(row_of + (q - q0)) : 0u;
    // One trip = (start of the lane's next walker if it has none) -> jump ->
    // Philox block and -ln u of the next step -> sojourn at the landing state.
    // The gathered slot is consumed in the trip that issued it, with the next
    // step's Philox and logarithm between the load and its first use.  (With
    // the landing state carried across the back edge instead, ptxas copies
    // loaded registers right behind the load and the lane waits for the
    // gather at once — the pattern found in K3, profiles/r02/README.md.)
    while (true) {
        if (!active) {
            if (q >= q1) break;
            i = inext;
            if (q + stride < q1) inext = __ldg(row_of + (q + stride - q0));
            klo = (uint32_t)q;
            tagv = kTagScatter ^ (uint32_t)(q >> 32);
            const RowRec rs = load_rec(rec, i);
            const double2 rc = __ldg(rowc + i);  // {1 - e^{-λ_i}, N / (β rate_i)}
            const U4 w = philox4x32_10(U4{0u, klo, 0u, tagv}, p.rk);
            // first holding time R / rate_i, R ~ Exp(1) truncated to [0, λ):
            // R = -log1p(-u (1 - e^{-λ})), u from w.x; the jump from w.y, w.w, w.z
            const float u = __fmul_rn(__uint2float_rn(w.x >> 8) + 0.5f, 0x1.0p-24f);
            const float R = -log1pf(-__fmul_rn(u, (float)rc.x));
            double tn = __dmul_rn((double)R, rc.y);
            if (!(tn < p.n_grid)) tn = __dmul_rn(p.n_grid, 1.0 - 0x1.0p-53);
            corr0 = p.strang ? __dmul_rn(0.5, rs.d) : 0.0;
            // first sojourn at the start: credit its grid points, then jump
            const double kk = ceil(tn);
            S = __dmul_rn(rs.d, kk);
            g = kk;
            t = tn;
            off = rs.off;
            degf = rs.deg_flags;
            wy = w.y; ww = w.w; wz = w.z;
            jc = 0;
            step = 0;
            active = true;
        }
        // the jump drawn at the previous step (or at the start) ...
        const Edge e = jump_edge(wy, ww, wz, off, degf, adj, thr, alias);
        ++jc;
        ++step;
        // ... and, under its gather, this step's Philox block and variate
        const U4 w = philox4x32_10(U4{step, klo, 0u, tagv}, p.rk);
        const float E = neg_ln_u(w.x);
        const float h = __fmul_rn(E, e.inv_rate);
        const double tn = __dadd_rn(t, __dmul_rn((double)h, p.inv_dt));
        if (tn >= p.n_grid) {
            S = __fma_rn(e.d, __dsub_rn(p.n_grid1, g), S);
            const double corr = p.strang ? __dadd_rn(corr0, __dmul_rn(0.5, e.d)) : e.d;
            const double f = __dmul_rn(v_sum, exp(__dmul_rn(p.dt, __dsub_rn(S, corr))));
            s1 = __dadd_rn(s1, f);
            s2 = __fma_rn(f, f, s2);
            jt += jc;
            if (acc) {
                fixed_add(acc, e.j, f, scale_hi);
            } else if (out_end) {
                out_end[q - q0] = e.j;
                out_f[q - q0] = f;
            }
            active = false;
            q += stride;
        } else {
            const double kk = ceil(tn);
            S = __fma_rn(e.d, __dsub_rn(kk, g), S);
            g = kk;
            t = tn;
            off = e.off;
            degf = e.deg_flags;
            wy = w.y; ww = w.w; wz = w.z;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
        s2 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, o));
        jt += __shfl_xor_sync(0xffffffffu, jt, o);
    }
    if (lane == 0) { sh1[warp] = s1; sh2[warp] = s2; shj[warp] = jt; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < 4; ++k) {
            s1 = __dadd_rn(s1, sh1[k]);
            s2 = __dadd_rn(s2, sh2[k]);
            jt += shj[k];
        }
        part_s1[blockIdx.x] = s1;
        part_s2[blockIdx.x] = s2;
        part_j[blockIdx.x] = jt;
    }
}

// ---------------------------------------------------------------------------
// Entry estimator for W >= 2^29 walkers per entry (entry_estimate,
// estimator.cpp:169-206, any `samples`): the K3 walker packs walker indices
// into 29 bits, so very large W take this grouped path instead.  Per listed
// row r (matrix row i = rows[r]): n0 = W - Binomial(W, 1 - e^{-λ_i})
// never-jumpers score f0 = e^{β d_i} v_i; the jumpers (numbered q globally,
// k = q - off[r] within the row) walk as vec_walk_kernel and score
// w v_end.  Sums are kept as deviations from K_r (f0 when never-jumpers
// are the majority, else 0 — K3's rule), so the never-jumpers add
// n0 (f0 - K) and no variance cancels.  Jumper deviations and their squares
// go to records in q order (= row order), summed per row by the
// deterministic run-sum passes; jump counts by integer atomics.

// rowc[r] = {1 - e^{-λ_i}, N / (β rate_i)}; rk[r] = {K_r, -}; s1/s2 start
// with the never-jumpers' n0 (f0 - K), n0 (f0 - K)^2.
__global__ void entry_big_rows_kernel(const uint32_t* __restrict__ rows, uint64_t nrows,
                                      const RowRec* __restrict__ rec,
                                      const double* __restrict__ rate, FastParams p,
                                      uint64_t* __restrict__ jcount, double2* __restrict__ rowc,
                                      double* __restrict__ Kr, double* __restrict__ s1,
                                      double* __restrict__ s2,
                                      unsigned long long* __restrict__ jumps) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nrows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = rows[r];
        const RowRec ri = load_rec(rec, i);
        const double lam = __dmul_rn(rate[i], p.beta);
        const double pj = -expm1(-lam);
        const uint64_t J = binomial(p.W, pj, i, 0u, kTagBigStay, p.rk);
        const uint64_t n0 = p.W - J;
        const double f0 = __dmul_rn(exp(__dmul_rn(p.beta, ri.d)), ri.v);
        const double K = pj <= 0.5 ? f0 : 0.0;  // e^{-λ} >= 1/2: never-jumpers dominate
        const double c = __dsub_rn(f0, K);
        rowc[r] = make_double2(pj, __ddiv_rn(p.inv_dt, rate[i]));
        Kr[r] = K;
        s1[r] = __dmul_rn((double)n0, c);
        s2[r] = __dmul_rn(__dmul_rn((double)n0, c), c);
        jcount[r] = J;
        jumps[r] = 0ull;
    }
}

// Jumper walks of the large-W entry path.  Jumper q of the batch [q0, q1)
// writes its deviation dev = f - K_r and dev^2 to records q - q0; the
// records are in row order (q numbers a row's jumpers consecutively), and
// the host sums them per row with the deterministic run-sum passes
// (scatter_sort.cu run_sums_sorted: fixed 32-record pieces, pieces in
// order, batches in order) — no fixed-point window, so rows of any scale
// keep full fp64 resolution whatever the largest e^{beta d} of the matrix.
// Jump counts: exact integer atomics.
__global__ void __launch_bounds__(128)
entry_big_walk_kernel(const RowRec* __restrict__ rec, const Edge* __restrict__ adj,
                      const uint32_t* __restrict__ thr, const uint32_t* __restrict__ alias,
                      const uint32_t* __restrict__ rows, const double2* __restrict__ rowc,
                      const double* __restrict__ Kr, const uint32_t* __restrict__ row_of,
                      const uint64_t* __restrict__ off, FastParams p, uint64_t q0, uint64_t q1,
                      double* __restrict__ dev1, double* __restrict__ dev2,
                      unsigned long long* __restrict__ jumps) {
    const uint64_t stride = blockDim.x;  // block-owned ranges, as vec_walk_kernel
    const uint64_t qb0 = q0 + blockIdx.x * (uint64_t)blockDim.x * kPer;
    const uint64_t qend = qb0 + (uint64_t)blockDim.x * kPer < q1 ? qb0 + (uint64_t)blockDim.x * kPer : q1;
    uint64_t q = qb0 + threadIdx.x;
    q1 = qend;
    bool active = false;
    uint32_t r = 0, i = 0, off_c = 0, degf = 0, step = 0, jc = 0, klo = 0, tagv = 0;
    uint32_t wy = 0, ww = 0, wz = 0;  // Philox words of the walker's next jump
    double t = 0.0, S = 0.0, g = 0.0, corr0 = 0.0, K = 0.0;
    uint32_t ar = 0xffffffffu;  // row of the lane's open jump count
    unsigned long long aj = 0;
    // trip order as vec_walk_kernel: start -> jump -> next Philox / -ln u -> sojourn
    while (true) {
        if (!active) {
            if (q >= q1) break;
            r = __ldg(row_of + (q - q0));
            if (r != ar) {
                if (ar != 0xffffffffu && aj) atomicAdd(jumps + ar, aj);
                ar = r;
                aj = 0;
            }
            i = __ldg(rows + r);
            K = __ldg(Kr + r);
            const uint64_t k = q - __ldg(off + r);
            klo = (uint32_t)k;
            tagv = kTagBig ^ (uint32_t)(k >> 32);
            const RowRec rs = load_rec(rec, i);
            const double2 rc = __ldg(rowc + r);
            const U4 w = philox4x32_10(U4{0u, klo, i, tagv}, p.rk);
            const float u = __fmul_rn(__uint2float_rn(w.x >> 8) + 0.5f, 0x1.0p-24f);
            const float R = -log1pf(-__fmul_rn(u, (float)rc.x));
            double tn = __dmul_rn((double)R, rc.y);
            if (!(tn < p.n_grid)) tn = __dmul_rn(p.n_grid, 1.0 - 0x1.0p-53);
            corr0 = p.strang ? __dmul_rn(0.5, rs.d) : rs.d;
            const double kk = ceil(tn);
            S = __dmul_rn(rs.d, kk);
            g = kk;
            t = tn;
            off_c = rs.off;
            degf = rs.deg_flags;
            wy = w.y; ww = w.w; wz = w.z;
            jc = 0;
            step = 0;
            active = true;
        }
        const Edge e = jump_edge(wy, ww, wz, off_c, degf, adj, thr, alias);
        ++jc;
        ++step;
        const U4 w = philox4x32_10(U4{step, klo, i, tagv}, p.rk);
        const float E = neg_ln_u(w.x);
        const float h = __fmul_rn(E, e.inv_rate);
        const double tn = __dadd_rn(t, __dmul_rn((double)h, p.inv_dt));
        if (tn >= p.n_grid) {
            S = __fma_rn(e.d, __dsub_rn(p.n_grid1, g), S);
            // Strang: half weights at both ends; Lie: after-weights only
            // (estimator.cpp:176-180) — K3's exponent
            const double Sx = p.strang ? __dsub_rn(S, __dmul_rn(0.5, e.d)) : S;
            const double f = __dmul_rn(exp(__dmul_rn(p.dt, __dsub_rn(Sx, corr0))), e.v);
            const double dv = __dsub_rn(f, K);
            dev1[q - q0] = dv;
            dev2[q - q0] = __dmul_rn(dv, dv);
            aj += jc;
            active = false;
            q += stride;
        } else {
            const double kk = ceil(tn);
            S = __fma_rn(e.d, __dsub_rn(kk, g), S);
            g = kk;
            t = tn;
            off_c = e.off;
            degf = e.deg_flags;
            wy = w.y; ww = w.w; wz = w.z;
        }
    }
    if (ar != 0xffffffffu && aj) atomicAdd(jumps + ar, aj);
}

// value = K + Σdev / W, SE from the one-pass variance of the deviations
// clamped at 0 (finalize, estimator.cpp:76-89).
__global__ void entry_big_finalize_kernel(uint64_t nrows, uint64_t W,
                                          const double* __restrict__ Kr,
                                          const double* __restrict__ s1,
                                          const double* __restrict__ s2,
                                          const unsigned long long* __restrict__ jumps,
                                          double* __restrict__ value, double* __restrict__ se,
                                          uint64_t* __restrict__ out_jumps) {
    const uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const double mm = (double)W;
    value[r] = __dadd_rn(Kr[r], __ddiv_rn(s1[r], mm));
    double e = 0.0;
    if (W > 1) {
        const double var =
            fmax(0.0, __ddiv_rn(__dsub_rn(s2[r], __ddiv_rn(__dmul_rn(s1[r], s1[r]), mm)),
                                __dsub_rn(mm, 1.0)));
        e = sqrt(__ddiv_rn(var, mm));
    }
    se[r] = e;
    out_jumps[r] = jumps[r];
}

__global__ void binomial_debug_kernel(uint64_t n, double p, uint64_t count, PhiloxKeys K,
                                      uint64_t* __restrict__ out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = binomial(n, p, (uint32_t)k, (uint32_t)(k >> 32), kTagDebug, K);
}

int tree_depth(uint64_t n) {
    int D = 0;
    while ((1ull << D) < n) ++D;
    return D;
}

}  // namespace

unsigned vec_rows_grid() { return kRowsBlocks; }
unsigned vec_walk_blocks(uint64_t count) {
    const uint64_t b = (count + 128ull * kPer - 1) / (128ull * kPer);
    return (unsigned)(b ? b : 1);
}

int launch_start_counts(uint64_t n, uint64_t M, const double* cum, const PhiloxKeys& K,
                        uint64_t* cnt, cudaStream_t s) {
    cudaMemsetAsync(cnt, 0, n * 8, s);
    set_root_kernel<<<1, 1, 0, s>>>(cnt, M);
    const int D = tree_depth(n);
    for (int L = 0; L < D; ++L) {  // (returns D + 1 launches with the root)
        const uint64_t nodes = 1ull << L;
        tree_level_kernel<<<(unsigned)((nodes + 255) / 256), 256, 0, s>>>(cnt, n, D, L, cum, K);
    }
    return D + 1;
}

void launch_vec_rows(const DevSplit& m, const uint64_t* cnt, const FastParams& p, double v_sum,
                     uint64_t lo, uint64_t hi, double* values, uint64_t* jcount, double2* rowc, double* part_s1, double* part_s2,
                     cudaStream_t s) {
    vec_rows_kernel<<<kRowsBlocks, kRowsThreads, 0, s>>>(cnt, m.rate, m.d, m.n, p, v_sum, lo, hi, values,
                                                          jcount, rowc, part_s1, part_s2);
}

size_t scan_u64_temp_bytes(uint64_t count) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int64_t)count);
    return b;
}

void launch_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, void* temp,
                     size_t temp_bytes, cudaStream_t s) {
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int64_t)count, s);
}

void launch_expand_rows(const uint64_t* off, uint64_t n, uint64_t q0, uint64_t q1,
                        uint32_t* row_of, cudaStream_t s) {
    if (q1 <= q0) return;
    const uint64_t chunks = (q1 - q0 + 1023) / 1024;  // one warp per chunk, 8 per block
    const unsigned blocks = (unsigned)std::min<uint64_t>((chunks + 7) / 8, 148 * 16);
    expand_rows_kernel<<<blocks, 256, 0, s>>>(off, n, q0, q1, row_of);
}

void launch_vec_walk(const DevSplit& m, const double2* rowc, const uint32_t* row_of,
                     const FastParams& p, double v_sum, uint64_t q0, uint64_t q1,
                     uint32_t* out_end, double* out_f, unsigned long long* acc,
                     double scale_hi, double* part_s1, double* part_s2,
                     unsigned long long* part_j, cudaStream_t s) {
    vec_walk_kernel<<<vec_walk_blocks(q1 - q0), 128, 0, s>>>(m.rec, m.adj, m.alias_thr, m.alias_idx,
                                                    rowc, row_of, p, v_sum, q0, q1, out_end,
                                                    out_f, acc, scale_hi, part_s1, part_s2,
                                                    part_j);
}

void launch_fixed_to_values(const unsigned long long* acc, uint64_t n, double inv_scale,
                            double* values, cudaStream_t s) {
    fixed_to_values_kernel<<<148 * 8, 256, 0, s>>>(acc, n, inv_scale, values);
}

void launch_entry_big_rows(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                           const FastParams& p, uint64_t* jcount, double2* rowc, double* Kr,
                           double* s1, double* s2, unsigned long long* jumps, cudaStream_t s) {
    const unsigned blocks = (unsigned)std::min<uint64_t>((nrows + 255) / 256, 148 * 8);
    entry_big_rows_kernel<<<blocks ? blocks : 1, 256, 0, s>>>(rows, nrows, m.rec, m.rate, p,
                                                               jcount, rowc, Kr, s1, s2, jumps);
}

void launch_entry_big_walk(const DevSplit& m, const uint32_t* rows, const double2* rowc,
                           const double* Kr, const uint32_t* row_of, const uint64_t* off,
                           const FastParams& p, uint64_t q0, uint64_t q1, double* dev1,
                           double* dev2, unsigned long long* jumps, cudaStream_t s) {
    entry_big_walk_kernel<<<vec_walk_blocks(q1 - q0), 128, 0, s>>>(m.rec, m.adj, m.alias_thr,
                                                          m.alias_idx, rows, rowc, Kr, row_of,
                                                          off, p, q0, q1, dev1, dev2, jumps);
}


void launch_entry_big_finalize(uint64_t nrows, uint64_t W, const double* Kr, const double* s1,
                               const double* s2, const unsigned long long* jumps, double* value,
                               double* se, uint64_t* out_jumps, cudaStream_t s) {
    entry_big_finalize_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(
        nrows, W, Kr, s1, s2, jumps, value, se, out_jumps);
}

void launch_binomial_debug(uint64_t n, double p, uint64_t count, const PhiloxKeys& K,
                           uint64_t* out, cudaStream_t s) {
    if (count == 0) return;
    binomial_debug_kernel<<<148 * 4, 256, 0, s>>>(n, p, count, K, out);
}

}  // namespace expmc_b200
