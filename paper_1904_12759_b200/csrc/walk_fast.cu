// K3 entry_fast / K4 scatter_fast / K6 gather_ceiling — the production
// walker kernels (sm_100a).
//
// Same estimators as the reference (Theorem 1: entry_estimate,
// proj/src/estimator.cpp:169-206; Theorem 2: vector_estimate / tc_estimate,
// :208-318) and the same law for every path, re-designed for the GPU:
//
//  * Continuous clock.  The reference restarts an exponential clock at every
//    Δt boundary (sampler.cpp:36-49); by memorylessness one clock per sojourn
//    has the same law (SURVEY finding 5).  A sojourn in state s
//    over grid time [t, t') credits d_s to every grid point k in [t, t'), so
//    the path weight is exp(Δt·Σ_k c_k d_{X_k}) with half weights at k = 0 and
//    k = N for Strang (run_path, estimator.cpp:26-39) — O(1 + jumps) per path
//    instead of O(N + jumps).
//  * Philox4x32-10 keyed by the seed with counter (step, walker, row, tag):
//    a walker's randomness is a pure function of (seed, row, walker), so the
//    result does not depend on grid shape, GPU count or row sharding.
//  * One-compare exit for walkers that never jump: P(no jump) =
//    exp(-rate_i β); such walkers score the deterministic f0 = e^{β d_i} v_i
//    and are accumulated as zero deviation from f0 (shifted sums), so they
//    cost one Philox block and no log / gather.
//  * Per-lane event loop: each iteration either retires a walker or performs
//    one sojourn + jump for it; walkers are assigned to lane slots
//    statically (l ≡ slot mod T) and reduced with a fixed xor tree, so the
//    per-row sums are bitwise deterministic.
//  * Row records are 32-byte sectors {off, deg|flags, 1/rate, d, v}: a jump
//    is two dependent gathers (neighbor id, landing record).
#include "kernels.cuh"

namespace expmc_b200 {

namespace {

__device__ __forceinline__ RowRec load_rec(const RowRec* __restrict__ rec, uint32_t j) {
    const int4* p = reinterpret_cast<const int4*>(rec + j);
    const int4 a = __ldg(p);
    const int4 b = __ldg(p + 1);
    RowRec r;
    r.off = (uint32_t)a.x;
    r.deg_flags = (uint32_t)a.y;
    r.inv_rate = __int_as_float(a.z);
    r.spare = (uint32_t)a.w;
    r.d = __hiloint2double(b.y, b.x);
    r.v = __hiloint2double(b.w, b.z);
    return r;
}

// Choose the landing row from the current record: uniform rows by degree
// scaling (sampler.cpp:25-27), weighted rows by the Walker alias table.
__device__ __forceinline__ uint32_t choose(const U4& w, uint32_t off, uint32_t degf,
                                          const uint32_t* __restrict__ nbr,
                                          const uint32_t* __restrict__ thr,
                                          const uint32_t* __restrict__ alias) {
    const uint32_t deg = degf & kDegMask;
    uint32_t k = pick_index(w.y, w.w, deg);
    if (degf & kNonUniform) {
        if (w.z >= __ldg(thr + off + k)) k = __ldg(alias + off + k);
    }
    return __ldg(nbr + off + k);
}

template <int WPR>
__global__ void __launch_bounds__(128)
entry_fast_kernel(const RowRec* __restrict__ rec, const double* __restrict__ rate,
                  const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ thr,
                  const uint32_t* __restrict__ alias, const uint32_t* __restrict__ rows,
                  uint64_t nrows, FastParams p, double* __restrict__ out_value,
                  double* __restrict__ out_se, uint64_t* __restrict__ out_jumps) {
    constexpr int RPB = 4 / WPR;   // rows per 128-thread block
    constexpr uint32_t T = 32 * WPR; // lane slots per row
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int rib = warp / WPR;     // row within block
    const int wir = warp % WPR;     // warp within row
    const uint32_t slot = (uint32_t)(wir * 32 + lane);
    __shared__ double sh1[4], sh2[4];
    __shared__ unsigned long long shj[4];

    for (uint64_t rb = blockIdx.x; rb * RPB < nrows; rb += gridDim.x) {
        const uint64_t r = rb * RPB + rib;
        double s1 = 0.0, s2 = 0.0;
        unsigned long long jt = 0;
        double f0 = 0.0;
        if (r < nrows) {
            const uint32_t i = rows[r];
            const RowRec ri = load_rec(rec, i);
            const double rate_i = __ldg(rate + i);
            // P(no jump over [0, β]) = exp(-rate β); threshold on a u32 draw
            const double p0 = exp(-__dmul_rn(rate_i, p.beta));
            const uint64_t T0 = (uint64_t)__dmul_rn(p0, 4294967296.0);
            f0 = __dmul_rn(exp(__dmul_rn(p.beta, ri.d)), ri.v);
            const double corr_i = p.strang ? __dmul_rn(0.5, ri.d) : ri.d;

            uint64_t l = slot;
            bool active = false;
            uint32_t off = 0, degf = 0, g = 0, step = 0, jc = 0;
            float ir = 0.f;
            double dcur = 0.0, vcur = 0.0, t = 0.0, S = 0.0;
            while (true) {
                bool fresh = false;
                if (!active) {
                    if (l >= p.W) break;
                    fresh = true;
                    off = ri.off; degf = ri.deg_flags; ir = ri.inv_rate;
                    dcur = ri.d; vcur = ri.v;
                    t = 0.0; S = 0.0; g = 0; step = 0; jc = 0;
                }
                const U4 w = philox4x32_10(U4{step, (uint32_t)l, i, kTagEntry}, p.k0, p.k1);
                if (fresh && (uint64_t)w.x < T0) {  // never jumps: deviation 0
                    l += T;
                    continue;
                }
                active = true;
                const float h = __fmul_rn(neg_ln_u(w.x), ir);
                const double tn = __dadd_rn(t, __dmul_rn((double)h, p.inv_dt));
                if (tn >= p.n_grid) {
                    // path ends in this sojourn: credit grid points g..N
                    S = __fma_rn(dcur, (double)(p.N + 1 - g), S);
                    const double corr =
                        p.strang ? __dadd_rn(corr_i, __dmul_rn(0.5, dcur)) : corr_i;
                    const double f = __dmul_rn(exp(__dmul_rn(p.dt, __dsub_rn(S, corr))), vcur);
                    const double dev = __dsub_rn(f, f0);
                    s1 = __dadd_rn(s1, dev);
                    s2 = __fma_rn(dev, dev, s2);
                    jt += jc;
                    active = false;
                    l += T;
                } else {
                    const uint32_t kk = (uint32_t)ceil(tn);
                    S = __fma_rn(dcur, (double)(kk - g), S);
                    g = kk;
                    t = tn;
                    const uint32_t j = choose(w, off, degf, nbr, thr, alias);
                    const RowRec nr = load_rec(rec, j);
                    off = nr.off; degf = nr.deg_flags; ir = nr.inv_rate;
                    dcur = nr.d; vcur = nr.v;
                    ++jc;
                    ++step;
                }
            }
        }
        // deterministic reduction: xor butterfly within the warp, then warps
        // of the row in index order
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
            s2 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, o));
            jt += __shfl_xor_sync(0xffffffffu, jt, o);
        }
        if (WPR > 1) {
            if (lane == 0) { sh1[warp] = s1; sh2[warp] = s2; shj[warp] = jt; }
            __syncthreads();
            if (wir == 0 && lane == 0) {
                for (int k = 1; k < WPR; ++k) {
                    s1 = __dadd_rn(s1, sh1[warp + k]);
                    s2 = __dadd_rn(s2, sh2[warp + k]);
                    jt += shj[warp + k];
                }
            }
            __syncthreads();
        }
        if (wir == 0 && lane == 0 && r < nrows) {
            const double W = (double)p.W;
            out_value[r] = __dadd_rn(f0, __ddiv_rn(s1, W));
            double se = 0.0;
            if (p.W > 1) {
                double var = __ddiv_rn(__dsub_rn(s2, __ddiv_rn(__dmul_rn(s1, s1), W)),
                                       __dsub_rn(W, 1.0));
                var = var > 0.0 ? var : 0.0;
                se = sqrt(__ddiv_rn(var, W));
            }
            out_se[r] = se;
            out_jumps[r] = jt;
        }
    }
}

// Theorem 2 walkers (vector_estimate / tc_estimate).  Grid-stride over the
// 64-bit walker index; the start state is drawn from Philox step 0xffffffff.
//   start_mode 0: uniform over n rows      1: categorical v / V (cum table)
// Lie weights sit on the state each segment leaves from (estimator.cpp:228-231).
// Per-end-state sums go through fp64 atomics (order not deterministic at
// the last ulp); the scalar tallies are reduced deterministically.
__global__ void __launch_bounds__(128)
scatter_fast_kernel(const RowRec* __restrict__ rec, const uint32_t* __restrict__ nbr,
                    const uint32_t* __restrict__ thr, const uint32_t* __restrict__ alias,
                    uint64_t n, int start_mode, const double* __restrict__ vcum, double v_sum,
                    FastParams p, double* __restrict__ values, double* __restrict__ part_s1,
                    double* __restrict__ part_s2, unsigned long long* __restrict__ part_j) {
    __shared__ double sh1[4], sh2[4];
    __shared__ unsigned long long shj[4];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    double s1 = 0.0, s2 = 0.0;
    unsigned long long jt = 0;
    bool active = false;
    uint32_t cur = 0, off = 0, degf = 0, g = 0, step = 0, jc = 0;
    float ir = 0.f;
    double dcur = 0.0, t = 0.0, S = 0.0, corr0 = 0.0;
    while (true) {
        if (!active) {
            if (l >= p.W) break;
            const U4 ws = philox4x32_10(U4{0xffffffffu, (uint32_t)l, (uint32_t)(l >> 32),
                                           kTagScatter}, p.k0, p.k1);
            uint32_t s;
            if (start_mode == 0) {
                s = pick_index(ws.x, ws.y, (uint32_t)n);
            } else {
                const double u = __dmul_rn((double)((((uint64_t)ws.x << 32) | ws.y) >> 11),
                                           0x1.0p-53);
                const double target = __dmul_rn(u, v_sum);
                uint64_t a = 0, b = n;
                while (a < b) {  // upper_bound, as StartSampler (estimator.cpp:113-121)
                    const uint64_t mid = a + (b - a) / 2;
                    if (target < __ldg(vcum + mid)) b = mid; else a = mid + 1;
                }
                if (a == n) --a;
                s = (uint32_t)a;
            }
            const RowRec rs = load_rec(rec, s);
            cur = s; off = rs.off; degf = rs.deg_flags; ir = rs.inv_rate; dcur = rs.d;
            corr0 = p.strang ? __dmul_rn(0.5, rs.d) : 0.0;
            t = 0.0; S = 0.0; g = 0; step = 0; jc = 0;
            active = true;
        }
        const U4 w = philox4x32_10(U4{step, (uint32_t)l, (uint32_t)(l >> 32), kTagScatter},
                                   p.k0, p.k1);
        const float h = __fmul_rn(neg_ln_u(w.x), ir);
        const double tn = __dadd_rn(t, __dmul_rn((double)h, p.inv_dt));
        if (tn >= p.n_grid) {
            S = __fma_rn(dcur, (double)(p.N + 1 - g), S);
            // Strang: half weights at both ends; Lie: no weight at the end state
            const double corr = p.strang ? __dadd_rn(corr0, __dmul_rn(0.5, dcur)) : dcur;
            const double f = __dmul_rn(v_sum, exp(__dmul_rn(p.dt, __dsub_rn(S, corr))));
            s1 = __dadd_rn(s1, f);
            s2 = __fma_rn(f, f, s2);
            jt += jc;
            if (values) atomicAdd(values + cur, f);
            active = false;
            l += stride;
        } else {
            const uint32_t kk = (uint32_t)ceil(tn);
            S = __fma_rn(dcur, (double)(kk - g), S);
            g = kk;
            t = tn;
            const uint32_t j = choose(w, off, degf, nbr, thr, alias);
            const RowRec nr = load_rec(rec, j);
            cur = j; off = nr.off; degf = nr.deg_flags; ir = nr.inv_rate; dcur = nr.d;
            ++jc;
            ++step;
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

// K6: memory-only walker with the K3 access pattern (neighbor id gather ->
// landing record gather) and a cheap integer hash instead of Philox / log /
// exp.  chains_per_row chains of chain_len jumps start at every listed row.
// Its jumps/s is the same-pattern random-gather ceiling for the roofline.
__global__ void __launch_bounds__(128)
gather_ceiling_kernel(const RowRec* __restrict__ rec, const uint32_t* __restrict__ nbr,
                      const uint32_t* __restrict__ rows, uint64_t nrows,
                      uint32_t chains_per_row, uint32_t chain_len, uint32_t salt,
                      unsigned long long* __restrict__ sink) {
    const uint64_t total = nrows * (uint64_t)chains_per_row;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long acc = 0;
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < total; c += stride) {
        // consecutive lanes walk chains of the same row, as in K3
        uint32_t cur = rows[c / chains_per_row];
        RowRec r = load_rec(rec, cur);
        uint32_t h = (uint32_t)c * 0x9E3779B9u ^ salt;
        for (uint32_t k = 0; k < chain_len; ++k) {
            h ^= h << 13; h ^= h >> 17; h ^= h << 5;
            const uint32_t deg = r.deg_flags & kDegMask;
            if (deg == 0) break;
            cur = __ldg(nbr + r.off + __umulhi(h, deg));
            r = load_rec(rec, cur);
        }
        acc += cur;
    }
    if (acc == 0x7fffffffffffffffull) *sink = acc;  // keep the loads live
}

}  // namespace

// ------------------------------------------------------------ launchers
static unsigned fast_grid(uint64_t blocks_needed) {
    const uint64_t cap = 148ull * 64;  // grid-stride beyond ~64 blocks/SM
    return (unsigned)(blocks_needed < cap ? (blocks_needed ? blocks_needed : 1) : cap);
}

int entry_fast_wpr(uint64_t W) { return W >= 8192 ? 4 : (W >= 4096 ? 2 : 1); }

void launch_entry_fast(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                       const FastParams& p, double* value, double* se, uint64_t* jumps,
                       cudaStream_t s) {
    if (nrows == 0) return;
    const int wpr = entry_fast_wpr(p.W);
    const uint64_t rpb = 4 / wpr;
    const unsigned grid = fast_grid((nrows + rpb - 1) / rpb);
    switch (wpr) {
        case 4:
            entry_fast_kernel<4><<<grid, 128, 0, s>>>(m.rec, m.rate, m.neighbor, m.alias_thr,
                                                      m.alias_idx, rows, nrows, p, value, se,
                                                      jumps);
            break;
        case 2:
            entry_fast_kernel<2><<<grid, 128, 0, s>>>(m.rec, m.rate, m.neighbor, m.alias_thr,
                                                      m.alias_idx, rows, nrows, p, value, se,
                                                      jumps);
            break;
        default:
            entry_fast_kernel<1><<<grid, 128, 0, s>>>(m.rec, m.rate, m.neighbor, m.alias_thr,
                                                      m.alias_idx, rows, nrows, p, value, se,
                                                      jumps);
    }
}

unsigned scatter_fast_grid() { return 148 * 12; }

void launch_scatter_fast(const DevSplit& m, int start_mode, const double* vcum, double v_sum,
                         const FastParams& p, double* values, double* part_s1, double* part_s2,
                         unsigned long long* part_j, cudaStream_t s) {
    scatter_fast_kernel<<<scatter_fast_grid(), 128, 0, s>>>(
        m.rec, m.neighbor, m.alias_thr, m.alias_idx, m.n, start_mode, vcum, v_sum, p, values,
        part_s1, part_s2, part_j);
}

void launch_gather_ceiling(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                           uint32_t chains_per_row, uint32_t chain_len, uint32_t salt,
                           unsigned long long* sink, cudaStream_t s) {
    if (nrows == 0 || chains_per_row == 0) return;
    gather_ceiling_kernel<<<148 * 16, 128, 0, s>>>(m.rec, m.neighbor, rows, nrows,
                                                  chains_per_row, chain_len, salt, sink);
}

}  // namespace expmc_b200
