// K4 scatter_fast (vector_estimate / tc_estimate) and K6 gather_ceiling.
//
// K4 runs the Theorem-2 estimators of the reference (vector_estimate,
// proj/src/estimator.cpp:208-278; tc_estimate, :280-318) with the same
// continuous-clock / Philox design as the entry walker (walk_entry.cu):
// one exponential per sojourn, grid points credited per sojourn, walker
// randomness keyed by (seed, walker).
#include "kernels.cuh"

namespace expmc_b200 {

namespace {

// Grid-stride over the 64-bit walker index; the start state is drawn from
// Philox step 0xffffffff.  start_mode 0: uniform over n rows; 1: categorical
// v / V through the cumulative table (StartSampler, estimator.cpp:92-128).
// Lie weights sit on the state each segment leaves from (estimator.cpp:228-231).
// Per-end-state sums use fp64 atomics (last-ulp order dependence); the
// scalar tallies are reduced deterministically.
__global__ void __launch_bounds__(128)
scatter_fast_kernel(const RowRec* __restrict__ rec, const Edge* __restrict__ adj,
                    const uint32_t* __restrict__ thr, const uint32_t* __restrict__ alias, uint64_t n, int start_mode, const double* __restrict__ vcum, double v_sum,
                    FastParams p, uint64_t l0, uint64_t lend, uint32_t* __restrict__ out_end,
                    double* __restrict__ out_f, double* __restrict__ part_s1,
                    double* __restrict__ part_s2, unsigned long long* __restrict__ part_j) {
    __shared__ double sh1[4], sh2[4];
    __shared__ unsigned long long shj[4];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t l = l0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    double s1 = 0.0, s2 = 0.0;
    unsigned long long jt = 0;
    bool active = false;
    uint32_t cur = 0, off = 0, degf = 0, g = 0, step = 0, jc = 0;
    float ir = 0.f;
    double dcur = 0.0, t = 0.0, S = 0.0, corr0 = 0.0;
    while (true) {
        if (!active) {
            if (l >= lend) break;
            const U4 ws = philox4x32_10(U4{0xffffffffu, (uint32_t)l, (uint32_t)(l >> 32),
                                           kTagScatter}, p.rk);
            uint32_t s;
            if (start_mode == 0) {
                s = pick_index(ws.x, ws.y, (uint32_t)n);
            } else {
                const double u = __dmul_rn((double)((((uint64_t)ws.x << 32) | ws.y) >> 11),
                                           0x1.0p-53);
                const double target = __dmul_rn(u, v_sum);
                uint64_t a = 0, b = n;
                while (a < b) {  // upper_bound
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
                                   p.rk);
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
            if (out_end) {  // (end, f) record for the deterministic per-end reduction
                out_end[l - l0] = cur;
                out_f[l - l0] = f;
            }
            active = false;
            l += stride;
        } else {
            const uint32_t kk = (uint32_t)ceil(tn);
            S = __fma_rn(dcur, (double)(kk - g), S);
            g = kk;
            t = tn;
            const Edge e = jump_edge(w.y, w.w, w.z, off, degf, adj, thr, alias);
            cur = e.j; off = e.off; degf = e.deg_flags; ir = e.inv_rate; dcur = e.d;
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
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long acc = 0;
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < total; c += stride) {
        uint32_t cur = rows[c / chains_per_row];
        const RowRec r = load_rec(rec, cur);  // start record, as K3
        uint32_t off = r.off, degf = r.deg_flags;
        uint32_t h = (uint32_t)c * 0x9E3779B9u ^ salt;
        double dsum = r.d;
        for (uint32_t k = 0; k < chain_len; ++k) {
            h ^= h << 13; h ^= h >> 17; h ^= h << 5;
            const uint32_t deg = degf & kDegMask;
            if (deg == 0) break;
            const Edge e = load_edge(adj, off + __umulhi(h, deg));  // one sector per jump
            cur = e.j; off = e.off; degf = e.deg_flags; dsum += e.d;
        }
        acc += cur + (dsum == 0.5 ? 1 : 0);
    }
    if (acc == 0x7fffffffffffffffull) *sink = acc;  // keep the loads live
}

}  // namespace

unsigned scatter_fast_grid() { return 148 * 12; }

void launch_scatter_fast(const DevSplit& m, int start_mode, const double* vcum, double v_sum,
                         const FastParams& p, uint64_t l0, uint64_t lend, uint32_t* out_end,
                         double* out_f, double* part_s1, double* part_s2,
                         unsigned long long* part_j, cudaStream_t s) {
    scatter_fast_kernel<<<scatter_fast_grid(), 128, 0, s>>>(
        m.rec, m.adj, m.alias_thr, m.alias_idx, m.n, start_mode, vcum, v_sum, p, l0, lend,
        out_end, out_f, part_s1, part_s2, part_j);
}

void launch_gather_ceiling(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                           uint32_t chains_per_row, uint32_t chain_len, uint32_t salt,
                           unsigned long long* sink, cudaStream_t s) {
    if (nrows == 0 || chains_per_row == 0) return;
    gather_ceiling_kernel<<<148 * 16, 128, 0, s>>>(m.rec, m.adj, rows, nrows,
                                                  chains_per_row, chain_len, salt, sink);
}

}  // namespace expmc_b200
