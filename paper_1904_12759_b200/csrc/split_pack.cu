// K1 split_pack: CSR adjacency -> SplitMatrix fields + packed row records +
// Walker alias tables, on the device.
//
// Restates split() (proj/src/sparse_matrix.cpp:101-142) bit-exactly: every
// row is summed sequentially in column order by one thread (:124-133), so
// rate / cum / d / uniform_row match the reference bit for bit; dbar is
// nnz / n in fp64 (:138-141, done on the host) and dmax the max degree.
// The symmetric-input checks of SparseSymmetric::from_entries
// (sparse_matrix.cpp:20-51) run in validate_csr.
#include "kernels.cuh"

namespace expmc_b200 {

// Per row: structural validation of the mirrored CSR.  Writes the first
// offending (kind, row, k) into *err with an atomicMin on a packed key so the
// reported error is deterministic (lowest row, then lowest position).
//   kind 1: column out of range   2: non-finite weight   3: zero weight
//        4: negative weight       5: unsorted/duplicate  6: self loop in adj
//        7: not symmetric (A_ij != A_ji or missing mirror)
__global__ void validate_csr_kernel(uint64_t n, const uint64_t* __restrict__ row_ptr,
                                    const uint32_t* __restrict__ col,
                                    const double* __restrict__ val,
                                    unsigned long long* __restrict__ err) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t lo = row_ptr[i], hi = row_ptr[i + 1];
    for (uint64_t k = lo; k < hi; ++k) {
        const uint32_t j = col[k];
        const double w = val[k];
        int kind = 0;
        if (j >= n) kind = 1;
        else if (!isfinite(w)) kind = 2;
        else if (w == 0.0) kind = 3;
        else if (w < 0.0) kind = 4;
        else if (k > lo && col[k - 1] >= j) kind = 5;
        else if (j == i) kind = 6;
        else {
            // mirror lookup: binary search row j for i
            uint64_t a = row_ptr[j], b = row_ptr[j + 1];
            while (a < b) {
                const uint64_t mid = a + (b - a) / 2;
                if (col[mid] < i) a = mid + 1; else b = mid;
            }
            if (a == row_ptr[j + 1] || col[a] != i || val[a] != w) kind = 7;
        }
        if (kind) {
            // key: row (40 bits) | kind (4 bits) | local position (20 bits, saturated)
            const uint64_t pos = (k - lo) < 0xfffffu ? (k - lo) : 0xfffffu;
            const unsigned long long key =
                ((unsigned long long)i << 24) | ((unsigned long long)kind << 20) | pos;
            atomicMin(err, key);
            return;
        }
    }
}

__global__ void split_pack_kernel(uint64_t n, const uint64_t* __restrict__ row_ptr,
                                  const double* __restrict__ weight,
                                  const double* __restrict__ diag,
                                  double* __restrict__ d, double* __restrict__ rate,
                                  double* __restrict__ cum, uint8_t* __restrict__ uniform_row,
                                  RowRec* __restrict__ rec,
                                  unsigned long long* __restrict__ dmax,
                                  unsigned int* __restrict__ any_nonuniform) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t lo = row_ptr[i], hi = row_ptr[i + 1];
    double sum = 0.0;
    bool uni = true;
    const double w0 = hi > lo ? weight[lo] : 0.0;
    for (uint64_t k = lo; k < hi; ++k) {
        const double w = weight[k];
        sum = __dadd_rn(sum, w);  // sequential, column order (bit-exact)
        cum[k] = sum;
        uni = uni && (w == w0);
    }
    const double dg = diag[i];
    const double di = __dadd_rn(dg, sum);
    rate[i] = sum;
    d[i] = di;
    uniform_row[i] = uni ? 1 : 0;
    const uint64_t deg = hi - lo;
    RowRec r;
    r.off = (uint32_t)lo;
    r.deg_flags = (uint32_t)deg | (uni ? 0u : kNonUniform);
    r.inv_rate = (float)__ddiv_rn(1.0, sum);
    r.spare = 0;
    r.d = di;
    r.v = 0.0;
    rec[i] = r;
    // warp-aggregated max (degrees fit 31 bits) / or
    const unsigned mask = __activemask();
    const unsigned m = __reduce_max_sync(mask, (unsigned)deg);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1)) atomicMax(dmax, (unsigned long long)m);
    if (!uni) atomicOr(any_nonuniform, 1u);
}

// Vose alias construction for non-uniform rows (one thread per row),
// identical operation order to orc_alias_row in oracle/expmc_oracle.c.
__device__ __forceinline__ uint32_t quant_prob(double p) {
    const double s = __dmul_rn(p, 4294967296.0);
    if (!(s < 4294967295.0)) return 0xffffffffu;
    if (s < 0.0) return 0u;
    return (uint32_t)s;
}

__global__ void alias_build_kernel(uint64_t n, const uint64_t* __restrict__ row_ptr,
                                   const double* __restrict__ weight,
                                   const double* __restrict__ rate,
                                   const uint8_t* __restrict__ uniform_row,
                                   uint32_t* __restrict__ thr, uint32_t* __restrict__ alias,
                                   double* __restrict__ p, uint32_t* __restrict__ small,
                                   uint32_t* __restrict__ large) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t lo = row_ptr[i], deg = row_ptr[i + 1] - lo;
    if (uniform_row[i] || deg == 0) {
        for (uint64_t k = 0; k < deg; ++k) {
            thr[lo + k] = 0xffffffffu;
            alias[lo + k] = (uint32_t)k;
        }
        return;
    }
    double* pp = p + lo;
    uint32_t* sm = small + lo;
    uint32_t* lg = large + lo;
    uint32_t* th = thr + lo;
    uint32_t* al = alias + lo;
    const double scale = __ddiv_rn((double)deg, rate[i]);
    uint64_t ns = 0, nl = 0;
    for (uint64_t k = 0; k < deg; ++k) {
        pp[k] = __dmul_rn(weight[lo + k], scale);
        if (pp[k] < 1.0) sm[ns++] = (uint32_t)k; else lg[nl++] = (uint32_t)k;
    }
    uint64_t is = 0, il = 0;
    while (is < ns && il < nl) {
        const uint32_t s = sm[is++];
        const uint32_t g = lg[il];
        th[s] = quant_prob(pp[s]);
        al[s] = g;
        pp[g] = __dsub_rn(__dadd_rn(pp[g], pp[s]), 1.0);
        if (pp[g] < 1.0) {
            ++il;
            sm[ns++] = g;
        }
    }
    while (il < nl) { const uint32_t g = lg[il++]; th[g] = 0xffffffffu; al[g] = g; }
    while (is < ns) { const uint32_t s = sm[is++]; th[s] = 0xffffffffu; al[s] = s; }
}

// Fat adjacency: one 32-B slot per directed edge (see Edge in common.cuh).
// One thread per edge; coalesced stores, gathers of the landing record.
__global__ void build_adj_kernel(uint64_t nnz, const uint32_t* __restrict__ neighbor,
                                 const RowRec* __restrict__ rec, Edge* __restrict__ adj) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const uint32_t j = neighbor[e];
    const RowRec r = rec[j];
    Edge x;
    x.j = j;
    x.off = r.off;
    x.deg_flags = r.deg_flags;
    x.inv_rate = r.inv_rate;
    x.d = r.d;
    x.v = r.v;
    adj[e] = x;
}

// Per call: refresh v_j in every fat-adjacency slot (8-B stores at a 32-B
// stride, gathers of v from an L2-resident vector).
// Per-call refresh of Edge.v: the landing row comes from the 4-byte CSR
// neighbour array (0.64 GB at config 5) rather than from the 32-byte slots
// themselves (5.1 GB), so the pass reads 8x less.  (2.55 ms at config 5;
// measured no better: streaming ld.cs / st.cs 2.52 ms, whole-slot 256-bit
// read-modify-write 2.78 ms — profiles/r02/k3_steps.txt, ab_x.)
__global__ void pack_v_adj_kernel(uint64_t nnz, const uint32_t* __restrict__ neighbor,
                                  const double* __restrict__ v, Edge* __restrict__ adj) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    adj[e].v = __ldg(v + __ldg(neighbor + e));
}

void launch_build_adj(uint64_t nnz, const uint32_t* neighbor, const RowRec* rec, Edge* adj,
                      cudaStream_t s) {
    if (nnz == 0) return;
    build_adj_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(nnz, neighbor, rec, adj);
}

void launch_pack_v_adj(uint64_t nnz, const uint32_t* neighbor, const double* v, Edge* adj,
                       cudaStream_t s) {
    if (nnz == 0) return;
    pack_v_adj_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(nnz, neighbor, v, adj);
}

__global__ void pack_v_kernel(uint64_t n, const double* __restrict__ v, RowRec* __restrict__ rec) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) rec[i].v = v[i];
}

__global__ void node_factors_kernel(uint64_t n, const double* __restrict__ d, double scale,
                                    double* __restrict__ f) {
    // node_factors: proj/src/estimator.cpp:41-45
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) f[i] = exp(__dmul_rn(scale, d[i]));
}

// ------------------------------------------------------------ launchers
void launch_validate_csr(uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                         const double* val, unsigned long long* err, cudaStream_t s) {
    if (n == 0) return;
    const unsigned bs = 256;
    validate_csr_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(n, row_ptr, col, val, err);
}

void launch_split_pack(uint64_t n, const uint64_t* row_ptr, const double* weight,
                       const double* diag, double* d, double* rate, double* cum,
                       uint8_t* uniform_row, RowRec* rec, unsigned long long* dmax,
                       unsigned int* any_nonuniform, cudaStream_t s) {
    if (n == 0) return;
    const unsigned bs = 128;
    split_pack_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(
        n, row_ptr, weight, diag, d, rate, cum, uniform_row, rec, dmax, any_nonuniform);
}

// Sum of the row rates (launch heuristics only: per-warp atomics, so the
// last bits depend on the schedule; never feeds a result) and max |d_i| (the
// bound that lets K3 drop exp_det's range clamps: exact, order-independent).
__global__ void rate_sum_kernel(uint64_t n, const double* __restrict__ rate,
                                const double* __restrict__ d, double* __restrict__ out,
                                unsigned long long* __restrict__ dabs_max) {
    double acc = 0.0, mx = 0.0;
    bool bad = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        acc += rate[i];
        const double a = fabs(d[i]);
        bad = bad || !(a <= 1.7976931348623157e308);  // NaN / inf: no bound
        mx = a > mx ? a : mx;
    }
    if (bad) mx = __longlong_as_double(0x7ff0000000000000ll);
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const double y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, acc);
        // non-negative doubles order like their bit patterns
        atomicMax(dabs_max, (unsigned long long)__double_as_longlong(mx));
    }
}

void launch_rate_sum(uint64_t n, const double* rate, const double* d, double* out,
                     unsigned long long* dabs_max, cudaStream_t s) {
    if (n == 0) return;
    const uint64_t want = (n + 255) / 256;
    rate_sum_kernel<<<(unsigned)(want < 1184 ? want : 1184), 256, 0, s>>>(n, rate, d, out,
                                                                         dabs_max);
}

void launch_alias_build(uint64_t n, const uint64_t* row_ptr, const double* weight,
                        const double* rate, const uint8_t* uniform_row, uint32_t* thr,
                        uint32_t* alias, double* p, uint32_t* small, uint32_t* large,
                        cudaStream_t s) {
    if (n == 0) return;
    const unsigned bs = 128;
    alias_build_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(
        n, row_ptr, weight, rate, uniform_row, thr, alias, p, small, large);
}

void launch_pack_v(uint64_t n, const double* v, RowRec* rec, cudaStream_t s) {
    if (n == 0) return;
    const unsigned bs = 256;
    pack_v_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(n, v, rec);
}

void launch_node_factors(uint64_t n, const double* d, double scale, double* f,
                         cudaStream_t s) {
    if (n == 0) return;
    const unsigned bs = 256;
    node_factors_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(n, d, scale, f);
}

}  // namespace expmc_b200
