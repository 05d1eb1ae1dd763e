// §8f row f1: SparseSymmetric::from_entries on the device
// (reference: proj/src/sparse_matrix.cpp:18-85).
//
//   1. validate every entry (range, finite, non-zero, positive off-diagonal)
//      and report the FIRST offending entry in input order with the
//      reference's message (the reference validates in input order, :20-40);
//   2. canonicalise to the upper triangle (row <= col), radix-sort by
//      (row, col) and reject the first duplicate in sorted order (:41-51);
//   3. emit the mirrored adjacency sorted by (row, col) for every directed
//      off-diagonal entry and the diagonal — exactly the CSR that
//      from_entries builds (:58-83) — ready for split_pack (K1).
// Integer work throughout: bit-exact with the reference.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>

#include "kernels.cuh"

namespace expmc_b200 {

namespace {

// kind codes in the error key (lower key = reported first)
//   key = input_index << 3 | kind  (validation: input order)
__global__ void validate_entries_kernel(uint64_t n, const uint32_t* __restrict__ r,
                                        const uint32_t* __restrict__ c,
                                        const double* __restrict__ w, uint64_t ne,
                                        unsigned long long* __restrict__ err) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= ne) return;
    int kind = 0;
    if (r[k] >= n || c[k] >= n) kind = 1;
    else if (!isfinite(w[k])) kind = 2;
    else if (w[k] == 0.0) kind = 3;
    else if (r[k] != c[k] && w[k] < 0.0) kind = 4;
    if (kind) atomicMin(err, ((unsigned long long)k << 3) | (unsigned long long)kind);
}

// canonical key (min << 32 | max) and value index
__global__ void canon_kernel(const uint32_t* __restrict__ r, const uint32_t* __restrict__ c,
                             uint64_t ne, unsigned long long* __restrict__ key,
                             uint64_t* __restrict__ idx) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= ne) return;
    const uint32_t a = r[k] < c[k] ? r[k] : c[k];
    const uint32_t b = r[k] < c[k] ? c[k] : r[k];
    key[k] = ((unsigned long long)a << 32) | b;
    idx[k] = k;
}

// first duplicate in sorted order -> err2 (sorted position)
__global__ void dup_kernel(const unsigned long long* __restrict__ key, uint64_t ne,
                           unsigned long long* __restrict__ err2) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k == 0 || k >= ne) return;
    if (key[k] == key[k - 1]) atomicMin(err2, (unsigned long long)k);
}

// per sorted canonical entry: diagonal -> diag[i]; off-diagonal -> two
// directed (row, col) keys + weight
__global__ void expand_kernel(const unsigned long long* __restrict__ key,
                              const uint64_t* __restrict__ idx, const double* __restrict__ w,
                              uint64_t ne, double* __restrict__ diag,
                              unsigned long long* __restrict__ dkey, double* __restrict__ dw,
                              unsigned int* __restrict__ deg) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= ne) return;
    const uint32_t a = (uint32_t)(key[k] >> 32), b = (uint32_t)key[k];
    const double x = w[idx[k]];
    if (a == b) {
        diag[a] = x;
        dkey[2 * k] = ~0ull;  // sorts last, dropped
        dkey[2 * k + 1] = ~0ull;
    } else {
        dkey[2 * k] = key[k];
        dkey[2 * k + 1] = ((unsigned long long)b << 32) | a;
        atomicAdd(deg + a, 1u);
        atomicAdd(deg + b, 1u);
    }
    dw[2 * k] = x;
    dw[2 * k + 1] = x;
}

__global__ void unpack_cols_kernel(const unsigned long long* __restrict__ dkey, uint64_t m,
                                   uint32_t* __restrict__ col) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k < m) col[k] = (uint32_t)dkey[k];
}

__global__ void deg_to_u64_kernel(const unsigned int* __restrict__ deg, uint64_t n,
                                  uint64_t* __restrict__ out) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = deg[k];
}

inline unsigned blocks(uint64_t x) { return (unsigned)((x + 255) / 256); }

// General-symmetry fold (matrix_market.cpp:136-164) over canonical keys
// sorted by (row, col): a run start is kept; a diagonal run must have length
// 1, an off-diagonal run length 2 with equal weights.  First failing run in
// sorted order -> err (sorted position << 1 | kind; kind 0 = duplicate
// diagonal, 1 = not symmetric).
__global__ void fold_check_kernel(const unsigned long long* __restrict__ key,
                                  const uint64_t* __restrict__ idx, const double* __restrict__ w,
                                  uint64_t ne, unsigned char* __restrict__ keep,
                                  unsigned long long* __restrict__ err) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= ne) return;
    const unsigned long long x = key[k];
    const bool start = k == 0 || key[k - 1] != x;
    keep[k] = start;
    if (!start) return;
    const bool has2 = k + 1 < ne && key[k + 1] == x;
    if ((uint32_t)(x >> 32) == (uint32_t)x) {
        if (has2) atomicMin(err, (unsigned long long)k << 1);
    } else {
        const bool has3 = k + 2 < ne && key[k + 2] == x;
        if (!has2 || has3 || w[idx[k]] != w[idx[k + 1]])
            atomicMin(err, ((unsigned long long)k << 1) | 1ull);
    }
}

__global__ void fold_unpack_kernel(const unsigned long long* __restrict__ key,
                                   const uint64_t* __restrict__ idx,
                                   const double* __restrict__ w, uint64_t m,
                                   uint32_t* __restrict__ r, uint32_t* __restrict__ c,
                                   double* __restrict__ fw) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    r[k] = (uint32_t)(key[k] >> 32);
    c[k] = (uint32_t)key[k];
    fw[k] = w[idx[k]];
}

}  // namespace

// Fold a general (two-triangle) entry list into its upper triangle on the
// device.  On success r_out / c_out / w_out hold *m entries (device memory
// owned by the caller), sorted by (row, col) with row <= col.  On failure
// *err_host = sorted position << 1 | kind and *err_key = that run's
// canonical key; outputs are left null.
void fold_general_device(const uint32_t* r, const uint32_t* c, const double* w, uint64_t ne,
                         uint32_t** r_out, uint32_t** c_out, double** w_out, uint64_t* m,
                         unsigned long long* err_host, unsigned long long* err_key,
                         cudaStream_t s) {
    *r_out = nullptr;
    *c_out = nullptr;
    *w_out = nullptr;
    *m = 0;
    *err_host = ~0ull;
    if (ne == 0) return;
    unsigned long long *key, *key2, *err;
    uint64_t *idx, *idx2;
    unsigned char* keep;
    int* nsel;
    cudaMalloc(&key, ne * 8);
    cudaMalloc(&key2, ne * 8);
    cudaMalloc(&idx, ne * 8);
    cudaMalloc(&idx2, ne * 8);
    cudaMalloc(&keep, ne);
    cudaMalloc(&err, 8);
    cudaMalloc(&nsel, 4);
    cudaMemcpyAsync(err, err_host, 8, cudaMemcpyHostToDevice, s);
    canon_kernel<<<blocks(ne), 256, 0, s>>>(r, c, ne, key, idx);
    size_t tb = 0, tk = 0, ti = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, idx2, (int)ne, 0, 64, s);
    cub::DeviceSelect::Flagged(nullptr, tk, key2, keep, key, nsel, (int)ne, s);
    cub::DeviceSelect::Flagged(nullptr, ti, idx2, keep, idx, nsel, (int)ne, s);
    void* tmp = nullptr;
    cudaMalloc(&tmp, std::max(tb, std::max(tk, ti)));
    cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, idx, idx2, (int)ne, 0, 64, s);
    fold_check_kernel<<<blocks(ne), 256, 0, s>>>(key2, idx2, w, ne, keep, err);
    cudaMemcpyAsync(err_host, err, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (*err_host != ~0ull) {
        cudaMemcpy(err_key, key2 + (*err_host >> 1), 8, cudaMemcpyDeviceToHost);
    } else {
        // compact the run starts (keys, then value indices)
        cub::DeviceSelect::Flagged(tmp, tk, key2, keep, key, nsel, (int)ne, s);
        cub::DeviceSelect::Flagged(tmp, ti, idx2, keep, idx, nsel, (int)ne, s);
        int cnt = 0;
        cudaMemcpyAsync(&cnt, nsel, 4, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        *m = (uint64_t)cnt;
        cudaMalloc(r_out, (cnt ? cnt : 1) * 4);
        cudaMalloc(c_out, (cnt ? cnt : 1) * 4);
        cudaMalloc(w_out, (cnt ? cnt : 1) * 8);
        if (cnt) fold_unpack_kernel<<<blocks(cnt), 256, 0, s>>>(key, idx, w, cnt, *r_out, *c_out, *w_out);
        cudaStreamSynchronize(s);
    }
    cudaFree(tmp); cudaFree(key); cudaFree(key2); cudaFree(idx); cudaFree(idx2);
    cudaFree(keep); cudaFree(err); cudaFree(nsel);
}

// Device arrays r, c, w (ne entries) -> row_ptr (n+1, u64), col (nnz), val
// (nnz), diag (n).  Scratch is allocated here.  Returns 0 on success, or the
// error key: validation (input index << 3 | kind) in err[0], first
// duplicate sorted position in err[1] (ulong max = none) with the duplicate
// canonical key in *dup_key.  nnz_out = number of directed off-diagonal
// entries.
void from_entries_device(uint64_t n, const uint32_t* r, const uint32_t* c, const double* w,
                         uint64_t ne, uint64_t* row_ptr, uint32_t** col_out, double** val_out,
                         double* diag, uint64_t* nnz_out, unsigned long long* err_host,
                         unsigned long long* dup_key, cudaStream_t s) {
    unsigned long long* err = nullptr;
    cudaMalloc(&err, 2 * sizeof(unsigned long long));
    const unsigned long long init[2] = {~0ull, ~0ull};
    cudaMemcpyAsync(err, init, sizeof(init), cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(diag, 0, n * 8, s);
    *col_out = nullptr;
    *val_out = nullptr;
    *nnz_out = 0;
    if (ne) validate_entries_kernel<<<blocks(ne), 256, 0, s>>>(n, r, c, w, ne, err);
    cudaMemcpyAsync(err_host, err, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    err_host[1] = ~0ull;
    if (err_host[0] != ~0ull || ne == 0) {
        if (ne == 0 && err_host[0] == ~0ull) {
            cudaMemsetAsync(row_ptr, 0, (n + 1) * 8, s);
            cudaStreamSynchronize(s);
        }
        cudaFree(err);
        return;
    }
    unsigned long long *key, *key2;
    uint64_t *idx, *idx2;
    cudaMalloc(&key, ne * 8);
    cudaMalloc(&key2, ne * 8);
    cudaMalloc(&idx, ne * 8);
    cudaMalloc(&idx2, ne * 8);
    canon_kernel<<<blocks(ne), 256, 0, s>>>(r, c, ne, key, idx);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, idx2, (int)ne, 0, 64, s);
    void* tmp = nullptr;
    cudaMalloc(&tmp, tb);
    cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, idx, idx2, (int)ne, 0, 64, s);
    cudaFree(tmp);
    dup_kernel<<<blocks(ne), 256, 0, s>>>(key2, ne, err + 1);
    cudaMemcpyAsync(err_host + 1, err + 1, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (err_host[1] != ~0ull) {
        cudaMemcpy(dup_key, key2 + err_host[1], 8, cudaMemcpyDeviceToHost);
        cudaFree(key); cudaFree(key2); cudaFree(idx); cudaFree(idx2); cudaFree(err);
        return;
    }
    // expand to directed entries and sort by (row, col)
    unsigned long long *dkey, *dkey2;
    double *dw, *dw2;
    unsigned int* deg;
    cudaMalloc(&dkey, 2 * ne * 8);
    cudaMalloc(&dkey2, 2 * ne * 8);
    cudaMalloc(&dw, 2 * ne * 8);
    cudaMalloc(&dw2, 2 * ne * 8);
    cudaMalloc(&deg, (n + 1) * 4);
    cudaMemsetAsync(deg, 0, (n + 1) * 4, s);
    expand_kernel<<<blocks(ne), 256, 0, s>>>(key2, idx2, w, ne, diag, dkey, dw, deg);
    tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, dkey, dkey2, dw, dw2, (int)(2 * ne), 0, 64, s);
    cudaMalloc(&tmp, tb);
    cub::DeviceRadixSort::SortPairs(tmp, tb, dkey, dkey2, dw, dw2, (int)(2 * ne), 0, 64, s);
    cudaFree(tmp);
    // row_ptr = exclusive scan of degrees (n + 1 entries, last = nnz)
    uint64_t* deg64;
    cudaMalloc(&deg64, (n + 1) * 8);
    cudaMemsetAsync(deg64, 0, (n + 1) * 8, s);
    deg_to_u64_kernel<<<blocks(n), 256, 0, s>>>(deg, n, deg64);
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, deg64, row_ptr, (int)(n + 1), s);
    cudaMalloc(&tmp, tb);
    cub::DeviceScan::ExclusiveSum(tmp, tb, deg64, row_ptr, (int)(n + 1), s);
    cudaFree(tmp);
    uint64_t nnz = 0;
    cudaMemcpyAsync(&nnz, row_ptr + n, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    uint32_t* col = nullptr;
    cudaMalloc(&col, (nnz ? nnz : 1) * 4);
    if (nnz) unpack_cols_kernel<<<blocks(nnz), 256, 0, s>>>(dkey2, nnz, col);
    double* val = nullptr;
    cudaMalloc(&val, (nnz ? nnz : 1) * 8);
    if (nnz) cudaMemcpyAsync(val, dw2, nnz * 8, cudaMemcpyDeviceToDevice, s);
    cudaStreamSynchronize(s);
    *col_out = col;
    *val_out = val;
    *nnz_out = nnz;
    cudaFree(key); cudaFree(key2); cudaFree(idx); cudaFree(idx2); cudaFree(dkey);
    cudaFree(dkey2); cudaFree(dw); cudaFree(dw2); cudaFree(deg); cudaFree(deg64); cudaFree(err);
}

}  // namespace expmc_b200
