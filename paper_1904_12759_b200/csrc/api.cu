// Host driver behind the C ABI (include/expmc_b200.h).
//
// Mirrors the reference's estimator entry points and their argument
// validation (proj/src/estimator.cpp:130-139, :161-173, :210-222, :283) with
// the same std::invalid_argument messages, then launches the sm_100a
// kernels.  No CPU fallback exists: every estimate is computed on the GPU.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "expmc_b200.h"
#include "host_io.h"
#include "kernels.cuh"

using namespace expmc_b200;

namespace {

// Last error message of this thread.  A trivially destructible buffer, not
// a std::string: a handle destroyed during static destruction (a cache of
// device copies in a caller's static map) may report an error after the
// thread's thread_local destructors have run.
struct ErrSlot {
    char s[2048];
};
thread_local ErrSlot g_err_slot;
void set_err(const char* m) { std::snprintf(g_err_slot.s, sizeof g_err_slot.s, "%s", m); }
void set_err(const std::string& m) { set_err(m.c_str()); }
std::atomic<uint64_t> g_launches{0};

struct InvalidArg : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct CudaErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess)                                                        \
            throw CudaErr(std::string(#x) + ": " + cudaGetErrorString(e_));           \
    } while (0)

void after_launch(uint64_t kernels) {
    g_launches += kernels;
    CK(cudaGetLastError());
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return EXPMC_OK;
    } catch (const CudaErr& e) {
        set_err(e.what());
        return EXPMC_CUDA_ERROR;
    } catch (const std::invalid_argument& e) {
        set_err(e.what());
        return EXPMC_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        set_err(e.what());
        return EXPMC_RUNTIME_ERROR;
    } catch (...) {
        set_err("unknown error");
        return EXPMC_RUNTIME_ERROR;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CK(cudaGetDevice(&prev));
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

// grow-only device scratch buffer
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <class T>
    T* get(size_t count) {
        const size_t bytes = count * sizeof(T) ? count * sizeof(T) : 16;
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CK(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

std::string pair_str(uint64_t a, uint64_t b) {
    if (a > b) std::swap(a, b);  // reference prints the canonical upper triangle
    return "(" + std::to_string(a) + ", " + std::to_string(b) + ")";
}

void validate_params(const expmc_path_params* p) {
    // PathParams::validate, estimator.cpp:161-167
    if (!p) throw InvalidArg("PathParams pointer is null");
    if (!(p->beta > 0.0) || !std::isfinite(p->beta))
        throw InvalidArg("beta must be positive and finite");
    if (p->n_steps == 0) throw InvalidArg("n_steps must be >= 1");
    if (p->samples == 0) throw InvalidArg("samples must be >= 1");
    if (p->splitting != EXPMC_LIE && p->splitting != EXPMC_STRANG)
        throw InvalidArg("unknown splitting");
    if (p->rng != EXPMC_RNG_PHILOX && p->rng != EXPMC_RNG_PCG_COMPAT)
        throw InvalidArg("unknown rng engine");
    if (p->rng == EXPMC_RNG_PHILOX && p->n_steps >= (1ull << 31))
        throw InvalidArg("n_steps must be < 2^31 for the continuous-clock walker");
}

FastParams fast_params(const expmc_path_params* p, uint64_t walkers) {
    FastParams f;
    f.beta = p->beta;
    f.dt = p->beta / (double)p->n_steps;  // PathParams::dt, estimator.hpp:27
    f.inv_dt = 1.0 / f.dt;
    f.n_grid = (double)p->n_steps;
    f.n_grid1 = (double)p->n_steps + 1.0;
    f.N = (uint32_t)p->n_steps;
    f.strang = p->splitting == EXPMC_STRANG;
    f.W = walkers;
    f.k0 = (uint32_t)p->seed;
    f.k1 = (uint32_t)(p->seed >> 32);
    f.rk = philox_keys(f.k0, f.k1);
    return f;
}

}  // namespace

struct expmc_matrix {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // D2H of result pieces (host API)
    cudaEvent_t piece_done = nullptr;
    DevSplit m;
    std::vector<void*> owned;
    DevBuf vdev, rows, out_val, out_se, out_j, fa, vcum, values, pa, pb, pc, scal, tmp1, tmp2,
        tmp3, iota, part, fa2, sort_tmp, lens, cnt, jcnt, joff, row_of, scan_tmp, rowc;
    uint64_t iota_n = 0;
    uint64_t last_jumpers = 0;  // K4: jumpers of the last vector / tc call
    int last_fixed = -1;        // K4: 1 fixed-point per-end sums, 0 sort-based
    double d_lo = 0.0, d_hi = 0.0;  // range of d (K4 fixed-point scale), once
    bool d_range = false;
    DevBuf acc;
    // One call at a time per handle: the scratch buffers, the packed v and
    // the stream are per handle (the reference's SplitMatrix is shareable
    // across threads; callers sharing a handle are serialised).
    mutable std::mutex mu;
    // Staged v (host entry calls): the packed RowRec.v / Edge.v / vdev hold
    // the v of host pointer vkey_ptr (length vkey_n) when vstaged.  Reused
    // without a copy only when the caller opted in (vcache, expmc_cuda_set_v_cache)
    // and promises to call expmc_cuda_invalidate_v after changing v in place.
    bool vcache = false, vstaged = false;
    const double* vkey_ptr = nullptr;
    uint64_t vkey_n = 0;
    uint64_t v_stagings = 0;  // H2D + pack passes done (tests / measurement)
    // host copies kept for K5 norm bounds
    std::vector<double> h_rate, h_diag;

    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        CK(cudaMalloc(&p, (count ? count : 1) * sizeof(T)));
        owned.push_back(p);
        return static_cast<T*>(p);
    }
    ~expmc_matrix() {
        for (void* p : owned) cudaFree(p);
        for (DevBuf* b : {&vdev, &rows, &out_val, &out_se, &out_j, &fa, &vcum, &values, &pa,
                          &pb, &pc, &scal, &tmp1, &tmp2, &tmp3, &iota, &part, &fa2, &sort_tmp, &lens, &cnt, &jcnt,
                          &joff, &row_of, &scan_tmp, &rowc, &acc})
            b->release();
        if (stream) cudaStreamDestroy(stream);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (piece_done) cudaEventDestroy(piece_done);
    }
};

namespace {

// Device-API stream argument: a cudaStream_t; NULL is the legacy default
// stream (CUDA's own convention), so torch's default stream handle works.
cudaStream_t pick_stream(expmc_matrix*, void* s) { return static_cast<cudaStream_t>(s); }

void check_vector(const expmc_matrix* h, const double* v, uint64_t nv) {
    // check_vector, estimator.cpp:130-139
    if (nv != h->m.n || (!v && nv)) throw InvalidArg("vector length does not match matrix");
    for (uint64_t k = 0; k < nv; ++k)
        if (!std::isfinite(v[k])) throw InvalidArg("non-finite entry in v");
}

const uint32_t* all_rows(expmc_matrix* h) {
    uint32_t* d = h->iota.get<uint32_t>(h->m.n);
    if (h->iota_n != h->m.n) {
        std::vector<uint32_t> tmp(h->m.n);
        for (uint64_t k = 0; k < h->m.n; ++k) tmp[k] = (uint32_t)k;
        CK(cudaMemcpy(d, tmp.data(), h->m.n * 4, cudaMemcpyHostToDevice));
        h->iota_n = h->m.n;
    }
    return d;
}

void alloc_split(expmc_matrix* h, uint64_t n, uint64_t nnz) {
    DevSplit& m = h->m;
    m.n = n;
    m.nnz = nnz;
    m.diag = h->alloc<double>(n);
    m.d = h->alloc<double>(n);
    m.rate = h->alloc<double>(n);
    m.row_offset = h->alloc<uint64_t>(n + 1);
    m.neighbor = h->alloc<uint32_t>(nnz);
    m.weight = h->alloc<double>(nnz);
    m.cum = h->alloc<double>(nnz);
    m.uniform_row = h->alloc<uint8_t>(n);
    m.rec = h->alloc<RowRec>(n);
}

// K1 on an uploaded (valid) mirrored CSR: split(), alias tables, fat
// adjacency (sparse_matrix.cpp:101-142 + the B200 walk layout).
void finish_split(expmc_matrix* h) {
    DevSplit& m = h->m;
    const uint64_t n = m.n, nnz = m.nnz;
    cudaStream_t s = h->stream;
    unsigned long long* sc = h->scal.get<unsigned long long>(8);
    const unsigned long long init[5] = {~0ull, 0ull, 0ull, 0ull, 0ull};
    CK(cudaMemcpyAsync(sc, init, sizeof(init), cudaMemcpyHostToDevice, s));
    launch_split_pack(n, m.row_offset, m.weight, m.diag, m.d, m.rate, m.cum, m.uniform_row, m.rec,
                      sc + 1, reinterpret_cast<unsigned int*>(sc + 2), s);
    after_launch(n ? 1 : 0);
    launch_rate_sum(n, m.rate, m.d, reinterpret_cast<double*>(sc + 3), sc + 4, s);
    after_launch(n ? 1 : 0);
    unsigned long long res[5];
    CK(cudaMemcpyAsync(res, sc, sizeof(res), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    m.dmax = res[1];
    m.any_nonuniform = (res[2] & 0xffffffffull) != 0;
    m.dbar = n > 0 ? (double)nnz / (double)n : 0.0;  // sparse_matrix.cpp:138-141
    {
        double rs;
        std::memcpy(&rs, &res[3], 8);
        m.mean_rate = n > 0 ? rs / (double)n : 0.0;
        std::memcpy(&m.dabs_max, &res[4], 8);
    }
    if (m.any_nonuniform) {
        m.alias_thr = h->alloc<uint32_t>(nnz);
        m.alias_idx = h->alloc<uint32_t>(nnz);
        double* p = h->tmp1.get<double>(nnz);
        uint32_t* sm = h->tmp2.get<uint32_t>(nnz);
        uint32_t* lg = h->tmp3.get<uint32_t>(nnz);
        launch_alias_build(n, m.row_offset, m.weight, m.rate, m.uniform_row, m.alias_thr,
                           m.alias_idx, p, sm, lg, s);
        after_launch(1);
        CK(cudaStreamSynchronize(s));
        h->tmp1.release();
        h->tmp2.release();
        h->tmp3.release();
    }
    m.adj = h->alloc<Edge>(nnz);
    launch_build_adj(nnz, m.neighbor, m.rec, m.adj, s);
    after_launch(nnz ? 1 : 0);
    CK(cudaStreamSynchronize(s));
}

expmc_matrix* build(uint64_t n, const uint64_t* row_ptr, const uint32_t* col, const double* val,
                    const double* diag, int device) {
    if (n >= (1ull << 32)) throw InvalidArg("n must be < 2^32 (NodeId is 32-bit)");
    if (n && !row_ptr) throw InvalidArg("row_ptr is null");
    if (n && row_ptr[0] != 0) throw InvalidArg("row_ptr[0] must be 0");
    for (uint64_t i = 0; i < n; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) throw InvalidArg("row_ptr must be non-decreasing");
    const uint64_t nnz = n ? row_ptr[n] : 0;
    if (nnz >= (1ull << 32)) throw InvalidArg("nnz must be < 2^32");
    if (nnz && (!col || !val)) throw InvalidArg("col / val is null");
    if (diag)
        for (uint64_t i = 0; i < n; ++i)
            if (!std::isfinite(diag[i]))
                throw InvalidArg("non-finite weight at " + pair_str(i, i));

    DeviceGuard g(device);
    auto* h = new expmc_matrix;
    try {
        h->device = device;
        CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->piece_done, cudaEventDisableTiming));
        alloc_split(h, n, nnz);
        DevSplit& m = h->m;
        cudaStream_t s = h->stream;
        if (n) {
            CK(cudaMemcpyAsync(m.row_offset, row_ptr, (n + 1) * 8, cudaMemcpyHostToDevice, s));
            if (diag)
                CK(cudaMemcpyAsync(m.diag, diag, n * 8, cudaMemcpyHostToDevice, s));
            else
                CK(cudaMemsetAsync(m.diag, 0, n * 8, s));
        }
        if (nnz) {
            CK(cudaMemcpyAsync(m.neighbor, col, nnz * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(m.weight, val, nnz * 8, cudaMemcpyHostToDevice, s));
        }
        // small device scalars: [0] err key, [1] dmax, [2] any_nonuniform
        unsigned long long* sc = h->scal.get<unsigned long long>(4);
        const unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
        CK(cudaMemcpyAsync(sc, init, sizeof(init), cudaMemcpyHostToDevice, s));
        launch_validate_csr(n, m.row_offset, m.neighbor, m.weight, sc, s);
        after_launch(n ? 1 : 0);
        unsigned long long res[4];
        CK(cudaMemcpyAsync(res, sc, sizeof(res), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (res[0] != ~0ull) {
            const uint64_t i = res[0] >> 24;
            const int kind = (int)((res[0] >> 20) & 0xf);
            const uint64_t k = row_ptr[i] + (res[0] & 0xfffff);
            const uint64_t j = col[k];
            switch (kind) {  // messages of from_entries, sparse_matrix.cpp:20-51
                case 1:
                    throw InvalidArg("entry " + pair_str(i, j) + " out of range for n = " +
                                     std::to_string(n));
                case 2: throw InvalidArg("non-finite weight at " + pair_str(i, j));
                case 3: throw InvalidArg("explicit zero entry at " + pair_str(i, j));
                case 4:
                    throw InvalidArg("negative off-diagonal weight at " + pair_str(i, j) +
                                     ": no CTMC interpretation");
                case 5:
                    if (k > row_ptr[i] && col[k - 1] == j)
                        throw InvalidArg("duplicate entry at " + pair_str(i, j));
                    throw InvalidArg("CSR row " + std::to_string(i) + " is not sorted by column");
                case 6:
                    throw InvalidArg("diagonal entry at " + pair_str(i, i) +
                                     " stored in the adjacency; pass it in diag");
                default:
                    throw InvalidArg("matrix is not symmetric at " + pair_str(i, j));
            }
        }
        finish_split(h);
    } catch (...) {
        delete h;
        throw;
    }
    return h;
}

// Device-side CSR (from_entries_device output, valid by construction).
expmc_matrix* build_device_csr(uint64_t n, uint64_t nnz, const uint64_t* row_ptr_d,
                               const uint32_t* col_d, const double* val_d, const double* diag_d,
                               int device) {
    DeviceGuard g(device);
    auto* h = new expmc_matrix;
    try {
        h->device = device;
        CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->piece_done, cudaEventDisableTiming));
        alloc_split(h, n, nnz);
        DevSplit& m = h->m;
        cudaStream_t s = h->stream;
        CK(cudaMemcpyAsync(m.row_offset, row_ptr_d, (n + 1) * 8, cudaMemcpyDeviceToDevice, s));
        if (n) CK(cudaMemcpyAsync(m.diag, diag_d, n * 8, cudaMemcpyDeviceToDevice, s));
        if (nnz) {
            CK(cudaMemcpyAsync(m.neighbor, col_d, nnz * 4, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(m.weight, val_d, nnz * 8, cudaMemcpyDeviceToDevice, s));
        }
        h->scal.get<unsigned long long>(4);
        finish_split(h);
    } catch (...) {
        delete h;
        throw;
    }
    return h;
}

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
};

// Device CSR produced by from_entries_device (owned here).
struct DevCsr {
    uint64_t* rp = nullptr;
    uint32_t* col = nullptr;
    double* val = nullptr;
    double* diag = nullptr;
    uint64_t nnz = 0;
    ~DevCsr() {
        cudaFree(rp); cudaFree(col); cudaFree(val); cudaFree(diag);
    }
};

template <class T>
struct DevArr {
    T* p = nullptr;
    ~DevArr() { cudaFree(p); }
};

// from_entries on device arrays; at(k) = (row, col) of input entry k, for the
// reference's messages (sparse_matrix.cpp:20-51).
template <class At>
void device_from_entries(uint64_t n, const uint32_t* r_d, const uint32_t* c_d, const double* w_d,
                         uint64_t ne, cudaStream_t s, At at, DevCsr& out) {
    CK(cudaMalloc(&out.diag, (n ? n : 1) * 8));
    CK(cudaMalloc(&out.rp, (n + 1) * 8));
    unsigned long long err[2] = {~0ull, ~0ull}, dup = 0;
    from_entries_device(n, r_d, c_d, w_d, ne, out.rp, &out.col, &out.val, out.diag, &out.nnz, err,
                        &dup, s);
    CK(cudaGetLastError());
    if (err[0] != ~0ull) {
        const auto e = at(err[0] >> 3);
        const std::string es = "(" + std::to_string(e.first) + ", " + std::to_string(e.second) + ")";
        switch ((int)(err[0] & 7)) {
            case 1:
                throw InvalidArg("entry " + es + " out of range for n = " + std::to_string(n));
            case 2: throw InvalidArg("non-finite weight at " + es);
            case 3: throw InvalidArg("explicit zero entry at " + es);
            default:
                throw InvalidArg("negative off-diagonal weight at " + es + ": no CTMC interpretation");
        }
    }
    if (err[1] != ~0ull)
        throw InvalidArg("duplicate entry at (" + std::to_string(dup >> 32) + ", " +
                         std::to_string(dup & 0xffffffffull) + ")");
    if (out.nnz >= (1ull << 32)) throw InvalidArg("nnz must be < 2^32");
}

// Host entry list -> device CSR.  general: fold both triangles first
// (matrix_market.cpp:136-164; errors are "path:last_line: ..." runtime errors).
void upload_and_convert(uint64_t n, const uint32_t* rows, const uint32_t* cols, const double* w,
                        uint64_t ne, bool general, const std::string& path, uint64_t last_line,
                        cudaStream_t s, DevCsr& out) {
    DevArr<uint32_t> r_d, c_d;
    DevArr<double> w_d;
    CK(cudaMalloc(&r_d.p, (ne ? ne : 1) * 4));
    CK(cudaMalloc(&c_d.p, (ne ? ne : 1) * 4));
    CK(cudaMalloc(&w_d.p, (ne ? ne : 1) * 8));
    if (ne) {
        CK(cudaMemcpyAsync(r_d.p, rows, ne * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(c_d.p, cols, ne * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(w_d.p, w, ne * 8, cudaMemcpyHostToDevice, s));
    }
    if (!general) {
        device_from_entries(n, r_d.p, c_d.p, w_d.p, ne, s,
                            [&](uint64_t k) { return std::make_pair(rows[k], cols[k]); }, out);
        return;
    }
    DevArr<uint32_t> fr, fc;
    DevArr<double> fw;
    uint64_t m = 0;
    unsigned long long err = ~0ull, key = 0;
    fold_general_device(r_d.p, c_d.p, w_d.p, ne, &fr.p, &fc.p, &fw.p, &m, &err, &key, s);
    CK(cudaGetLastError());
    if (err != ~0ull) {
        const std::string at = "(" + std::to_string((key >> 32) + 1) + ", " +
                               std::to_string((key & 0xffffffffull) + 1) + ")";
        throw std::runtime_error(mm_message(path, last_line,
                                            (err & 1) ? "general matrix is not symmetric at " + at
                                                      : "duplicate diagonal entry " + at));
    }
    device_from_entries(n, fr.p, fc.p, fw.p, m, s,
                        [&](uint64_t k) {
                            uint32_t a = 0, b = 0;
                            cudaMemcpy(&a, fr.p + k, 4, cudaMemcpyDeviceToHost);
                            cudaMemcpy(&b, fc.p + k, 4, cudaMemcpyDeviceToHost);
                            return std::make_pair(a, b);
                        },
                        out);
}

// Entry estimator for samples >= 2^29 (walk_vec.cu, entry_big_*): rows and
// outputs are device arrays on stream s; v must already be packed.
void run_entries_big(expmc_matrix* h, const uint32_t* rows_d, uint64_t nrows,
                     const expmc_path_params* p, double* value, double* se, uint64_t* jumps,
                     cudaStream_t s) {
    if (nrows == 0) return;
    if (nrows >= (1ull << 32)) throw InvalidArg("at most 2^32 - 1 rows per call");
    const uint64_t W = p->samples;
    const FastParams fp = fast_params(p, W);
    uint64_t* jc = h->jcnt.get<uint64_t>(nrows + 1);
    uint64_t* off = h->joff.get<uint64_t>(nrows + 1);
    double2* rowc = h->rowc.get<double2>(nrows);
    double* Kr = h->fa.get<double>(nrows);
    double* s1 = h->fa2.get<double>(2 * nrows);
    double* s2 = s1 + nrows;
    unsigned long long* jr = h->pc.get<unsigned long long>(std::max<uint64_t>(nrows, 1));
    launch_entry_big_rows(h->m, rows_d, nrows, fp, jc, rowc, Kr, s1, s2, jr, s);
    CK(cudaMemsetAsync(jc + nrows, 0, 8, s));
    const size_t scan_bytes = scan_u64_temp_bytes(nrows + 1);
    void* scan_tmp = h->scan_tmp.get<unsigned char>(scan_bytes);
    launch_scan_u64(jc, off, nrows + 1, scan_tmp, scan_bytes, s);
    after_launch(2);
    uint64_t J = 0;
    CK(cudaMemcpyAsync(&J, off + nrows, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // jumpers in batches of B; per batch, each jumper's dev and dev^2 go to
    // records in q (= row) order and the deterministic run-sum passes add
    // each row's run to s1 / s2 (batches in order: bitwise reproducible)
    const uint64_t B = 1ull << 26;  // fixed, so repeated calls never regrow
    uint32_t* row_of = h->row_of.get<uint32_t>(B);
    double* dev1 = h->acc.get<double>(2 * B);
    double* dev2 = dev1 + B;
    const size_t rs_bytes = run_sums_temp_bytes(B);
    void* rs_tmp = h->sort_tmp.get<unsigned char>(rs_bytes);
    for (uint64_t q0 = 0; q0 < J; q0 += B) {
        const uint64_t q1 = std::min(J, q0 + B);
        launch_expand_rows(off, nrows, q0, q1, row_of, s);
        launch_entry_big_walk(h->m, rows_d, rowc, Kr, row_of, off, fp, q0, q1, dev1, dev2, jr,
                              s);
        run_sums_sorted(row_of, dev1, q1 - q0, rs_tmp, rs_bytes, s1, s);
        run_sums_sorted(row_of, dev2, q1 - q0, rs_tmp, rs_bytes, s2, s);
        after_launch(6);
    }
    launch_entry_big_finalize(nrows, W, Kr, s1, s2, jr, value, se, jumps, s);
    after_launch(1);
    CK(cudaGetLastError());
}

// Run the entry estimator for host rows / host v; outputs to host.
void run_entries(expmc_matrix* h, const double* v, uint64_t nv, const uint32_t* rows,
                 uint64_t nrows, const expmc_path_params* p, double* value, double* se,
                 uint64_t* jumps, uint64_t* total_jumps = nullptr) {
    validate_params(p);
    const bool fast = p->rng == EXPMC_RNG_PHILOX;
    if (fast) {
        // length here; finiteness on the device (same message), so the host
        // does not scan v on the critical path
        if (nv != h->m.n || (!v && nv)) throw InvalidArg("vector length does not match matrix");
    } else {
        check_vector(h, v, nv);
    }
    const uint64_t n = h->m.n;
    bool bad_row = false;
    if (rows) {
        for (uint64_t r = 0; r < nrows; ++r)
            if (rows[r] >= n) {
                bad_row = true;
                break;
            }
    } else if (nrows != n) {
        throw InvalidArg("rows == NULL requires nrows == n");
    }
    if (bad_row) {
        // the reference checks v before the index (estimator.cpp:172-173):
        // a non-finite v wins, found by the device scan the Philox path uses
        if (fast && n) {
            DeviceGuard g(h->device);
            double* vd = h->vdev.get<double>(n);
            unsigned int* flag = h->scal.get<unsigned int>(4);
            h->vstaged = false;
            CK(cudaMemcpyAsync(vd, v, n * 8, cudaMemcpyHostToDevice, h->stream));
            CK(cudaMemsetAsync(flag, 0, 4, h->stream));
            launch_count_nonfinite(n, vd, flag, h->stream);
            after_launch(1);
            unsigned int bad = 0;
            CK(cudaMemcpyAsync(&bad, flag, 4, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            if (bad) throw InvalidArg("non-finite entry in v");
        }
        throw InvalidArg("entry index out of range");
    }
    // W >= 2^29 walkers per entry: the grouped large-W path (K3 packs walker
    // indices into 29 bits)
#ifdef EXPMC_EXPERIMENTS
    // experiment builds only (make variants): route W < 2^29 through the
    // grouped path too — a different random-number contract, never in the
    // shipped library
    static const bool force_big = getenv("EXPMC_FORCE_BIG") != nullptr;
#else
    constexpr bool force_big = false;
#endif
    const bool big = fast && (p->samples >= (1ull << 29) || force_big);
    if (nrows == 0) return;
    DeviceGuard g(h->device);
    cudaStream_t s = h->stream;
    // EXPMC_DEBUG=2: per-stage device timeline of the call on stderr
    static const bool trace = [] {
        const char* e = getenv("EXPMC_DEBUG");
        return e && atoi(e) >= 2;
    }();
    cudaEvent_t ev[16];
    int nev = 0;
    auto mark = [&](cudaStream_t st) {
        if (!trace || nev >= 16) return;
        cudaEventCreate(&ev[nev]);
        cudaEventRecord(ev[nev++], st);
    };
    const auto t_host0 = std::chrono::steady_clock::now();
    mark(s);
    double* vd = h->vdev.get<double>(n);
    // staged-v reuse (opt-in): same host array, same length, nothing staged
    // since — skip the H2D copy, the finiteness scan and the O(nnz) repack
    const bool reuse = h->vcache && h->vstaged && v == h->vkey_ptr && nv == h->vkey_n;
    if (!reuse) {
        h->vstaged = false;
        CK(cudaMemcpyAsync(vd, v, n * 8, cudaMemcpyHostToDevice, s));
    }
    mark(s);
    if (fast) {
        // E2E path: device finiteness check, then the rows in pieces whose
        // results are copied back on a second stream while the next piece
        // runs (the walker work of different rows is independent).
        // scal: [0] non-finite flag (u32), [1] total jumps (u64)
        unsigned long long* sc = h->scal.get<unsigned long long>(4);
        unsigned int* flag = reinterpret_cast<unsigned int*>(sc);
        unsigned long long* jtot = sc + 1;
        CK(cudaMemsetAsync(sc, 0, 16, s));
        if (!reuse) {
            launch_count_nonfinite(n, vd, flag, s);
            launch_pack_v(n, vd, h->m.rec, s);
            launch_pack_v_adj(h->m.nnz, h->m.neighbor, vd, h->m.adj, s);
            after_launch(3);
            ++h->v_stagings;
        }
        mark(s);
        if (nrows >= (1ull << 30)) throw InvalidArg("at most 2^30 rows per call");
        const uint32_t* rd;
        if (rows) {
            uint32_t* r = h->rows.get<uint32_t>(nrows);
            CK(cudaMemcpyAsync(r, rows, nrows * 4, cudaMemcpyHostToDevice, s));
            rd = r;
        } else {
            rd = all_rows(h);
        }
        double* ov = h->out_val.get<double>(nrows);
        double* os = h->out_se.get<double>(nrows);
        uint64_t* oj = h->out_j.get<uint64_t>(nrows);
        if (big) {
            run_entries_big(h, rd, nrows, p, ov, os, oj, s);
            launch_sum_u64(nrows, oj, jtot, s);
            after_launch(1);
            unsigned long long res[2] = {0, 0};
            CK(cudaMemcpyAsync(value, ov, nrows * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(se, os, nrows * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(jumps, oj, nrows * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(res, sc, 16, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if ((unsigned int)res[0]) throw InvalidArg("non-finite entry in v");
            if (total_jumps) *total_jumps = res[1];
            h->vstaged = true;
            h->vkey_ptr = v;
            h->vkey_n = nv;
            return;
        }
        // Pieces by halving — 1/2, 1/4, ..., and the last two 1/32 of the rows
        // each: a piece's results copy back under the next piece's walk, and
        // only the last, small piece's copy (0.14 ms at config 5, against
        // 0.55 ms for an eighth of the rows) is exposed at the end.
        static const int env_pieces = [] {
            const char* e = getenv("EXPMC_PIECES");  // tests and experiments only
            return e ? atoi(e) : 0;
        }();
        const uint64_t pieces = env_pieces > 0 ? (uint64_t)(env_pieces < 32 ? env_pieces : 32)
                                               : (nrows >= (1ull << 20) ? 6 : 1);
        auto piece_lo = [&](uint64_t k) { return k >= pieces ? nrows : nrows - (nrows >> k); };
        void* scratch =
            h->part.get<unsigned char>(entry_fast_scratch_bytes(piece_lo(1), p->samples));
        FastParams fp = fast_params(p, p->samples);
        for (uint64_t k = 0; k < pieces; ++k) {
            const uint64_t lo = piece_lo(k), hi = piece_lo(k + 1);
            if (hi == lo) continue;
            // all rows (rows == NULL): the contiguous-range form, no row array
            fp.row0 = (uint32_t)lo;
            int kl = launch_entry_fast(h->m, rows ? rd + lo : nullptr, hi - lo, fp, ov + lo,
                                       os + lo, oj + lo, scratch, s);
            if (total_jumps) {
                launch_sum_u64(hi - lo, oj + lo, jtot, s);
                ++kl;
            }
            after_launch(kl);
            mark(s);
            CK(cudaEventRecord(h->piece_done, s));
            CK(cudaStreamWaitEvent(h->copy_stream, h->piece_done, 0));
            CK(cudaMemcpyAsync(value + lo, ov + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost,
                               h->copy_stream));
            CK(cudaMemcpyAsync(se + lo, os + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost,
                               h->copy_stream));
            CK(cudaMemcpyAsync(jumps + lo, oj + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost,
                               h->copy_stream));
        }
        unsigned long long res[2] = {0, 0};
        CK(cudaMemcpyAsync(res, sc, 16, cudaMemcpyDeviceToHost, s));
        mark(h->copy_stream);
        CK(cudaStreamSynchronize(s));
        CK(cudaStreamSynchronize(h->copy_stream));
        if (trace) {
            const double host_ms = std::chrono::duration<double, std::milli>(
                                       std::chrono::steady_clock::now() - t_host0).count();
            fprintf(stderr, "entries trace: host %.3f ms | device:", host_ms);
            for (int k = 1; k < nev; ++k) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, ev[0], ev[k]);
                fprintf(stderr, " %.3f", ms);
            }
            fprintf(stderr, " (H2D v, staged v, pieces..., D2H)\n");
            for (int k = 0; k < nev; ++k) cudaEventDestroy(ev[k]);
        }
        if ((unsigned int)res[0]) throw InvalidArg("non-finite entry in v");
        if (total_jumps) *total_jumps = res[1];
        h->vstaged = true;
        h->vkey_ptr = v;
        h->vkey_n = nv;
        return;
    }
    const uint32_t* rd;
    if (rows) {
        uint32_t* r = h->rows.get<uint32_t>(nrows);
        CK(cudaMemcpyAsync(r, rows, nrows * 4, cudaMemcpyHostToDevice, s));
        rd = r;
    } else {
        rd = all_rows(h);
    }
    double* ov = h->out_val.get<double>(nrows);
    double* os = h->out_se.get<double>(nrows);
    uint64_t* oj = h->out_j.get<uint64_t>(nrows);
    {  // PCG-compat parity walker
        const double dt = p->beta / (double)p->n_steps;
        const bool strang = p->splitting == EXPMC_STRANG;
        double* f = h->fa.get<double>(n);
        launch_node_factors(n, h->m.d, strang ? dt / 2.0 : dt, f, s);
        launch_entry_compat(h->m, vd, rd, nrows, dt, p->n_steps, p->samples,
                            strang ? f : nullptr, f, p->seed, ov, os, oj, s);
        after_launch(2);
    }
    CK(cudaMemcpyAsync(value, ov, nrows * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(se, os, nrows * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(jumps, oj, nrows * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (total_jumps) {
        uint64_t t = 0;
        for (uint64_t r = 0; r < nrows; ++r) t += jumps[r];
        *total_jumps = t;
    }
}

// K4 (Philox): Theorem-2 walkers grouped by start row (walk_vec.cu).
// Multinomial start counts -> per-row never-jumpers (scored in place) and
// jumper counts -> exclusive scan -> jumper walks in batches, whose (end, f)
// records go through the deterministic sort-based per-end reduction.
// Tallies: row partials, then batch partials, added on the host in order.
// Rows [lo, hi) only (a shard): the counts and the global jumper numbering
// are computed for every row — identical on every shard — but only walkers
// starting in [lo, hi) are scored and walked, so the shards of a partition
// run exactly the walkers of the unsharded call.
void run_grouped(expmc_matrix* h, const double* vcum, double v_sum, const expmc_path_params* p,
                 double* vals, double* values_host, double* sum_out, double* sq_out,
                 uint64_t* jumps_out, uint64_t lo = 0, uint64_t hi = ~0ull) {
    cudaStream_t s = h->stream;
    const uint64_t n = h->m.n, M = p->samples;
    const FastParams fp = fast_params(p, M);
    uint64_t* cnt = h->cnt.get<uint64_t>(n);
    uint64_t* jc = h->jcnt.get<uint64_t>(n + 1);
    uint64_t* off = h->joff.get<uint64_t>(n + 1);
    const int levels = launch_start_counts(n, M, vcum, fp.rk, cnt, s);
    after_launch(levels);
    const unsigned rparts = vec_rows_grid();
    // walk tally parts: one per block of the largest batch (B <= 2^28)
    const unsigned parts = std::max(rparts, vec_walk_blocks(std::min<uint64_t>(M, 1ull << 28)));
    double* pa = h->pa.get<double>(parts);
    double* pb = h->pb.get<double>(parts);
    unsigned long long* pc = h->pc.get<unsigned long long>(parts);
    double* tot = h->scal.get<double>(4);
    double2* rowc = h->rowc.get<double2>(n);
    if (hi > n) hi = n;
    launch_vec_rows(h->m, cnt, fp, v_sum, lo, hi, vals, jc, rowc, pa, pb, s);
    CK(cudaMemsetAsync(jc + n, 0, 8, s));
    CK(cudaMemsetAsync(pc, 0, rparts * sizeof(unsigned long long), s));
    launch_final_reduce(pa, pb, pc, rparts, tot, tot + 1,
                        reinterpret_cast<unsigned long long*>(tot + 2), s);
    const size_t scan_bytes = scan_u64_temp_bytes(n + 1);
    void* scan_tmp = h->scan_tmp.get<unsigned char>(scan_bytes);
    launch_scan_u64(jc, off, n + 1, scan_tmp, scan_bytes, s);
    after_launch(3);
    double res[3];
    uint64_t qa = 0, qb = 0;  // the shard's jumpers
    CK(cudaMemcpyAsync(res, tot, sizeof(res), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&qa, off + std::min(lo, n), 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&qb, off + hi, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (qb < qa) qb = qa;
    const uint64_t J = qb - qa;
    double sum = res[0], sq = res[1];
    uint64_t jumps = 0;
    h->last_jumpers = J;
    // batch buffers sized by M (>= J), not by the random J, so repeated calls
    // with the same M never regrow (and re-allocate) them
    uint32_t *rec_end = nullptr, *end_sorted = nullptr;
    double *rec_f = nullptr, *f_sorted = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    // Per-end sums: exact 128-bit fixed point when every f = V w fits
    // (w in [e^{β d_min}, e^{β d_max}]: M f_max 2^s < 2^127 and
    // f_min 2^s >= 2^53), else the sort-based reduction.
    unsigned long long* acc = nullptr;
    int scale_exp = 0;
    if (vals) {
        if (!h->d_range) {
            std::vector<double> hd(n);
            CK(cudaMemcpy(hd.data(), h->m.d, n * 8, cudaMemcpyDeviceToHost));
            h->d_lo = n ? *std::min_element(hd.begin(), hd.end()) : 0.0;
            h->d_hi = n ? *std::max_element(hd.begin(), hd.end()) : 0.0;
            h->d_range = true;
        }
        const double lmax = std::log2(v_sum) + p->beta * h->d_hi / std::log(2.0) + 1.0;
        const double lmin = std::log2(v_sum) + p->beta * h->d_lo / std::log(2.0) - 1.0;
        const double lM = std::log2((double)M);
        const int sx = (int)std::floor(126.0 - lM - lmax);
        const bool fits = std::isfinite(lmax) && std::isfinite(lmin) && lmin + sx >= 54.0 &&
                          sx - 64 > -1000 && sx - 64 < 1000 &&
                          std::getenv("EXPMC_K4_SORT") == nullptr;  // A/B switch
        if (fits) {
            scale_exp = sx;
            acc = h->acc.get<unsigned long long>(2 * n);
            CK(cudaMemsetAsync(acc, 0, n * 16, s));
        }
        h->last_fixed = fits ? 1 : 0;
    }
    // batches of 2^26 jumpers when (end, f) records are kept (sort path),
    // else 2^28 (only the 4-byte start rows per jumper): fewer batch tails
    const uint64_t B = std::min<uint64_t>(M, (vals && !acc) ? 1ull << 26 : 1ull << 28);
    uint32_t* row_of = h->row_of.get<uint32_t>(B);
    if (vals && !acc) {
        rec_end = h->tmp1.get<uint32_t>(B * 2);
        end_sorted = rec_end + B;
        rec_f = h->tmp2.get<double>(B * 2);
        f_sorted = rec_f + B;
        temp_bytes = scatter_sort_temp_bytes(B, n);
        temp = h->sort_tmp.get<unsigned char>(temp_bytes);
    }
    for (uint64_t q0 = qa; q0 < qb; q0 += B) {
        const uint64_t q1 = std::min(qb, q0 + B);
        launch_expand_rows(off, n, q0, q1, row_of, s);
        launch_vec_walk(h->m, rowc, row_of, fp, v_sum, q0, q1, rec_end, rec_f, acc,
                        std::ldexp(1.0, scale_exp - 64), pa, pb, pc, s);
        // batch tallies added to the running totals on the device, in batch
        // order (the same fp sequence as adding them on the host)
        launch_final_reduce_acc(pa, pb, pc, vec_walk_blocks(q1 - q0), tot, tot + 1,
                                reinterpret_cast<unsigned long long*>(tot + 2), s);
        after_launch(3);
        if (vals && !acc) {
            scatter_sort_accumulate(rec_end, rec_f, end_sorted, f_sorted, q1 - q0, n, temp,
                                    temp_bytes, vals, s);
            after_launch(3);
            CK(cudaGetLastError());
        }
    }
    CK(cudaMemcpyAsync(res, tot, sizeof(res), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::memcpy(&jumps, &res[2], 8);
    sum = res[0];
    sq = res[1];
    CK(cudaGetLastError());
    if (acc) {
        launch_fixed_to_values(acc, n, std::ldexp(1.0, -scale_exp), vals, s);
        after_launch(1);
    }
    if (vals) {
        launch_scale(n, vals, 1.0 / (double)M, s);
        after_launch(1);
        CK(cudaMemcpyAsync(values_host, vals, n * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    *sum_out = sum;
    *sq_out = sq;
    *jumps_out = jumps;
}

// Theorem 2 walkers (vector / tc).  start_mode 0 uniform, 1 categorical.
void run_scatter(expmc_matrix* h, int start_mode, const std::vector<double>* cum, double v_sum,
                 const expmc_path_params* p, double* values_host, double* sum_out,
                 double* sq_out, uint64_t* jumps_out, uint64_t lo = 0, uint64_t hi = ~0ull) {
    DeviceGuard g(h->device);
    cudaStream_t s = h->stream;
    const uint64_t n = h->m.n;
    double* vals = nullptr;
    if (values_host) {
        vals = h->values.get<double>(n);
        CK(cudaMemsetAsync(vals, 0, n * 8, s));
    }
    const double* vc = nullptr;
    if (start_mode == 1) {
        double* c = h->vcum.get<double>(n);
        CK(cudaMemcpyAsync(c, cum->data(), n * 8, cudaMemcpyHostToDevice, s));
        vc = c;
    }
    if (p->rng == EXPMC_RNG_PHILOX) {
        run_grouped(h, vc, v_sum, p, vals, values_host, sum_out, sq_out, jumps_out, lo, hi);
        return;
    }
    const unsigned parts = scatter_compat_grid();
    double* pa = h->pa.get<double>(parts);
    double* pb = h->pb.get<double>(parts);
    unsigned long long* pc = h->pc.get<unsigned long long>(parts);
    const double dt = p->beta / (double)p->n_steps;
    const bool strang = p->splitting == EXPMC_STRANG;
    double* fac = h->fa.get<double>(n);
    launch_node_factors(n, h->m.d, strang ? dt / 2.0 : dt, fac, s);
    after_launch(1);
    // walkers in batches; per batch: (end, f) records -> stable sort by end
    // -> per-run sequential sums added to values[] (deterministic, no atomics);
    // scalar tallies reduced per batch and added on the host in batch order
    const uint64_t M = p->samples;
    const uint64_t B = vals ? std::min<uint64_t>(M, 1ull << 25) : M;
    uint32_t *rec_end = nullptr, *end_sorted = nullptr;
    double *rec_f = nullptr, *f_sorted = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    if (vals) {
        rec_end = h->tmp1.get<uint32_t>(B * 2);
        end_sorted = rec_end + B;
        rec_f = h->tmp2.get<double>(B * 2);
        f_sorted = rec_f + B;
        temp_bytes = scatter_sort_temp_bytes(B, n);
        temp = h->sort_tmp.get<unsigned char>(temp_bytes);
    }
    double* tot = h->scal.get<double>(4);
    double sum = 0.0, sq = 0.0;
    uint64_t jumps = 0;
    for (uint64_t l0 = 0; l0 < M; l0 += B) {
        const uint64_t lend = std::min(M, l0 + B);
        // Lie weight on the state each segment leaves from (estimator.cpp:228-231)
        launch_scatter_compat(h->m, start_mode, vc, v_sum, dt, p->n_steps, M, fac,
                              strang ? fac : nullptr, p->seed, l0, lend, rec_end, rec_f, pa, pb,
                              pc, s);
        launch_final_reduce(pa, pb, pc, parts, tot, tot + 1,
                            reinterpret_cast<unsigned long long*>(tot + 2), s);
        after_launch(2);
        if (vals) {
            scatter_sort_accumulate(rec_end, rec_f, end_sorted, f_sorted, lend - l0, n, temp,
                                    temp_bytes, vals, s);
            after_launch(3);
            CK(cudaGetLastError());
        }
        double res[3];
        CK(cudaMemcpyAsync(res, tot, sizeof(res), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        uint64_t j;
        std::memcpy(&j, &res[2], 8);
        sum += res[0];
        sq += res[1];
        jumps += j;
    }
    if (vals) {
        launch_scale(n, vals, 1.0 / (double)M, s);
        after_launch(1);
        CK(cudaMemcpyAsync(values_host, vals, n * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    *sum_out = sum;
    *sq_out = sq;
    *jumps_out = jumps;
}

void finalize(double sum, double sum_sq, uint64_t ms, double* value, double* se) {
    // estimator.cpp:76-89
    const double mm = (double)ms;
    *value = sum / mm;
    *se = 0.0;
    if (ms > 1) {
        const double var = std::max(0.0, (sum_sq - sum * sum / mm) / (mm - 1.0));
        *se = std::sqrt(var / mm);
    }
}

// y = exp(tau * (B + shift I)) x by Taylor on device buffers; B = A (mode 0)
// or -L (mode 1).  x is overwritten with the result.
void taylor_step(expmc_matrix* h, int mode, double shift, double tau, double tol, double* x,
                 double* term, double* tmp, cudaStream_t s) {
    const uint64_t n = h->m.n;
    const unsigned parts = norm_parts();
    double* part = h->pa.get<double>(parts);
    std::vector<double> hp(parts);
    auto norm = [&](const double* y) {
        launch_norm_inf(n, y, part, parts, s);
        after_launch(1);
        CK(cudaMemcpyAsync(hp.data(), part, parts * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double m = 0.0;
        for (double v : hp) m = std::max(m, v);
        return m;
    };
    CK(cudaMemcpyAsync(term, x, n * 8, cudaMemcpyDeviceToDevice, s));
    for (int k = 1; k <= 200; ++k) {
        launch_spmv(h->m, mode, shift, term, tmp, s);
        after_launch(1);
        launch_scale(n, tmp, tau / (double)k, s);
        after_launch(1);
        std::swap(term, tmp);
        launch_axpy(n, 1.0, term, x, s);
        after_launch(1);
        const double nt = norm(term);
        if (nt <= tol * norm(x)) return;
    }
}

// exp(t (B)) x with B = A (mode 0) or -L (mode 1), Gershgorin-shifted and
// split into substeps of norm <= 2.
void expmv_dev(expmc_matrix* h, int mode, double t, double tol, double* x, cudaStream_t s) {
    const uint64_t n = h->m.n;
    if (n == 0) return;
    if (h->h_rate.size() != n) {
        h->h_rate.resize(n);
        h->h_diag.resize(n);
        CK(cudaMemcpyAsync(h->h_rate.data(), h->m.rate, n * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(h->h_diag.data(), h->m.diag, n * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    double lo = INFINITY, hi = -INFINITY;
    for (uint64_t i = 0; i < n; ++i) {
        const double c = mode == 0 ? h->h_diag[i] : -h->h_rate[i];
        lo = std::min(lo, c - h->h_rate[i]);
        hi = std::max(hi, c + h->h_rate[i]);
    }
    const double mu = 0.5 * (lo + hi), rad = 0.5 * (hi - lo);
    const uint64_t steps = std::max<uint64_t>(1, (uint64_t)std::ceil(std::fabs(t) * rad / 2.0));
    const double tau = t / (double)steps;
    double* term = h->tmp1.get<double>(n);
    double* tmp = h->tmp2.get<double>(n);
    for (uint64_t k = 0; k < steps; ++k) taylor_step(h, mode, -mu, tau, tol, x, term, tmp, s);
    launch_scale(n, x, std::exp(t * mu), s);
    after_launch(1);
}

}  // namespace

namespace {
// vector_estimate's checks and StartSampler table (estimator.cpp:208-222,
// :92-128): returns V; cum stays empty for the exact-uniform case.
double vector_setup(expmc_matrix* h, const double* v, uint64_t nv, const expmc_path_params* p,
                    std::vector<double>& cum) {
    if (!h) throw InvalidArg("matrix handle is null");
    validate_params(p);
    check_vector(h, v, nv);
    double v_sum = 0.0;  // estimator.cpp:212-222
    for (uint64_t k = 0; k < nv; ++k) {
        if (v[k] < 0.0) throw InvalidArg("vector_estimate requires v >= 0 entrywise");
        v_sum += v[k];
    }
    if (!(v_sum > 0.0)) throw InvalidArg("vector_estimate requires sum(v) > 0");
    bool uniform = true;  // exact uniform test (estimator.cpp:95-100)
    for (uint64_t k = 0; k < nv; ++k)
        if (v[k] != v[0]) { uniform = false; break; }
    cum.clear();
    if (!uniform) {
        cum.resize(nv);
        double acc = 0.0;
        for (uint64_t k = 0; k < nv; ++k) { acc += v[k]; cum[k] = acc; }
    }
    return v_sum;
}

void check_shard(const expmc_matrix* h, const expmc_path_params* p, uint64_t lo, uint64_t hi) {
    if (lo > hi || hi > h->m.n) throw InvalidArg("row range out of bounds");
    if (p->rng != EXPMC_RNG_PHILOX) throw InvalidArg("row shards need the Philox engine");
}
}  // namespace

extern "C" {

const char* expmc_cuda_last_error(void) { return g_err_slot.s; }
int expmc_cuda_abi_version(void) { return 1; }
uint64_t expmc_cuda_launch_count(void) { return g_launches.load(); }
uint32_t expmc_cuda_entry_slots(uint64_t walkers) {
    return 32u * (uint32_t)entry_fast_wpr(walkers);
}

int expmc_cuda_create_from_csr(uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                               const double* val, const double* diag, int device,
                               expmc_matrix** out) {
    return guarded([&] {
        if (!out) throw InvalidArg("out is null");
        *out = build(n, row_ptr, col, val, diag, device);
    });
}

int expmc_cuda_rank(const double* scores, uint64_t n, int device, uint32_t* order) {
    // rank(), proj/src/metrics.cpp:10-25
    return guarded([&] {
        if (n >= (1ull << 31)) throw InvalidArg("rank: at most 2^31 scores");
        if (n && (!scores || !order)) throw InvalidArg("rank: null array");
        DeviceGuard g(device);
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        const bool ok = rank_device(scores, n, order, s);
        after_launch(2);
        cudaStreamDestroy(s);
        if (!ok) throw InvalidArg("rank: NaN score");
    });
}

int expmc_cuda_isim(const uint32_t* order_x, const uint32_t* order_y, uint64_t nx, uint64_t ny,
                    double top_fraction, int device, double* out) {
    // isim(), proj/src/metrics.cpp:27-55 (same checks and messages)
    return guarded([&] {
        if (nx != ny) throw InvalidArg("isim: length mismatch");
        if (!(top_fraction > 0.0) || top_fraction > 1.0)
            throw InvalidArg("isim: top_fraction must be in (0, 1]");
        if (nx == 0) throw InvalidArg("isim: empty ranking");
        if (nx >= (1ull << 31)) throw InvalidArg("isim: at most 2^31 nodes");
        for (uint64_t i = 0; i < nx; ++i)
            if (order_x[i] >= nx || order_y[i] >= nx) throw InvalidArg("isim: order out of range");
        const uint64_t k = (uint64_t)std::ceil(top_fraction * (double)nx);
        DeviceGuard g(device);
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        *out = isim_device(order_x, order_y, nx, k, s);
        after_launch(5);
        cudaStreamDestroy(s);
    });
}

int expmc_cuda_create_from_entries(uint64_t n, const uint32_t* rows, const uint32_t* cols,
                                   const double* w, uint64_t ne, int device, expmc_matrix** out) {
    // SparseSymmetric::from_entries (sparse_matrix.cpp:18-85) on the device
    return guarded([&] {
        if (!out) throw InvalidArg("out is null");
        if (n >= (1ull << 32)) throw InvalidArg("n must be < 2^32 (NodeId is 32-bit)");
        if (ne >= (1ull << 30)) throw InvalidArg("at most 2^30 entries");
        if (ne && (!rows || !cols || !w)) throw InvalidArg("entry arrays are null");
        DeviceGuard g(device);
        Stream s;
        DevCsr csr;
        upload_and_convert(n, rows, cols, w, ne, false, "", 0, s.s, csr);
        *out = build_device_csr(n, csr.nnz, csr.rp, csr.col, csr.val, csr.diag, device);
    });
}

int expmc_cuda_create_from_mm(const char* path, int device, expmc_matrix** out) {
    // load_matrix_market (matrix_market.cpp:51-165) -> split, on the device
    return guarded([&] {
        if (!out) throw InvalidArg("out is null");
        expmc_mm mm;
        mm_parse(path, mm);
        DeviceGuard g(device);
        Stream s;
        DevCsr csr;
        upload_and_convert(mm.n, mm.r.data(), mm.c.data(), mm.w.data(), mm.r.size(), mm.general,
                           mm.path, mm.last_line, s.s, csr);
        *out = build_device_csr(mm.n, csr.nnz, csr.rp, csr.col, csr.val, csr.diag, device);
    });
}

int expmc_cuda_mm_load(const char* path, int device, expmc_csr** out) {
    // load_matrix_market -> the SparseSymmetric adjacency, back on the host
    return guarded([&] {
        if (!out) throw InvalidArg("out is null");
        expmc_mm mm;
        mm_parse(path, mm);
        DeviceGuard g(device);
        Stream s;
        DevCsr csr;
        upload_and_convert(mm.n, mm.r.data(), mm.c.data(), mm.w.data(), mm.r.size(), mm.general,
                           mm.path, mm.last_line, s.s, csr);
        auto* c = new expmc_csr;
        try {
            c->n = mm.n;
            c->row_ptr.resize(mm.n + 1);
            c->col.resize(csr.nnz);
            c->val.resize(csr.nnz);
            c->diag.resize(mm.n);
            CK(cudaMemcpyAsync(c->row_ptr.data(), csr.rp, (mm.n + 1) * 8, cudaMemcpyDeviceToHost, s.s));
            CK(cudaMemcpyAsync(c->diag.data(), csr.diag, mm.n * 8, cudaMemcpyDeviceToHost, s.s));
            if (csr.nnz) {
                CK(cudaMemcpyAsync(c->col.data(), csr.col, csr.nnz * 4, cudaMemcpyDeviceToHost, s.s));
                CK(cudaMemcpyAsync(c->val.data(), csr.val, csr.nnz * 8, cudaMemcpyDeviceToHost, s.s));
            }
            CK(cudaStreamSynchronize(s.s));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int expmc_cuda_create_from_split(uint64_t n, const uint64_t* row_offset,
                                 const uint32_t* neighbor, const double* weight,
                                 const double* diag, int device, expmc_matrix** out) {
    return expmc_cuda_create_from_csr(n, row_offset, neighbor, weight, diag, device, out);
}

int expmc_cuda_destroy(expmc_matrix* m) {
    return guarded([&] {
        if (!m) return;
        DeviceGuard g(m->device);
        cudaStreamSynchronize(m->stream);
        delete m;
    });
}

int expmc_cuda_matrix_info(const expmc_matrix* h, uint64_t* n, uint64_t* nnz, double* dbar,
                           uint64_t* dmax, int32_t* any_nonuniform, int32_t* device) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        if (n) *n = h->m.n;
        if (nnz) *nnz = h->m.nnz;
        if (dbar) *dbar = h->m.dbar;
        if (dmax) *dmax = h->m.dmax;
        if (any_nonuniform) *any_nonuniform = h->m.any_nonuniform ? 1 : 0;
        if (device) *device = h->device;
    });
}

int expmc_cuda_split_export(const expmc_matrix* h, double* diag, double* d, double* rate,
                            uint64_t* row_offset, uint32_t* neighbor, double* weight,
                            double* cum, uint8_t* uniform_row) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        DeviceGuard g(h->device);
        const DevSplit& m = h->m;
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            if (dst && bytes) CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
        };
        cp(diag, m.diag, m.n * 8);
        cp(d, m.d, m.n * 8);
        cp(rate, m.rate, m.n * 8);
        cp(row_offset, m.row_offset, (m.n + 1) * 8);
        cp(neighbor, m.neighbor, m.nnz * 4);
        cp(weight, m.weight, m.nnz * 8);
        cp(cum, m.cum, m.nnz * 8);
        cp(uniform_row, m.uniform_row, m.n);
    });
}

int expmc_cuda_alias_export(const expmc_matrix* h, uint32_t* thr, uint32_t* alias) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        DeviceGuard g(h->device);
        const DevSplit& m = h->m;
        if (!m.any_nonuniform) {  // uniform everywhere: identity tables
            std::vector<uint64_t> ro(m.n + 1);
            if (m.n) CK(cudaMemcpy(ro.data(), m.row_offset, (m.n + 1) * 8, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < m.n; ++i)
                for (uint64_t k = ro[i]; k < ro[i + 1]; ++k) {
                    if (thr) thr[k] = 0xffffffffu;
                    if (alias) alias[k] = (uint32_t)(k - ro[i]);
                }
            return;
        }
        if (thr) CK(cudaMemcpy(thr, m.alias_thr, m.nnz * 4, cudaMemcpyDeviceToHost));
        if (alias) CK(cudaMemcpy(alias, m.alias_idx, m.nnz * 4, cudaMemcpyDeviceToHost));
    });
}

int expmc_cuda_records_export(const expmc_matrix* h, void* out) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        DeviceGuard g(h->device);
        if (h->m.n) CK(cudaMemcpy(out, h->m.rec, h->m.n * sizeof(RowRec), cudaMemcpyDeviceToHost));
    });
}

int expmc_cuda_entry_estimate(expmc_matrix* h, const double* v, uint64_t nv, uint32_t i,
                              const expmc_path_params* p, expmc_estimate* out) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        // run_entries applies the reference's checks in its order
        // (estimator.cpp:171-173); the Philox path scans v for finiteness on
        // the device when it stages v, not with an O(n) host loop per call
        double val, se;
        uint64_t j;
        run_entries(h, v, nv, &i, 1, p, &val, &se, &j);
        out->value = val;
        out->std_error = se;
        out->samples_used = p->samples;
        out->total_jumps = j;
    });
}

int expmc_cuda_entries(expmc_matrix* h, const double* v, uint64_t nv, const uint32_t* rows,
                       uint64_t nrows, const expmc_path_params* p, double* value,
                       double* std_error, uint64_t* jumps, uint64_t* total_jumps) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        if (total_jumps) *total_jumps = 0;
        run_entries(h, v, nv, rows, nrows, p, value, std_error, jumps, total_jumps);
    });
}

int expmc_cuda_vector_estimate(expmc_matrix* h, const double* v, uint64_t nv,
                               const expmc_path_params* p, double* values,
                               double* std_error_global, uint64_t* total_jumps,
                               double* v_sum_out) {
    return guarded([&] {
        std::unique_lock<std::mutex> lk;
        if (h) lk = std::unique_lock<std::mutex>(h->mu);
        std::vector<double> cum;
        const double v_sum = vector_setup(h, v, nv, p, cum);
        double sum, sq;
        uint64_t j;
        run_scatter(h, cum.empty() ? 0 : 1, &cum, v_sum, p, values, &sum, &sq, &j);
        double value;
        finalize(sum, sq, p->samples, &value, std_error_global);
        *total_jumps = j;
        *v_sum_out = v_sum;
    });
}

int expmc_cuda_vector_estimate_rows(expmc_matrix* h, const double* v, uint64_t nv,
                                    const expmc_path_params* p, uint64_t row_lo,
                                    uint64_t row_hi, double* values, double* sum,
                                    double* sum_sq, uint64_t* total_jumps) {
    return guarded([&] {
        std::unique_lock<std::mutex> lk;
        if (h) lk = std::unique_lock<std::mutex>(h->mu);
        std::vector<double> cum;
        const double v_sum = vector_setup(h, v, nv, p, cum);
        check_shard(h, p, row_lo, row_hi);
        run_scatter(h, cum.empty() ? 0 : 1, &cum, v_sum, p, values, sum, sum_sq, total_jumps,
                    row_lo, row_hi);
    });
}

int expmc_cuda_tc_estimate_rows(expmc_matrix* h, const expmc_path_params* p, uint64_t row_lo,
                                uint64_t row_hi, double* sum, double* sum_sq,
                                uint64_t* total_jumps) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        validate_params(p);
        if (h->m.n == 0) throw InvalidArg("empty matrix");  // estimator.cpp:283
        check_shard(h, p, row_lo, row_hi);
        run_scatter(h, 0, nullptr, (double)h->m.n, p, nullptr, sum, sum_sq, total_jumps, row_lo,
                    row_hi);
    });
}

int expmc_cuda_tc_estimate(expmc_matrix* h, const expmc_path_params* p, expmc_estimate* out) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        validate_params(p);
        if (h->m.n == 0) throw InvalidArg("empty matrix");  // estimator.cpp:283
        double sum, sq;
        uint64_t j;
        run_scatter(h, 0, nullptr, (double)h->m.n, p, nullptr, &sum, &sq, &j);
        finalize(sum, sq, p->samples, &out->value, &out->std_error);
        out->samples_used = p->samples;
        out->total_jumps = j;
    });
}

int expmc_cuda_set_v_device(expmc_matrix* h, const double* v_dev, uint64_t nv, void* stream) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        if (nv != h->m.n) throw InvalidArg("vector length does not match matrix");
        h->vstaged = false;  // the packed v now comes from device memory
        DeviceGuard g(h->device);
        cudaStream_t s = pick_stream(h, stream);
        unsigned int* flag = h->scal.get<unsigned int>(4);
        CK(cudaMemsetAsync(flag, 0, 4, s));
        launch_count_nonfinite(nv, v_dev, flag, s);
        after_launch(1);
        unsigned int bad = 0;
        CK(cudaMemcpyAsync(&bad, flag, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (bad) throw InvalidArg("non-finite entry in v");
        launch_pack_v(nv, v_dev, h->m.rec, s);
        launch_pack_v_adj(h->m.nnz, h->m.neighbor, v_dev, h->m.adj, s);
        after_launch(2);
    });
}

int expmc_cuda_entries_device(expmc_matrix* h, const uint32_t* rows_dev, uint64_t nrows,
                              const expmc_path_params* p, double* value_dev,
                              double* std_error_dev, uint64_t* jumps_dev, void* stream) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        validate_params(p);
        if (p->rng != EXPMC_RNG_PHILOX)
            throw InvalidArg("entries_device supports the Philox walker only");
        DeviceGuard g(h->device);
        if (p->samples >= (1ull << 29)) {  // large-W grouped path (synchronises the stream)
            run_entries_big(h, rows_dev, nrows, p, value_dev, std_error_dev, jumps_dev,
                            pick_stream(h, stream));
            return;
        }
        if (nrows >= (1ull << 30)) throw InvalidArg("at most 2^30 rows per call");
        // scratch is owned by the handle: one stream per handle at a time
        void* scratch = h->part.get<unsigned char>(entry_fast_scratch_bytes(nrows, p->samples));
        const int k = launch_entry_fast(h->m, rows_dev, nrows, fast_params(p, p->samples),
                                        value_dev, std_error_dev, jumps_dev, scratch,
                                        pick_stream(h, stream));
        after_launch(k);
    });
}

int expmc_cuda_entries_device_range(expmc_matrix* h, uint64_t row_lo, uint64_t nrows,
                                    const expmc_path_params* p, double* value_dev,
                                    double* std_error_dev, uint64_t* jumps_dev, void* stream) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        validate_params(p);
        if (p->rng != EXPMC_RNG_PHILOX)
            throw InvalidArg("entries_device supports the Philox walker only");
        if (row_lo > h->m.n || nrows > h->m.n - row_lo) throw InvalidArg("entry index out of range");
        DeviceGuard g(h->device);
        if (p->samples >= (1ull << 29)) {  // large-W grouped path: needs the row list
            run_entries_big(h, all_rows(h) + row_lo, nrows, p, value_dev, std_error_dev,
                            jumps_dev, pick_stream(h, stream));
            return;
        }
        if (nrows >= (1ull << 30)) throw InvalidArg("at most 2^30 rows per call");
        void* scratch = h->part.get<unsigned char>(entry_fast_scratch_bytes(nrows, p->samples));
        FastParams fp = fast_params(p, p->samples);
        fp.row0 = (uint32_t)row_lo;
        const int k = launch_entry_fast(h->m, nullptr, nrows, fp, value_dev, std_error_dev,
                                        jumps_dev, scratch, pick_stream(h, stream));
        after_launch(k);
    });
}

int expmc_cuda_set_v_cache(expmc_matrix* h, int enable) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        h->vcache = enable != 0;
        h->vstaged = false;  // the first call after (re-)enabling stages v
    });
}

int expmc_cuda_invalidate_v(expmc_matrix* h) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        h->vstaged = false;
    });
}

int expmc_cuda_v_stagings(const expmc_matrix* h, uint64_t* count) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        if (count) *count = h->v_stagings;
    });
}

int expmc_cuda_entries_multi(expmc_matrix* const* handles, int nh, const double* v, uint64_t nv,
                             const uint32_t* rows, uint64_t nrows, const expmc_path_params* p,
                             double* value, double* std_error, uint64_t* jumps,
                             uint64_t* total_jumps) {
    // Rows in nh contiguous, equal-count shards, shard k on
    // handles[k] (one replica per GPU, or several handles on one GPU), each
    // driven by its own host thread: the H2D of v, the walk and the D2H of
    // the shard's slice straight into the caller's arrays run concurrently
    // on all devices.  Keyed RNG + the fixed per-row reduction make the
    // result bitwise identical to a single-handle call, for any nh.
    return guarded([&] {
        if (nh < 1 || !handles) throw InvalidArg("need at least one matrix handle");
        for (int k = 0; k < nh; ++k) {
            if (!handles[k]) throw InvalidArg("matrix handle is null");
            if (handles[k]->m.n != handles[0]->m.n || handles[k]->m.nnz != handles[0]->m.nnz)
                throw InvalidArg("shard handles hold different matrices");
            for (int j = 0; j < k; ++j)
                if (handles[j] == handles[k]) throw InvalidArg("shard handles must be distinct");
        }
        if (total_jumps) *total_jumps = 0;
        const uint64_t n = handles[0]->m.n;
        if (!rows && nrows != n) throw InvalidArg("rows == NULL requires nrows == n");
        std::vector<uint32_t> iota;
        const uint32_t* rr = rows;
        if (!rows && nh > 1) {  // shards of the full vector need explicit rows
            iota.resize(n);
            for (uint64_t i = 0; i < n; ++i) iota[i] = (uint32_t)i;
            rr = iota.data();
        }
        std::vector<int> rc(nh, EXPMC_OK);
        std::vector<std::string> msg(nh);
        std::vector<uint64_t> tj(nh, 0);
        auto shard = [&](int k) {
            const uint64_t lo = nrows * k / nh, hi = nrows * (k + 1) / nh;
            rc[k] = guarded([&] {
                std::lock_guard<std::mutex> lk(handles[k]->mu);
                run_entries(handles[k], v, nv, rr ? rr + lo : nullptr, hi - lo, p, value + lo,
                            std_error + lo, jumps + lo, &tj[k]);
            });
            if (rc[k] != EXPMC_OK) msg[k] = g_err_slot.s;
        };
        std::vector<std::thread> pool;
        for (int k = 1; k < nh; ++k) pool.emplace_back(shard, k);
        shard(0);
        for (auto& t : pool) t.join();
        for (int k = 0; k < nh; ++k)
            if (rc[k] != EXPMC_OK) {
                set_err(msg[k]);
                if (rc[k] == EXPMC_INVALID_ARGUMENT) throw InvalidArg(msg[k]);
                if (rc[k] == EXPMC_CUDA_ERROR) throw CudaErr(msg[k]);
                throw std::runtime_error(msg[k]);
            }
        if (total_jumps)
            for (uint64_t t : tj) *total_jumps += t;
    });
}

int expmc_cuda_exp_law(int device, uint64_t count, uint64_t seed, double bin_width,
                       uint32_t nbins, uint64_t* hist, double* moments) {
    return guarded([&] {
        if (count % 4 || nbins < 2 || nbins > 8192 || !(bin_width > 0.0) || !hist || !moments)
            throw InvalidArg("exp_law: needs count % 4 == 0, 2 <= nbins <= 8192, width > 0");
        DeviceGuard g(device);
        unsigned long long* d = nullptr;
        CK(cudaMalloc(&d, (nbins + 2) * sizeof(unsigned long long)));
        CK(cudaMemset(d, 0, (nbins + 2) * sizeof(unsigned long long)));
        launch_exp_law(count, seed, bin_width, nbins, d, d + nbins, nullptr);
        after_launch(1);
        std::vector<unsigned long long> hv(nbins + 2);
        const cudaError_t e = cudaMemcpy(hv.data(), d, hv.size() * 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
        CK(e);
        for (uint32_t b = 0; b < nbins; ++b) hist[b] = hv[b];
        moments[0] = std::ldexp((double)hv[nbins], -30);
        moments[1] = std::ldexp((double)hv[nbins + 1], -30);
    });
}

int expmc_cuda_last_k4_stats(const expmc_matrix* h, uint64_t* jumpers, int* fixed_point) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        if (jumpers) *jumpers = h->last_jumpers;
        if (fixed_point) *fixed_point = h->last_fixed;
    });
}

int expmc_cuda_binomial_samples(int device, uint64_t trials, double p, uint64_t count,
                                uint64_t seed, uint64_t* out) {
    return guarded([&] {
        if (!out && count) throw InvalidArg("out is null");
        if (!(p >= 0.0 && p <= 1.0)) throw InvalidArg("p must be in [0, 1]");
        DeviceGuard g(device);
        uint64_t* d = nullptr;
        CK(cudaMalloc(&d, (count ? count : 1) * 8));
        launch_binomial_debug(trials, p, count,
                              philox_keys((uint32_t)seed, (uint32_t)(seed >> 32)), d, 0);
        after_launch(count ? 1 : 0);
        const cudaError_t e = cudaMemcpy(out, d, count * 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
        CK(e);
    });
}

int expmc_cuda_start_counts(expmc_matrix* h, const double* v, uint64_t nv, uint64_t samples,
                            uint64_t seed, uint64_t* counts) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        if (!counts) throw InvalidArg("counts is null");
        DeviceGuard g(h->device);
        cudaStream_t s = h->stream;
        const uint64_t n = h->m.n;
        if (n == 0) throw InvalidArg("empty matrix");
        const double* vc = nullptr;
        if (v) {
            check_vector(h, v, nv);
            std::vector<double> cum(n);
            double acc = 0.0;
            for (uint64_t k = 0; k < n; ++k) {
                if (v[k] < 0.0) throw InvalidArg("vector_estimate requires v >= 0 entrywise");
                acc += v[k];
                cum[k] = acc;
            }
            if (!(acc > 0.0)) throw InvalidArg("vector_estimate requires sum(v) > 0");
            bool uniform = true;  // StartSampler's exact uniform test (estimator.cpp:95-100)
            for (uint64_t k = 0; k < n; ++k)
                if (v[k] != v[0]) { uniform = false; break; }
            if (uniform) v = nullptr;
        }
        if (v) {
            std::vector<double> cum(n);
            double acc = 0.0;
            for (uint64_t k = 0; k < n; ++k) { acc += v[k]; cum[k] = acc; }
            double* c = h->vcum.get<double>(n);
            CK(cudaMemcpyAsync(c, cum.data(), n * 8, cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
            vc = c;
        }
        uint64_t* cnt = h->cnt.get<uint64_t>(n);
        after_launch(launch_start_counts(n, samples, vc,
                                         philox_keys((uint32_t)seed, (uint32_t)(seed >> 32)),
                                         cnt, s));
        CK(cudaMemcpyAsync(counts, cnt, n * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

int expmc_cuda_gather_ceiling_device(expmc_matrix* h, const uint32_t* rows_dev, uint64_t nrows,
                                     uint32_t chains_per_row, uint32_t chain_len,
                                     void* stream) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        DeviceGuard g(h->device);
        unsigned long long* sink = h->scal.get<unsigned long long>(4);
        launch_gather_ceiling(h->m, rows_dev, nrows, chains_per_row, chain_len, 0x2545F491u,
                              sink, pick_stream(h, stream));
        after_launch(1);
    });
}

int expmc_cuda_expmv(expmc_matrix* h, const double* v, uint64_t nv, double t, double tol,
                     double* out) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        check_vector(h, v, nv);
        if (!std::isfinite(t)) throw InvalidArg("t must be finite");
        if (!(tol > 0.0)) throw InvalidArg("tol must be positive");
        DeviceGuard g(h->device);
        cudaStream_t s = h->stream;
        const uint64_t n = h->m.n;
        double* x = h->tmp3.get<double>(n);
        CK(cudaMemcpyAsync(x, v, n * 8, cudaMemcpyHostToDevice, s));
        expmv_dev(h, 0, t, tol, x, s);
        CK(cudaMemcpyAsync(out, x, n * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

int expmc_cuda_lambda_max(expmc_matrix* h, uint64_t power_iters, double* lambda_max,
                          double* rel_change) {
    // stats(): proj/src/sparse_matrix.cpp:176-217 (power iteration on A
    // shifted by its Gershgorin lower bound), on the device.
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        const uint64_t n = h->m.n;
        *lambda_max = 0.0;
        if (rel_change) *rel_change = 0.0;
        if (power_iters == 0 || n == 0) return;
        DeviceGuard g(h->device);
        cudaStream_t s = h->stream;
        if (h->h_rate.size() != n) {
            h->h_rate.resize(n);
            h->h_diag.resize(n);
            CK(cudaMemcpyAsync(h->h_rate.data(), h->m.rate, n * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(h->h_diag.data(), h->m.diag, n * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        double shift = 0.0;
        for (uint64_t i = 0; i < n; ++i) shift = std::max(shift, h->h_rate[i] - h->h_diag[i]);
        double* x = h->tmp1.get<double>(n);
        double* y = h->tmp2.get<double>(n);
        std::vector<double> x0(n, 1.0 / std::sqrt((double)n));
        CK(cudaMemcpyAsync(x, x0.data(), n * 8, cudaMemcpyHostToDevice, s));
        const unsigned parts = norm_parts();
        double* pa = h->pa.get<double>(parts);
        double* pb = h->pb.get<double>(parts);
        unsigned long long* pc = h->pc.get<unsigned long long>(parts);
        double* tot = h->scal.get<double>(4);
        double lambda = 0.0, prev = 0.0, rel = 0.0;
        for (uint64_t it = 0; it < power_iters; ++it) {
            launch_spmv(h->m, 0, shift, x, y, s);  // y = (A + shift I) x
            launch_dot2(n, x, y, pa, pb, pc, parts, s);
            launch_final_reduce(pa, pb, pc, parts, tot, tot + 1,
                                reinterpret_cast<unsigned long long*>(tot + 2), s);
            after_launch(3);
            double res[2];
            CK(cudaMemcpyAsync(res, tot, sizeof(res), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            prev = lambda;
            lambda = res[0] - shift;
            const double norm = std::sqrt(res[1]);
            if (norm == 0.0) break;
            CK(cudaMemcpyAsync(x, y, n * 8, cudaMemcpyDeviceToDevice, s));
            launch_scale(n, x, 1.0 / norm, s);
            after_launch(1);
            if (it > 0) rel = std::fabs(lambda - prev) / std::max(std::fabs(lambda), 1e-300);
        }
        CK(cudaStreamSynchronize(s));
        *lambda_max = lambda;
        if (rel_change) *rel_change = rel;
    });
}

int expmc_cuda_splitting_product(expmc_matrix* h, const double* v, uint64_t nv,
                                 const expmc_path_params* p, double tol, double* out) {
    return guarded([&] {
        if (!h) throw InvalidArg("matrix handle is null");
        std::lock_guard<std::mutex> lk(h->mu);
        validate_params(p);
        check_vector(h, v, nv);
        if (!(tol > 0.0)) throw InvalidArg("tol must be positive");
        DeviceGuard g(h->device);
        cudaStream_t s = h->stream;
        const uint64_t n = h->m.n;
        double* x = h->tmp3.get<double>(n);
        CK(cudaMemcpyAsync(x, v, n * 8, cudaMemcpyHostToDevice, s));
        const double dt = p->beta / (double)p->n_steps;
        const bool strang = p->splitting == EXPMC_STRANG;
        for (uint64_t k = 0; k < p->n_steps; ++k) {
            launch_scale_diag(n, h->m.d, strang ? dt / 2.0 : dt, x, s);
            after_launch(1);
            expmv_dev(h, 1, dt, tol, x, s);
            if (strang) {
                launch_scale_diag(n, h->m.d, dt / 2.0, x, s);
                after_launch(1);
            }
        }
        CK(cudaMemcpyAsync(out, x, n * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
