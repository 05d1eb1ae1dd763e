// Deterministic per-end-state accumulation for the Theorem-2 estimators
// (vector_estimate, proj/src/estimator.cpp:250 `local_values[out.end] += f`)
// and per-row sums of the large-W entry path.
//
// The walkers of a batch emit (end, f) records in a fixed order (walker /
// jumper index); a stable radix sort by end keeps that order inside each end
// state.  Every run of equal keys is then summed by a fixed 32-ary tree:
// level 0 sums each 32-record chunk's run pieces sequentially; a run that
// lies inside one chunk is added to values[key] there, and each chunk hands
// its first and last run pieces (0.0 when that run is already complete) to
// the next level as two (key, piece) records — still sorted, pieces in chunk
// order — and the level recurses until a level fits one chunk.  Each run is
// completed, and added to values[key], by exactly one thread at one level,
// so there are no atomics and the result is bitwise reproducible; batches
// are applied in order.  Depth log_16(count): runs of any length (a hub end
// state, one row of 2^30 walkers) cost the same as short ones.  (CUB's
// ReduceByKey combines tile prefixes in a timing-dependent order, which is
// not bitwise reproducible for doubles.)
#include <stdexcept>

#include <cub/device/device_radix_sort.cuh>

#include "kernels.cuh"

namespace expmc_b200 {

namespace {

constexpr uint32_t kChunk = 32;  // records per thread in the run-sum passes

constexpr int kPieceThreads = 128;
constexpr int kPad = kChunk + 1;  // smem row stride (bank-conflict-free chunk walks)
constexpr size_t kPieceSmem = (size_t)kPieceThreads * kPad * (sizeof(uint32_t) + sizeof(double));

// One level: thread k owns chunk [kC, kC + C) of the sorted records and sums
// every run piece in it sequentially.  A run that starts and ends in the
// chunk is added to values[] here.  The chunk's first run piece (when its run
// started in an earlier chunk) and its last run piece (when its run goes on
// past the chunk) become the next level's records 2k and 2k + 1, keyed by the
// chunk's first and last keys (0.0 where there is no such piece).  The
// block's records are staged through shared memory with coalesced loads.
__global__ void __launch_bounds__(kPieceThreads)
run_level_kernel(const uint32_t* __restrict__ keys, const double* __restrict__ f,
                 uint64_t count, double* __restrict__ values, uint32_t* __restrict__ nkeys,
                 double* __restrict__ nvals) {
    extern __shared__ double smem[];
    double* sf = smem;
    uint32_t* sk = reinterpret_cast<uint32_t*>(smem + kPieceThreads * kPad);
    const uint64_t base = (uint64_t)blockIdx.x * kPieceThreads * kChunk;
    for (uint32_t i = threadIdx.x; i < kPieceThreads * kChunk; i += kPieceThreads) {
        if (base + i < count) {
            const uint32_t slot = (i / kChunk) * kPad + i % kChunk;
            sk[slot] = keys[base + i];
            sf[slot] = f[base + i];
        }
    }
    __syncthreads();
    const uint64_t k = (uint64_t)blockIdx.x * kPieceThreads + threadIdx.x;
    const uint64_t lo = k * kChunk;
    if (lo >= count) return;
    const uint32_t len = (uint32_t)(count - lo < kChunk ? count - lo : kChunk);
    const uint32_t* ck = sk + threadIdx.x * kPad;
    const double* cf = sf + threadIdx.x * kPad;
    const bool last_chunk = lo + len == count;
    double head = 0.0, tail = 0.0;
    uint32_t pos = 0;
    while (pos < len) {
        const uint32_t key = ck[pos];
        const bool started = pos > 0 || lo == 0 || keys[lo - 1] != key;
        double s = cf[pos];
        uint32_t j = pos + 1;
        while (j < len && ck[j] == key) s = __dadd_rn(s, cf[j++]);
        const bool ends = j < len || last_chunk || keys[lo + len] != key;
        if (!started) head = s;       // (the run may also go on past the chunk)
        else if (ends) values[key] = __dadd_rn(values[key], s);
        else tail = s;
        pos = j;
    }
    if (nkeys) {
        nkeys[2 * k] = ck[0];
        nvals[2 * k] = head;
        nkeys[2 * k + 1] = ck[len - 1];
        nvals[2 * k + 1] = tail;
    }
}

int key_bits(uint64_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}

}  // namespace

size_t scatter_sort_temp_bytes(uint64_t batch, uint64_t n) {
    size_t a = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const double*)nullptr, (double*)nullptr, (int)batch, 0,
                                    key_bits(n));
    return a + 256 + run_sums_temp_bytes(batch);
}

void scatter_sort_accumulate(uint32_t* end, double* f, uint32_t* end_sorted, double* f_sorted,
                             uint64_t count, uint64_t n, void* temp, size_t temp_bytes,
                             double* values, cudaStream_t s) {
    if (count == 0) return;
    size_t tb = 0;  // the sort's own share of temp (the piece buffers follow it)
    cub::DeviceRadixSort::SortPairs(nullptr, tb, end, end_sorted, f, f_sorted, (int)count, 0,
                                    key_bits(n));
    if (((tb + 255) & ~(size_t)255) + run_sums_temp_bytes(count) > temp_bytes)
        throw std::runtime_error("scatter_sort: temp storage too small");
    cub::DeviceRadixSort::SortPairs(temp, tb, end, end_sorted, f, f_sorted, (int)count, 0,
                                    key_bits(n), s);
    const size_t sort_bytes = (tb + 255) & ~(size_t)255;
    run_sums_sorted(end_sorted, f_sorted, count, static_cast<unsigned char*>(temp) + sort_bytes,
                    temp_bytes - sort_bytes, values, s);
}

size_t run_sums_temp_bytes(uint64_t count) {
    // two ping-pong levels of (u32 key, f64 piece) records, 2 per chunk
    const uint64_t c1 = 2 * ((count + kChunk - 1) / kChunk);
    return 2 * (c1 * (sizeof(uint32_t) + sizeof(double)) + 512) + 256;
}

// out[key] += sum of each run of equal keys (keys sorted), in record order
// grouped by the fixed 32-ary tree above.
void run_sums_sorted(const uint32_t* keys, const double* vals, uint64_t count, void* temp,
                     size_t temp_bytes, double* out, cudaStream_t s) {
    if (count == 0) return;
    if (run_sums_temp_bytes(count) > temp_bytes)
        throw std::runtime_error("run_sums: temp storage too small");
    const uint64_t c1 = 2 * ((count + kChunk - 1) / kChunk);
    const size_t region = ((c1 * (sizeof(uint32_t) + sizeof(double)) + 511) / 256) * 256;
    unsigned char* t = static_cast<unsigned char*>(temp);
    t = reinterpret_cast<unsigned char*>(((uintptr_t)t + 255) & ~(uintptr_t)255);
    double* vbuf[2] = {reinterpret_cast<double*>(t), reinterpret_cast<double*>(t + region)};
    uint32_t* kbuf[2] = {reinterpret_cast<uint32_t*>(vbuf[0] + c1),
                         reinterpret_cast<uint32_t*>(vbuf[1] + c1)};
    cudaFuncSetAttribute(run_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kPieceSmem);  // per device; cheap
    const uint32_t* k = keys;
    const double* v = vals;
    uint64_t n = count;
    for (int lvl = 0;; ++lvl) {
        const uint64_t chunks = (n + kChunk - 1) / kChunk;
        const unsigned grid = (unsigned)((chunks + kPieceThreads - 1) / kPieceThreads);
        if (chunks == 1) {
            run_level_kernel<<<grid, kPieceThreads, kPieceSmem, s>>>(k, v, n, out, nullptr,
                                                                    nullptr);
            break;
        }
        uint32_t* nk = kbuf[lvl & 1];
        double* nv = vbuf[lvl & 1];
        run_level_kernel<<<grid, kPieceThreads, kPieceSmem, s>>>(k, v, n, out, nk, nv);
        k = nk;
        v = nv;
        n = 2 * chunks;
    }
}

}  // namespace expmc_b200
