// Deterministic per-end-state accumulation for the Theorem-2 estimators
// (vector_estimate, proj/src/estimator.cpp:250 `local_values[out.end] += f`).
//
// The walkers of a batch emit (end, f) records in a fixed order (walker /
// jumper index); a stable radix sort by end keeps that order inside each end
// state.  Every run is then summed in that order in fixed 32-record pieces
// (pass A: pieces, runs inside one piece added at once; pass B: runs that
// cross piece boundaries, pieces added in order) and added to values[end].
// Each run is added by exactly one thread, so there are no atomics; batches
// are applied in order, so the result is bitwise reproducible.  (CUB's
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

// Pass A: thread k owns chunk [kC, kC + C) of the sorted records and sums
// every run piece in it sequentially.  A run that starts and ends in the
// chunk is added to values[] here; the piece of a run that started earlier
// goes to head[k]; the piece of a run that starts here and continues past
// the chunk goes to tail[k] (completed in pass B).  The block's records are
// staged through shared memory with coalesced loads first.
__global__ void __launch_bounds__(kPieceThreads)
run_pieces_kernel(const uint32_t* __restrict__ keys, const double* __restrict__ f,
                  uint64_t count, double* __restrict__ head, double* __restrict__ tail,
                  double* __restrict__ values) {
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
    uint32_t pos = 0;
    while (pos < len) {
        const uint32_t key = ck[pos];
        const bool started = pos > 0 || lo == 0 || keys[lo - 1] != key;
        double s = cf[pos];
        uint32_t j = pos + 1;
        while (j < len && ck[j] == key) s = __dadd_rn(s, cf[j++]);
        const bool ends = j < len || last_chunk || keys[lo + len] != key;
        if (!started) head[k] = s;
        else if (ends) values[key] = __dadd_rn(values[key], s);
        else tail[k] = s;
        pos = j;
    }
}

// Pass B: thread k completes the run that starts in its chunk and crosses
// its end: tail[k] + head[k+1] + head[k+2] + ... in chunk order.
__global__ void run_spans_kernel(const uint32_t* __restrict__ keys, uint64_t count,
                                 const double* __restrict__ head,
                                 const double* __restrict__ tail, double* __restrict__ values) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t lo = k * kChunk, hi = lo + kChunk;
    if (hi >= count) return;  // the last chunk has nothing past its end
    const uint32_t key = keys[hi - 1];
    if (keys[hi] != key) return;  // no run crosses the end of this chunk
    // the crossing run started here unless it also covers this chunk's start
    if (keys[lo] == key && (lo > 0 && keys[lo - 1] == key)) return;
    double s = tail[k];
    for (uint64_t c = k + 1; c * kChunk < count && keys[c * kChunk] == key; ++c) {
        s = __dadd_rn(s, head[c]);
        const uint64_t e = (c + 1) * kChunk;
        if (e >= count || keys[e] != key) break;
    }
    values[key] = __dadd_rn(values[key], s);
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
    const uint64_t chunks = (batch + kChunk - 1) / kChunk;
    return a + 256 + 2 * chunks * sizeof(double) + 256;
}

void scatter_sort_accumulate(uint32_t* end, double* f, uint32_t* end_sorted, double* f_sorted,
                             uint64_t count, uint64_t n, void* temp, size_t temp_bytes,
                             double* values, cudaStream_t s) {
    if (count == 0) return;
    size_t tb = 0;  // the sort's own share of temp (the piece buffers follow it)
    cub::DeviceRadixSort::SortPairs(nullptr, tb, end, end_sorted, f, f_sorted, (int)count, 0,
                                    key_bits(n));
    if (tb + 512 + 2 * ((count + kChunk - 1) / kChunk) * sizeof(double) > temp_bytes)
        throw std::runtime_error("scatter_sort: temp storage too small");
    cub::DeviceRadixSort::SortPairs(temp, tb, end, end_sorted, f, f_sorted, (int)count, 0,
                                    key_bits(n), s);
    const size_t sort_bytes = (tb + 255) & ~(size_t)255;
    run_sums_sorted(end_sorted, f_sorted, count, static_cast<unsigned char*>(temp) + sort_bytes,
                    temp_bytes - sort_bytes, values, s);
}

size_t run_sums_temp_bytes(uint64_t count) {
    return 2 * ((count + kChunk - 1) / kChunk) * sizeof(double) + 256;
}

// out[key] += sum of each run of equal keys (keys sorted), in record order.
void run_sums_sorted(const uint32_t* keys, const double* vals, uint64_t count, void* temp,
                     size_t temp_bytes, double* out, cudaStream_t s) {
    if (count == 0) return;
    const uint64_t chunks = (count + kChunk - 1) / kChunk;
    if (2 * chunks * sizeof(double) > temp_bytes)
        throw std::runtime_error("run_sums: temp storage too small");
    double* head = static_cast<double*>(temp);
    double* tail = head + chunks;
    cudaFuncSetAttribute(run_pieces_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kPieceSmem);  // per device; cheap
    run_pieces_kernel<<<(unsigned)((chunks + kPieceThreads - 1) / kPieceThreads), kPieceThreads,
                        kPieceSmem, s>>>(keys, vals, count, head, tail, out);
    run_spans_kernel<<<(unsigned)((chunks + 255) / 256), 256, 0, s>>>(keys, count, head, tail,
                                                                      out);
}

}  // namespace expmc_b200
