// Deterministic per-end-state accumulation for the Theorem-2 estimators
// (vector_estimate, proj/src/estimator.cpp:250 `local_values[out.end] += f`).
//
// The walkers of a batch emit (end, f) records indexed by walker; a stable
// radix sort by end keeps walker order inside each end state; run-length
// encoding (integer) + an exclusive scan of the run lengths give each end
// state's segment, and a segmented reduction sums every segment with one
// fixed-shape block reduction (no decoupled look-back: ReduceByKey's
// cross-tile prefix combination order depends on timing and is not bitwise
// reproducible for doubles).  Run sums are added to values[] in batch order.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_reduce.cuh>

#include "kernels.cuh"

namespace expmc_b200 {

namespace {

__global__ void add_runs_kernel(const uint32_t* __restrict__ keys, const double* __restrict__ sums,
                                int nruns, double* __restrict__ values) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nruns) values[keys[k]] = __dadd_rn(values[keys[k]], sums[k]);
}

int key_bits(uint64_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}

}  // namespace

size_t scatter_sort_temp_bytes(uint64_t batch, uint64_t n) {
    size_t a = 0, b = 0, c = 0, d = 0;
    const int nb = (int)batch;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const double*)nullptr, (double*)nullptr, nb, 0,
                                    key_bits(n));
    cub::DeviceRunLengthEncode::Encode(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                       (int*)nullptr, (int*)nullptr, nb);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (const int*)nullptr, (int*)nullptr, nb + 1);
    cub::DeviceSegmentedReduce::Sum(nullptr, d, (const double*)nullptr, (double*)nullptr, nb,
                                    (const int*)nullptr, (const int*)nullptr);
    size_t m = a;
    for (size_t x : {b, c, d}) m = x > m ? x : m;
    return m + 256;
}

// run_keys / run_sums: `count` entries; run_len / run_off: count + 1 ints
// (laid out in `lens`, 2 * (count + 1) ints).
void scatter_sort_accumulate(uint32_t* end, double* f, uint32_t* end_sorted, double* f_sorted,
                             uint64_t count, uint64_t n, uint32_t* run_keys, double* run_sums,
                             int* lens, void* temp, size_t temp_bytes, double* values,
                             cudaStream_t s) {
    if (count == 0) return;
    const int nb = (int)count;
    int* run_len = lens;
    int* run_off = lens + count + 1;
    int* nruns_d = run_off + count + 1;
    size_t tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp, tb, end, end_sorted, f, f_sorted, nb, 0, key_bits(n),
                                    s);
    tb = temp_bytes;
    cub::DeviceRunLengthEncode::Encode(temp, tb, end_sorted, run_keys, run_len, nruns_d, nb, s);
    int nruns = 0;
    cudaMemcpyAsync(&nruns, nruns_d, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaMemsetAsync(run_len + nruns, 0, sizeof(int), s);
    tb = temp_bytes;
    cub::DeviceScan::ExclusiveSum(temp, tb, run_len, run_off, nruns + 1, s);
    tb = temp_bytes;
    cub::DeviceSegmentedReduce::Sum(temp, tb, f_sorted, run_sums, nruns, run_off, run_off + 1, s);
    add_runs_kernel<<<(unsigned)((nruns + 255) / 256), 256, 0, s>>>(run_keys, run_sums, nruns,
                                                                   values);
}

}  // namespace expmc_b200
