// Deterministic per-end-state accumulation for the Theorem-2 estimators
// (vector_estimate, proj/src/estimator.cpp:250 `local_values[out.end] += f`).
//
// The walkers of a batch emit (end, f) records indexed by walker; a stable
// radix sort by end keeps walker order inside each end state, a
// reduce-by-key sums each run (no atomics), and the run sums are added to
// values[] in batch order.  Bitwise reproducible for a fixed (samples,
// batch size) — unlike fp64 atomics — and independent of the launch grid.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>

#include "kernels.cuh"

namespace expmc_b200 {

namespace {

__global__ void add_runs_kernel(const uint32_t* __restrict__ keys, const double* __restrict__ sums,
                                const int* __restrict__ nruns, double* __restrict__ values) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < *nruns) values[keys[k]] = __dadd_rn(values[keys[k]], sums[k]);
}

int key_bits(uint64_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}

}  // namespace

size_t scatter_sort_temp_bytes(uint64_t batch, uint64_t n) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const double*)nullptr, (double*)nullptr, (int)batch, 0,
                                    key_bits(n));
    cub::DeviceReduce::ReduceByKey(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                   (const double*)nullptr, (double*)nullptr, (int*)nullptr,
                                   cuda::std::plus<double>(), (int)batch);
    return (a > b ? a : b) + 256;
}

void scatter_sort_accumulate(uint32_t* end, double* f, uint32_t* end_sorted, double* f_sorted,
                             uint64_t count, uint64_t n, uint32_t* run_keys, double* run_sums,
                             int* nruns, void* temp, size_t temp_bytes, double* values,
                             cudaStream_t s) {
    if (count == 0) return;
    size_t tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp, tb, end, end_sorted, f, f_sorted, (int)count, 0,
                                    key_bits(n), s);
    tb = temp_bytes;
    cub::DeviceReduce::ReduceByKey(temp, tb, end_sorted, run_keys, f_sorted, run_sums, nruns,
                                   cuda::std::plus<double>(), (int)count, s);
    add_runs_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(run_keys, run_sums, nruns,
                                                                   values);
}

}  // namespace expmc_b200
