// C++ host-API check (include/expmc_b200.hpp): the reference-shaped calls on
// the single-edge graph and the reference's error text.
// Built by tests/test_host.py (compile-only on CPU) and run by
// tests/test_gpu_parity.py on a GPU.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "expmc_b200.hpp"

using namespace expmc::b200;

int main() {
    const std::vector<std::uint64_t> rp = {0, 1, 2};
    const std::vector<std::uint32_t> col = {1, 0};
    const std::vector<double> val = {1.0, 1.0};
    SplitMatrix m(2, rp, col, val);
    PathParams p;
    p.samples = 400'000;
    p.seed = 7;
    const std::vector<double> v = {1.0, 0.0};
    const Estimate e = entry_estimate(m, v, 0, p);
    const Estimate tc = tc_estimate(m, p);
    std::printf("entry %.6f +- %.6f (cosh 1 = %.6f)  tc %.9f (2e = %.9f)\n", e.value, e.std_error,
                std::cosh(1.0), tc.value, 2 * std::exp(1.0));
    if (std::fabs(e.value - std::cosh(1.0)) > 5 * e.std_error) return 1;
    if (std::fabs(tc.value - 2 * std::exp(1.0)) > 1e-9) return 2;
    try {
        entry_estimate(m, v, 2, p);
        return 3;
    } catch (const std::invalid_argument& ex) {
        if (std::string(ex.what()) != "entry index out of range") return 4;
    }
    // workers -> replicas: the same rows over 3 replicas on device 0
    // (virtual shards) are bitwise identical to the single-replica call
    {
        const std::vector<std::uint64_t> rp4 = {0, 1, 3, 5, 6};
        const std::vector<std::uint32_t> col4 = {1, 0, 2, 1, 3, 2};
        const std::vector<double> val4 = {1.0, 1.0, 2.0, 2.0, 0.5, 0.5};
        std::vector<SplitMatrix> reps = replicas(1, 4, rp4, col4, val4);
        reps.emplace_back(4, rp4, col4, val4);
        reps.emplace_back(4, rp4, col4, val4);
        const std::vector<double> v4 = {0.5, -1.0, 2.0, 0.25};
        const std::vector<NodeId> rows = {3, 0, 1, 2, 2, 1, 0};
        PathParams q;
        q.samples = 5000;
        q.seed = 11;
        const EntriesEstimate one = entries_estimate(reps[0], v4, rows, q);
        std::vector<const SplitMatrix*> sh = {&reps[0], &reps[1], &reps[2]};
        const EntriesEstimate many = entries_estimate(sh, v4, rows, q);
        for (std::size_t k = 0; k < rows.size(); ++k)
            if (one.values[k] != many.values[k] || one.std_errors[k] != many.std_errors[k] ||
                one.jumps[k] != many.jumps[k])
                return 5;
        if (one.total_jumps != many.total_jumps) return 6;
    }
    std::puts("api_demo ok");
    return 0;
}
