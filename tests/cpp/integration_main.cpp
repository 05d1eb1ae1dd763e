// Runs the INTEGRATION.md binding (expmc::gpu, generated into
// tests/cpp/_bin/gpu_backend.hpp from the document) against the compiled
// reference (oracle/_ref/libexpmc_ref.so: the reference's own generate /
// split / entry_estimate / vector_estimate / tc_estimate).  Built here by
// tests/cpp/build_integration.sh (needs /root/reference headers); run on
// the GPU by tests/test_gpu_parity.py::test_integration_binding_runs.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "expmc/estimator.hpp"
#include "expmc/generators.hpp"
#include "expmc/sparse_matrix.hpp"
#include "gpu_backend.hpp"

using namespace expmc;

static int fail(const char* what, double a = 0, double b = 0) {
    std::printf("FAIL %s %.17g %.17g\n", what, a, b);
    return 1;
}

static SplitMatrix make(std::uint64_t seed) {
    GenSpec g;
    g.kind = GraphKind::ScaleFree;
    g.n = 20000;
    g.m0 = 5;
    g.seed = seed;
    return split(generate(g));
}

#define STEP(x) std::printf("step %s\n", x)

int main() {
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    PathParams p;
    p.beta = 0.05;
    p.n_steps = 32;
    p.samples = 20000;
    p.seed = 3;
    SplitMatrix m = make(1);
    std::vector<double> v(m.n);
    for (std::size_t i = 0; i < m.n; ++i) v[i] = std::sin(0.37 * (double)i) + 0.1;
    const NodeId rows[] = {0, 1, 7, 123, 4567, 19999};
    STEP("1. the drop-in");
    // 1. the drop-in call against the reference's own estimator
    for (NodeId i : rows) {
        const Estimate g = gpu::entry_estimate(m, v, i, p);
        PathParams q = p;
        q.seed = 100 + i;
        const Estimate r = entry_estimate(m, v, i, q, 8);
        const double z = (g.value - r.value) / std::sqrt(g.std_error * g.std_error +
                                                         r.std_error * r.std_error);
        if (!(std::fabs(z) < 5.0)) return fail("entry z", g.value, r.value);
    }
    STEP("2. same errors");
    // 2. same errors as the reference
    try {
        gpu::entry_estimate(m, v, (NodeId)m.n, p);
        return fail("no range error");
    } catch (const std::invalid_argument& e) {
        if (std::string(e.what()) != "entry index out of range") return fail("range message");
    }
    STEP("3. a different ma");
    // 3. a different matrix at the same address (a seed sweep) is not served
    //    from the stale device copy
    const Estimate before = gpu::entry_estimate(m, v, 7, p);
    m = make(2);
    const Estimate after = gpu::entry_estimate(m, v, 7, p);
    {
        PathParams q = p;
        q.seed = 999;
        const Estimate r = entry_estimate(m, v, 7, q, 8);
        const double z = (after.value - r.value) / std::sqrt(after.std_error * after.std_error +
                                                             r.std_error * r.std_error);
        if (!(std::fabs(z) < 5.0)) return fail("rebuilt-matrix z", after.value, r.value);
        if (before.value == after.value) return fail("stale device copy", before.value);
    }
    STEP("4. concurrent cal");
    // 4. concurrent callers share one SplitMatrix: each gets its
    //    serial result
    std::vector<Estimate> serial;
    for (NodeId i : rows) serial.push_back(gpu::entry_estimate(m, v, i, p));
    std::vector<Estimate> par(std::size(rows));
    std::vector<std::thread> ts;
    for (std::size_t k = 0; k < std::size(rows); ++k)
        ts.emplace_back([&, k] { par[k] = gpu::entry_estimate(m, v, rows[k], p); });
    for (auto& t : ts) t.join();
    for (std::size_t k = 0; k < std::size(rows); ++k)
        if (par[k].value != serial[k].value || par[k].total_jumps != serial[k].total_jumps)
            return fail("concurrent", par[k].value, serial[k].value);
    STEP("5. the batched");
    // 5. the batched multi-device call equals the single-row calls
    const std::vector<Estimate> many = gpu::entries_estimate(m, v, rows, p, 1);
    for (std::size_t k = 0; k < std::size(rows); ++k)
        if (many[k].value != serial[k].value) return fail("batched", many[k].value);
    STEP("6. Theorem-2");
    // 6. Theorem-2 estimators against the reference
    std::vector<double> w(m.n);
    for (std::size_t i = 0; i < m.n; ++i) w[i] = 1.0 + 0.5 * std::cos(0.11 * (double)i);
    PathParams pv = p;
    pv.samples = 2'000'000;
    const VectorEstimate gv = gpu::vector_estimate(m, w, pv);
    const VectorEstimate rv = vector_estimate(m, w, pv, 8);
    double gs = 0, rs = 0;
    for (std::size_t i = 0; i < m.n; ++i) gs += gv.values[i], rs += rv.values[i];
    const double zv = (gs - rs) / std::sqrt(gv.std_error_global * gv.std_error_global +
                                            rv.std_error_global * rv.std_error_global);
    if (!(std::fabs(zv) < 5.0)) return fail("vector z", gs, rs);
    const Estimate gt = gpu::tc_estimate(m, pv);
    const Estimate rt = tc_estimate(m, pv, 8);
    const double zt = (gt.value - rt.value) / std::sqrt(gt.std_error * gt.std_error +
                                                        rt.std_error * rt.std_error);
    if (!(std::fabs(zt) < 5.0)) return fail("tc z", gt.value, rt.value);
    std::puts("integration ok");
    return 0;
}
