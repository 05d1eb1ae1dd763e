// Host-side synthetic inputs for the benchmark configurations (BASELINE.json
// configs 1-5): FD Laplacians, Barabasi-Albert, Watts-Strogatz, seeded
// vectors and row samples.  Input plumbing only — the estimators never run
// here.
//
// BA restates generate({ScaleFree, n, m0, seed}) (proj/src/generators.cpp:
// 58-103) draw for draw, so the graph is identical to the reference's; the
// CSR is built straight into the mirrored, row-sorted layout that
// SparseSymmetric::from_entries produces (proj/src/sparse_matrix.cpp:58-83)
// with a counting sort instead of a comparison sort of the entry list.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "host_io.h"

namespace expmc_b200 {
namespace {
struct HostErr {
    char s[2048];
};
thread_local HostErr g_host_err;
}  // namespace
void set_host_error(const char* m) { std::snprintf(g_host_err.s, sizeof g_host_err.s, "%s", m); }
const char* host_error_str() { return g_host_err.s; }
}  // namespace expmc_b200

namespace {

// PCG32 RngStream, proj/include/expmc/rng.hpp:14-63
struct Pcg {
    uint64_t state = 0, inc;
    Pcg(uint64_t seed, uint64_t stream) : inc((stream << 1u) | 1u) {
        next_u32();
        state += seed;
        next_u32();
    }
    uint32_t next_u32() {
        const uint64_t old = state;
        state = old * 6364136223846793005ULL + inc;
        const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
        const uint32_t rot = (uint32_t)(old >> 59u);
        return (xs >> rot) | (xs << ((32u - rot) & 31u));
    }
    uint64_t next_u64() {
        const uint64_t hi = next_u32();
        return (hi << 32) | next_u32();
    }
    double uniform() { return (double)(next_u64() >> 11) * 0x1.0p-53; }
    uint64_t uniform_index(uint64_t n) {
        const uint64_t k = (uint64_t)(uniform() * (double)n);
        return k < n ? k : n - 1;
    }
};

template <class F>
int guarded(F&& f) {
    return expmc_b200::host_guarded(f);
}

// Mirrored CSR from an undirected edge list (a != b, no duplicates),
// every row sorted by column.
expmc_csr* csr_from_edges(uint64_t n, const std::vector<uint32_t>& ea,
                          const std::vector<uint32_t>& eb, double w) {
    auto* c = new expmc_csr;
    c->n = n;
    c->row_ptr.assign(n + 1, 0);
    for (size_t k = 0; k < ea.size(); ++k) {
        ++c->row_ptr[ea[k] + 1];
        ++c->row_ptr[eb[k] + 1];
    }
    for (uint64_t i = 0; i < n; ++i) c->row_ptr[i + 1] += c->row_ptr[i];
    c->col.resize(c->row_ptr[n]);
    std::vector<uint64_t> fill(c->row_ptr.begin(), c->row_ptr.end() - 1);
    for (size_t k = 0; k < ea.size(); ++k) {
        c->col[fill[ea[k]]++] = eb[k];
        c->col[fill[eb[k]]++] = ea[k];
    }
    for (uint64_t i = 0; i < n; ++i)
        std::sort(c->col.begin() + c->row_ptr[i], c->col.begin() + c->row_ptr[i + 1]);
    c->val.assign(c->col.size(), w);
    c->diag.assign(n, 0.0);
    return c;
}

}  // namespace

extern "C" {

const char* expmc_gen_last_error(void) { return expmc_b200::host_error_str(); }

int expmc_gen_fd(int dim, uint64_t side, double s, expmc_csr** out) {
    return guarded([&] {
        if (dim != 2 && dim != 3) throw std::invalid_argument("fd: dim must be 2 or 3");
        if (side < 1) throw std::invalid_argument("fd: side must be >= 1");
        const uint64_t L = side, L2 = side * side;
        const uint64_t n = dim == 2 ? L2 : L2 * L;
        auto* c = new expmc_csr;
        c->n = n;
        c->row_ptr.assign(n + 1, 0);
        c->col.reserve(n * 2 * dim);
        c->diag.assign(n, -2.0 * dim * s);
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t x = i % L, y = (i / L) % L, z = dim == 3 ? i / L2 : 0;
            // neighbours in increasing index order
            if (dim == 3 && z > 0) c->col.push_back((uint32_t)(i - L2));
            if (y > 0) c->col.push_back((uint32_t)(i - L));
            if (x > 0) c->col.push_back((uint32_t)(i - 1));
            if (x + 1 < L) c->col.push_back((uint32_t)(i + 1));
            if (y + 1 < L) c->col.push_back((uint32_t)(i + L));
            if (dim == 3 && z + 1 < L) c->col.push_back((uint32_t)(i + L2));
            c->row_ptr[i + 1] = c->col.size();
        }
        c->val.assign(c->col.size(), s);
        *out = c;
    });
}

int expmc_gen_ba(uint64_t n, uint64_t m0, uint64_t seed, expmc_csr** out) {
    // generators.cpp:58-103, draw for draw
    return guarded([&] {
        if (m0 < 1 || n < m0 + 1)
            throw std::invalid_argument("scale-free: need m0 >= 1 and n >= m0 + 1");
        if (n >= (1ull << 32)) throw std::invalid_argument("scale-free: n must be < 2^32");
        Pcg rng(seed, 0);
        const uint64_t seed_nodes = m0 + 1;
        std::vector<uint32_t> ea, eb, endpoints;
        ea.reserve(m0 * n);
        eb.reserve(m0 * n);
        endpoints.reserve(2 * m0 * n);
        for (uint32_t i = 0; i < seed_nodes; ++i)
            for (uint32_t j = i + 1; j < seed_nodes; ++j) {
                ea.push_back(i);
                eb.push_back(j);
                endpoints.push_back(i);
                endpoints.push_back(j);
            }
        // Look-ahead prefetch: the draw sequence does not depend on the
        // graph, so endpoints[] slots about to be read can be prefetched.
        constexpr int kAhead = 16;
        Pcg ahead = rng;
        for (int k = 0; k < kAhead; ++k) ahead.next_u64();
        std::vector<uint32_t> picked;
        picked.reserve(m0);
        for (uint64_t v = seed_nodes; v < n; ++v) {
            picked.clear();
            while (picked.size() < m0) {
                const uint64_t sz = endpoints.size();
                {
                    const uint64_t k = (uint64_t)((double)(ahead.next_u64() >> 11) * 0x1.0p-53 *
                                                  (double)sz);
                    __builtin_prefetch(endpoints.data() + (k < sz ? k : sz - 1));
                }
                const uint32_t t = endpoints[rng.uniform_index(sz)];
                if (std::find(picked.begin(), picked.end(), t) == picked.end())
                    picked.push_back(t);
            }
            for (const uint32_t t : picked) {
                ea.push_back(t);
                eb.push_back((uint32_t)v);
                endpoints.push_back(t);
                endpoints.push_back((uint32_t)v);
            }
        }
        std::vector<uint32_t>().swap(endpoints);
        *out = csr_from_edges(n, ea, eb, 1.0);
    });
}

int expmc_gen_ws(uint64_t n, uint64_t half_k, double p, uint64_t seed, expmc_csr** out) {
    // Watts-Strogatz: for r = 1..half_k, for u = 0..n-1, the lattice edge
    // (u, u+r mod n) is rewired with probability p to (u, w), w uniform over
    // nodes with w != u and (u, w) not already an edge.
    return guarded([&] {
        if (half_k < 1 || n < 2 * half_k + 2)
            throw std::invalid_argument("watts-strogatz: need k/2 >= 1 and n >= k + 2");
        if (!(p >= 0.0 && p <= 1.0))
            throw std::invalid_argument("watts-strogatz: p must be in [0, 1]");
        if (n >= (1ull << 32)) throw std::invalid_argument("watts-strogatz: n must be < 2^32");
        auto key = [](uint64_t a, uint64_t b) { return a < b ? (a << 32) | b : (b << 32) | a; };
        const uint64_t m = n * half_k;
        std::vector<uint32_t> ea(m), eb(m);
        std::unordered_set<uint64_t> edges;
        edges.reserve(m * 2);
        for (uint64_t r = 1; r <= half_k; ++r)
            for (uint64_t u = 0; u < n; ++u) {
                const uint64_t v = (u + r) % n;
                ea[(r - 1) * n + u] = (uint32_t)u;
                eb[(r - 1) * n + u] = (uint32_t)v;
                edges.insert(key(u, v));
            }
        Pcg rng(seed, 0);
        for (uint64_t r = 1; r <= half_k; ++r)
            for (uint64_t u = 0; u < n; ++u) {
                if (rng.uniform() >= p) continue;
                const uint64_t e = (r - 1) * n + u;
                uint64_t w;
                do {
                    w = rng.uniform_index(n);
                } while (w == u || edges.count(key(u, w)));
                edges.erase(key(u, eb[e]));
                edges.insert(key(u, w));
                eb[e] = (uint32_t)w;
            }
        *out = csr_from_edges(n, ea, eb, 1.0);
    });
}

int expmc_csr_sizes(const expmc_csr* c, uint64_t* n, uint64_t* nnz) {
    if (!c) return EXPMC_INVALID_ARGUMENT;
    if (n) *n = c->n;
    if (nnz) *nnz = c->col.size();
    return EXPMC_OK;
}

int expmc_csr_export(const expmc_csr* c, uint64_t* row_ptr, uint32_t* col, double* val,
                     double* diag) {
    if (!c) return EXPMC_INVALID_ARGUMENT;
    if (row_ptr) std::memcpy(row_ptr, c->row_ptr.data(), (c->n + 1) * 8);
    if (col) std::memcpy(col, c->col.data(), c->col.size() * 4);
    if (val) std::memcpy(val, c->val.data(), c->val.size() * 8);
    if (diag) std::memcpy(diag, c->diag.data(), c->n * 8);
    return EXPMC_OK;
}

int expmc_csr_view(const expmc_csr* c, const uint64_t** row_ptr, const uint32_t** col,
                   const double** val, const double** diag) {
    if (!c) return EXPMC_INVALID_ARGUMENT;
    if (row_ptr) *row_ptr = c->row_ptr.data();
    if (col) *col = c->col.data();
    if (val) *val = c->val.data();
    if (diag) *diag = c->diag.data();
    return EXPMC_OK;
}

void expmc_csr_free(expmc_csr* c) { delete c; }

int expmc_gen_vector(int kind, uint64_t n, uint64_t side, double sigma, uint64_t seed,
                     double* out) {
    return guarded([&] {
        Pcg rng(seed, 0);
        if (kind == 0) {
            for (uint64_t i = 0; i < n; ++i) out[i] = rng.uniform();
        } else if (kind == 1) {
            for (uint64_t i = 0; i < n; ++i) out[i] = 2.0 * rng.uniform() - 1.0;
        } else if (kind == 2) {
            if (side * side * side != n) throw std::invalid_argument("bump: n must be side^3");
            if (!(sigma > 0.0)) throw std::invalid_argument("bump: sigma must be positive");
            const double h = 1.0 / (double)(side + 1);
            for (uint64_t i = 0; i < n; ++i) {
                const double x = (double)(i % side + 1) * h - 0.5;
                const double y = (double)((i / side) % side + 1) * h - 0.5;
                const double z = (double)(i / (side * side) + 1) * h - 0.5;
                out[i] = std::exp(-(x * x + y * y + z * z) / (2.0 * sigma * sigma)) +
                         rng.uniform();
            }
        } else {
            throw std::invalid_argument("unknown vector kind");
        }
    });
}

int expmc_gen_row_sample(uint64_t n, uint64_t k, uint64_t seed, uint32_t* out) {
    return guarded([&] {
        if (k > n) throw std::invalid_argument("row sample larger than n");
        if (n >= (1ull << 32)) throw std::invalid_argument("n must be < 2^32");
        std::vector<uint32_t> a(n);
        for (uint64_t i = 0; i < n; ++i) a[i] = (uint32_t)i;
        Pcg rng(seed, 0);
        for (uint64_t j = 0; j < k; ++j) {
            const uint64_t r = j + rng.uniform_index(n - j);
            std::swap(a[j], a[r]);
        }
        std::sort(a.begin(), a.begin() + k);
        std::memcpy(out, a.data(), k * 4);
    });
}

}  // extern "C"
