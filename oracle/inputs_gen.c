/*
 * TEST INFRASTRUCTURE ONLY — input builders for bench.py's reference arm
 * (--impl reference / cpu_baseline), so that the reference process never
 * loads the product library.  Never linked into the product.
 *
 * Plain-C restatements of the synthetic inputs of BASELINE.json configs 1-5
 * (SURVEY §8d).  The Barabási–Albert graphs (configs 2 and 5) come from the
 * reference's own generate({ScaleFree, ...}) (proj/src/generators.cpp:58-103,
 * through oracle/ref_shim.cpp ref_generate) and are not restated here.  The
 * rest follows the same definitions as the product's input plumbing:
 *
 *   FD2D / FD3D Dirichlet Laplacian   (5- / 7-point stencil, scaled by s)
 *   Watts–Strogatz rewiring           (lattice (u, u+r), rewired w.p. p)
 *   seeded vectors                    (RngStream(seed, 0), rng.hpp:14-63)
 *   row sample                        (partial Fisher–Yates, then sorted)
 *
 * tests/test_oracle_inputs.py pins every builder byte-for-byte against the
 * product's builders on small and full sizes.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- PCG32 */
/* proj/include/expmc/rng.hpp:14-63 */
typedef struct {
    uint64_t state, inc;
} gen_rng;

static uint32_t g_next_u32(gen_rng* r) {
    uint64_t old = r->state;
    r->state = old * 6364136223846793005ULL + r->inc;
    uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
}
static void g_init(gen_rng* r, uint64_t seed, uint64_t stream) {
    r->state = 0u;
    r->inc = (stream << 1u) | 1u;
    g_next_u32(r);
    r->state += seed;
    g_next_u32(r);
}
static double g_uniform(gen_rng* r) {
    uint64_t hi = g_next_u32(r);
    uint64_t x = (hi << 32) | g_next_u32(r);
    return (double)(x >> 11) * 0x1.0p-53;
}
static uint64_t g_index(gen_rng* r, uint64_t n) {
    uint64_t k = (uint64_t)(g_uniform(r) * (double)n);
    return k < n ? k : n - 1;
}

/* ------------------------------------------------------------- FD grids */
/* Number of directed entries of the dim-D side^D Dirichlet grid. */
uint64_t orc_gen_fd_nnz(int dim, uint64_t side) {
    uint64_t faces = (side - 1) * side * (dim == 3 ? side : 1); /* per axis */
    return 2ull * (uint64_t)dim * faces;
}

/* Mirrored CSR, rows sorted by column; diag = -2 dim s, off-diagonal s. */
int orc_gen_fd(int dim, uint64_t side, double s, uint64_t* row_ptr, uint32_t* col,
               double* val, double* diag) {
    if ((dim != 2 && dim != 3) || side < 1) return 1;
    const uint64_t L = side, L2 = side * side, n = dim == 2 ? L2 : L2 * L;
    uint64_t k = 0;
    row_ptr[0] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t x = i % L, y = (i / L) % L, z = dim == 3 ? i / L2 : 0;
        if (dim == 3 && z > 0) col[k++] = (uint32_t)(i - L2);
        if (y > 0) col[k++] = (uint32_t)(i - L);
        if (x > 0) col[k++] = (uint32_t)(i - 1);
        if (x + 1 < L) col[k++] = (uint32_t)(i + 1);
        if (y + 1 < L) col[k++] = (uint32_t)(i + L);
        if (dim == 3 && z + 1 < L) col[k++] = (uint32_t)(i + L2);
        row_ptr[i + 1] = k;
        diag[i] = -2.0 * dim * s;
    }
    for (uint64_t e = 0; e < k; ++e) val[e] = s;
    return 0;
}

/* ----------------------------------------------------- Watts–Strogatz */
/* Open-addressing set of undirected edge keys (min << 32 | max), with
 * tombstones for erase. */
typedef struct {
    uint64_t* slot;
    uint64_t mask;
} eset;
#define ES_EMPTY 0xffffffffffffffffull
#define ES_DEAD 0xfffffffffffffffeull

static uint64_t es_hash(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}
static int es_has(const eset* s, uint64_t k) {
    for (uint64_t h = es_hash(k) & s->mask;; h = (h + 1) & s->mask) {
        if (s->slot[h] == k) return 1;
        if (s->slot[h] == ES_EMPTY) return 0;
    }
}
static void es_add(eset* s, uint64_t k) {
    uint64_t tomb = ES_EMPTY;
    for (uint64_t h = es_hash(k) & s->mask;; h = (h + 1) & s->mask) {
        if (s->slot[h] == k) return;
        if (s->slot[h] == ES_DEAD && tomb == ES_EMPTY) tomb = h;
        if (s->slot[h] == ES_EMPTY) {
            s->slot[tomb != ES_EMPTY ? tomb : h] = k;
            return;
        }
    }
}
static void es_del(eset* s, uint64_t k) {
    for (uint64_t h = es_hash(k) & s->mask;; h = (h + 1) & s->mask) {
        if (s->slot[h] == k) {
            s->slot[h] = ES_DEAD;
            return;
        }
        if (s->slot[h] == ES_EMPTY) return;
    }
}
static uint64_t ekey(uint64_t a, uint64_t b) { return a < b ? (a << 32) | b : (b << 32) | a; }

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}

/* For r = 1..half_k, u = 0..n-1: the lattice edge (u, u+r mod n) is rewired
 * with probability p to (u, w), w = uniform_index(n) redrawn while w == u or
 * (u, w) is already an edge.  Output: mirrored CSR (2 n half_k entries),
 * rows sorted by column, weight 1, diag 0. */
int orc_gen_ws(uint64_t n, uint64_t half_k, double p, uint64_t seed, uint64_t* row_ptr,
               uint32_t* col, double* val, double* diag) {
    if (half_k < 1 || n < 2 * half_k + 2 || !(p >= 0.0 && p <= 1.0) || n >= (1ull << 32))
        return 1;
    const uint64_t m = n * half_k;
    uint32_t* ea = malloc(m * 4);
    uint32_t* eb = malloc(m * 4);
    uint64_t cap = 1;
    while (cap < 4 * m) cap <<= 1;
    eset s = {malloc(cap * 8), cap - 1};
    uint64_t* fill = malloc((n + 1) * 8);
    if (!ea || !eb || !s.slot || !fill) {
        free(ea), free(eb), free(s.slot), free(fill);
        return 2;
    }
    memset(s.slot, 0xff, cap * 8);
    for (uint64_t r = 1; r <= half_k; ++r)
        for (uint64_t u = 0; u < n; ++u) {
            const uint64_t v = (u + r) % n;
            ea[(r - 1) * n + u] = (uint32_t)u;
            eb[(r - 1) * n + u] = (uint32_t)v;
            es_add(&s, ekey(u, v));
        }
    gen_rng rng;
    g_init(&rng, seed, 0);
    for (uint64_t r = 1; r <= half_k; ++r)
        for (uint64_t u = 0; u < n; ++u) {
            if (g_uniform(&rng) >= p) continue;
            const uint64_t e = (r - 1) * n + u;
            uint64_t w;
            do {
                w = g_index(&rng, n);
            } while (w == u || es_has(&s, ekey(u, w)));
            es_del(&s, ekey(u, eb[e]));
            es_add(&s, ekey(u, w));
            eb[e] = (uint32_t)w;
        }
    free(s.slot);
    memset(row_ptr, 0, (n + 1) * 8);
    for (uint64_t k = 0; k < m; ++k) {
        ++row_ptr[ea[k] + 1];
        ++row_ptr[eb[k] + 1];
    }
    for (uint64_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
    memcpy(fill, row_ptr, n * 8);
    for (uint64_t k = 0; k < m; ++k) {
        col[fill[ea[k]]++] = eb[k];
        col[fill[eb[k]]++] = ea[k];
    }
    for (uint64_t i = 0; i < n; ++i)
        qsort(col + row_ptr[i], row_ptr[i + 1] - row_ptr[i], 4, cmp_u32);
    for (uint64_t k = 0; k < 2 * m; ++k) val[k] = 1.0;
    for (uint64_t i = 0; i < n; ++i) diag[i] = 0.0;
    free(ea), free(eb), free(fill);
    return 0;
}

/* ------------------------------------------------------------- vectors */
/* kind 0: U[0,1); 1: U[-1,1) = 2u - 1; 2: Gaussian bump of width sigma at
 * the centre of the unit cube (grid point (x,y,z) at ((i+1) h - 1/2), h =
 * 1/(side+1)) plus U[0,1). */
int orc_gen_vector(int kind, uint64_t n, uint64_t side, double sigma, uint64_t seed,
                   double* out) {
    gen_rng rng;
    g_init(&rng, seed, 0);
    if (kind == 0) {
        for (uint64_t i = 0; i < n; ++i) out[i] = g_uniform(&rng);
    } else if (kind == 1) {
        for (uint64_t i = 0; i < n; ++i) out[i] = 2.0 * g_uniform(&rng) - 1.0;
    } else if (kind == 2) {
        if (side * side * side != n || !(sigma > 0.0)) return 1;
        const double h = 1.0 / (double)(side + 1);
        for (uint64_t i = 0; i < n; ++i) {
            const double x = (double)(i % side + 1) * h - 0.5;
            const double y = (double)((i / side) % side + 1) * h - 0.5;
            const double z = (double)(i / (side * side) + 1) * h - 0.5;
            out[i] = exp(-(x * x + y * y + z * z) / (2.0 * sigma * sigma)) + g_uniform(&rng);
        }
    } else {
        return 1;
    }
    return 0;
}

/* k of n rows without replacement: partial Fisher–Yates with
 * uniform_index(n - j), then sorted ascending. */
int orc_gen_row_sample(uint64_t n, uint64_t k, uint64_t seed, uint32_t* out) {
    if (k > n || n >= (1ull << 32)) return 1;
    uint32_t* a = malloc(n * 4 + 4);
    if (!a) return 2;
    for (uint64_t i = 0; i < n; ++i) a[i] = (uint32_t)i;
    gen_rng rng;
    g_init(&rng, seed, 0);
    for (uint64_t j = 0; j < k; ++j) {
        const uint64_t r = j + g_index(&rng, n - j);
        const uint32_t t = a[j];
        a[j] = a[r];
        a[r] = t;
    }
    qsort(a, k, 4, cmp_u32);
    memcpy(out, a, k * 4);
    free(a);
    return 0;
}
