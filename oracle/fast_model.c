/*
 * TEST INFRASTRUCTURE ONLY — a CPU model of the B200 production walker
 * (K3 entry_walk_kernel, paper_1904_12759_b200/csrc/walk_entry.cu), written
 * independently from the kernel's contract so the GPU can be pinned walker
 * for walker, not only statistically.
 *
 * The law it samples is the reference's (entry_estimate, Theorem 1:
 * proj/src/estimator.cpp:169-206 with run_path :26-39 and advance
 * sampler.cpp:36-49), with the two re-formulations the kernel makes:
 *   - one exponential clock per sojourn instead of one per Δt segment
 *     (memorylessness), crediting d_s to each grid point kΔt
 *     covered by the sojourn (half weight at k = 0 and k = N for Strang);
 *   - Philox4x32-10 keyed by the seed, counter (step, walker, row, 'ENTR').
 * That this law matches the reference is checked statistically against
 * oracle/_ref (tests/test_oracle.py); that the GPU matches this model is
 * checked per entry (tests/test_gpu_parity.py).
 *
 * Build with -ffp-contract=off: every float/double operation below is a
 * single IEEE operation, exactly like the __*_rn intrinsics of the kernel.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint32_t off, degf;
    float inv_rate;
    uint32_t spare;
    double d, v;
} fm_rec;

#define FM_NONUNIFORM 0x80000000u
#define FM_DEGMASK 0x7fffffffu
#define FM_TAG_ENTRY 0x454e5452u

void fm_philox(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* neg_ln_u of csrc/common.cuh: -ln(u), u = (w | 1) 2^-32, same operations
 * in the same order. */
float fm_neg_ln_u(uint32_t w) {
    const float fx = (float)(w | 1u); /* round to nearest, as __uint2float_rn */
    uint32_t bits;
    memcpy(&bits, &fx, 4);
    int e = (int)(bits >> 23) - 127;
    const uint32_t mb = (bits & 0x007fffffu) | 0x3f800000u;
    float m;
    memcpy(&m, &mb, 4);
    if (m > 1.41421356f) {
        m = m * 0.5f;
        e += 1;
    }
    const float f = m - 1.0f;
    float q = 0.08743945509195328f;
    q = fmaf(q, f, -0.14377330243587494f);
    q = fmaf(q, f, 0.14949095249176025f);
    q = fmaf(q, f, -0.16560696065425873f);
    q = fmaf(q, f, 0.19956977665424347f);
    q = fmaf(q, f, -0.2500215470790863f);
    q = fmaf(q, f, 0.3333418369293213f);
    q = fmaf(q, f, -0.49999988079071045f);
    q = fmaf(q, f, 1.0f);
    const float E = fmaf((float)(32 - e), 0.693147182f, -(f * q));
    return E > 0.0f ? E : 0.0f;
}

/* exp_det of csrc/common.cuh: the kernel's deterministic fp64 exp
 * (table-driven, double-double 2^(j/32), degree-6 e^r - 1, branch-free
 * range handling; same operations in the same order). */
static const double fm_exptab[32][2] = {
    {0x1.0000000000000p+0, 0x0.0p+0},
    {0x1.059b0d3158574p+0, 0x1.d73e2a475b465p-55},
    {0x1.0b5586cf9890fp+0, 0x1.8a62e4adc610bp-54},
    {0x1.11301d0125b51p+0, -0x1.6c51039449b3ap-54},
    {0x1.172b83c7d517bp+0, -0x1.19041b9d78a76p-55},
    {0x1.1d4873168b9aap+0, 0x1.e016e00a2643cp-54},
    {0x1.2387a6e756238p+0, 0x1.9b07eb6c70573p-54},
    {0x1.29e9df51fdee1p+0, 0x1.612e8afad1255p-55},
    {0x1.306fe0a31b715p+0, 0x1.6f46ad23182e4p-55},
    {0x1.371a7373aa9cbp+0, -0x1.63aeabf42eae2p-54},
    {0x1.3dea64c123422p+0, 0x1.ada0911f09ebcp-55},
    {0x1.44e086061892dp+0, 0x1.89b7a04ef80d0p-59},
    {0x1.4bfdad5362a27p+0, 0x1.d4397afec42e2p-56},
    {0x1.5342b569d4f82p+0, -0x1.07abe1db13cadp-55},
    {0x1.5ab07dd485429p+0, 0x1.6324c054647adp-54},
    {0x1.6247eb03a5585p+0, -0x1.383c17e40b497p-54},
    {0x1.6a09e667f3bcdp+0, -0x1.bdd3413b26456p-54},
    {0x1.71f75e8ec5f74p+0, -0x1.16e4786887a99p-55},
    {0x1.7a11473eb0187p+0, -0x1.41577ee04992fp-55},
    {0x1.82589994cce13p+0, -0x1.d4c1dd41532d8p-54},
    {0x1.8ace5422aa0dbp+0, 0x1.6e9f156864b27p-54},
    {0x1.93737b0cdc5e5p+0, -0x1.75fc781b57ebcp-57},
    {0x1.9c49182a3f090p+0, 0x1.c7c46b071f2bep-56},
    {0x1.a5503b23e255dp+0, -0x1.d2f6edb8d41e1p-54},
    {0x1.ae89f995ad3adp+0, 0x1.7a1cd345dcc81p-54},
    {0x1.b7f76f2fb5e47p+0, -0x1.5584f7e54ac3bp-56},
    {0x1.c199bdd85529cp+0, 0x1.11065895048ddp-55},
    {0x1.cb720dcef9069p+0, 0x1.503cbd1e949dbp-56},
    {0x1.d5818dcfba487p+0, 0x1.2ed02d75b3707p-55},
    {0x1.dfc97337b9b5fp+0, -0x1.1a5cd4f184b5cp-54},
    {0x1.ea4afa2a490dap+0, -0x1.e9c23179c2893p-54},
    {0x1.f50765b6e4540p+0, 0x1.9d3e12dd8a18bp-54}};

double fm_exp(double x) {
    if (x != x) return x;
    x = x > 710.0 ? 710.0 : x;
    x = x < -746.0 ? -746.0 : x;
    const double n = rint(x * 0x1.71547652b82fep+5);
    double r = fma(-n, 0x1.62e42fee00000p-6, x);
    r = fma(-n, 0x1.a39ef35793c76p-38, r);
    double p = 1.0 / 720.0;
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = p * r;
    const int ni = (int)n;
    const double* t = fm_exptab[ni & 31];
    const double y = t[0] + fma(t[0], p, t[1]);
    const int k = ni >> 5;
    const int k1 = k >> 1, k2 = k - k1;
    uint64_t b1 = (uint64_t)(k1 + 1023) << 52, b2 = (uint64_t)(k2 + 1023) << 52;
    double s1, s2;
    memcpy(&s1, &b1, 8);
    memcpy(&s2, &b2, 8);
    return (y * s1) * s2;
}

static uint32_t fm_pick(uint32_t hi, uint32_t lo, uint32_t n) {
    const uint64_t x = ((uint64_t)hi << 32) | lo;
    return (uint32_t)(((unsigned __int128)x * n) >> 64);
}

/* Records as split_pack builds them (csrc/split_pack.cu). */
void fm_build_records(uint64_t n, const uint64_t* row_ptr, const double* rate,
                      const double* d, const uint8_t* uniform_row, const double* v,
                      fm_rec* rec) {
    for (uint64_t i = 0; i < n; ++i) {
        rec[i].off = (uint32_t)row_ptr[i];
        rec[i].degf = (uint32_t)(row_ptr[i + 1] - row_ptr[i]) |
                      (uniform_row[i] ? 0u : FM_NONUNIFORM);
        rec[i].inv_rate = (float)(1.0 / rate[i]);
        rec[i].spare = 0;
        rec[i].d = d[i];
        rec[i].v = v[i];
    }
}

/* Deviation f - f0 of jumper l of row i, whose first holding time is
 * E0 / rate_i (E0 = R of its gap, already < λ).  Jump j draws counter
 * (j, l, i, tag): y,w = 64-bit pick, z = alias coin, x = next holding time. */
static double fm_walker(const fm_rec* rec, const uint32_t* nbr, const uint32_t* thr,
                        const uint32_t* alias, uint32_t i, uint32_t l, float E0, double f0,
                        double corr_i, double dt, double inv_dt, double n_grid, uint64_t N,
                        int strang, uint32_t k0, uint32_t k1, uint64_t* jumps) {
    fm_rec cur = rec[i];
    float E = E0;
    uint32_t g = 0, jc = 0;
    double t = 0.0, S = 0.0;
    for (;;) {
        const float h = E * cur.inv_rate;
        const double tn = t + (double)h * inv_dt;
        if (tn >= n_grid) {
            S = fma(cur.d, (double)(N + 1 - g), S);
            /* the kernel parks S - d_end/2 (Strang) and forms the exponent
             * at accumulation: x = dt * (S' - corr_i) */
            const double Sp = strang ? S - 0.5 * cur.d : S;
            const double x = dt * (Sp - corr_i);
            *jumps += jc;
            return fm_exp(x) * cur.v - f0;
        }
        const uint32_t kk = (uint32_t)ceil(tn);
        S = fma(cur.d, (double)(kk - g), S);
        g = kk;
        t = tn;
        const uint32_t ctr[4] = {jc, l, i, FM_TAG_ENTRY};
        uint32_t w[4];
        fm_philox(ctr, k0, k1, w);
        uint32_t k = fm_pick(w[1], w[3], cur.degf & FM_DEGMASK);
        if (cur.degf & FM_NONUNIFORM) {
            if (w[2] >= thr[cur.off + k]) k = alias[cur.off + k];
        }
        cur = rec[nbr[cur.off + k]];
        E = fm_neg_ln_u(w[0]);
        ++jc;
    }
}

/* Accumulation contract of the kernel.  Part w (of WPR = T/32 parts) owns
 * the walkers [floor(wW/WPR), floor((w+1)W/WPR)).  They are decided by a
 * stream of gap rounds: round r draws Philox counters (0xfffffff0 | w,
 * 32r + s, i, tag) for s = 0..31, and the 128 words, in order (s, word),
 * give E = -ln u ~ Exp(1), K = min(floor(E * (1/λ)), 2^27) never-jumpers
 * and then one jumper with first holding time R/rate, R = max(E - λK, 0)
 * (fp32, λ = rate β).  The part's jumpers, numbered k = 0, 1, ... in walker
 * order, are summed by lane k mod 32 in increasing k; xor butterfly over
 * lanes; parts in index order. */
void fm_entries(const fm_rec* rec, const double* rate, const uint32_t* nbr,
                const uint32_t* thr, const uint32_t* alias, const uint32_t* rows,
                uint64_t nrows, double beta, uint64_t N, uint64_t W, int strang,
                uint64_t seed, uint32_t T, double* value, double* se,
                uint64_t* jumps) {
    const double dt = beta / (double)N;
    const double inv_dt = 1.0 / dt;
    const double n_grid = (double)N;
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    const uint32_t wpr = T / 32;
    for (uint64_t r = 0; r < nrows; ++r) {
        const uint32_t i = rows[r];
        const fm_rec ri = rec[i];
        const double lam = rate[i] * beta;
        const double p0 = fm_exp(-lam);
        const uint64_t T0 = (uint64_t)(p0 * 4294967296.0);
        const double f0 = fm_exp(beta * ri.d) * ri.v;
        /* deviation shift: f0 if never-jumpers are the majority, else 0 */
        const double K = T0 >= (1ull << 31) ? f0 : 0.0;
        const double corr_i = strang ? 0.5 * ri.d : ri.d;
        const int dead = (T0 >> 32) != 0;
        const float lamf = (float)lam;
        const float ilam = dead ? 0.0f : (float)(1.0 / lam);
        double w1 = 0.0, w2 = 0.0;
        uint64_t wj = 0;
        for (uint32_t wi = 0; wi < wpr; ++wi) {
            const uint32_t L0 = (uint32_t)(W * wi / wpr);
            const uint32_t nw = (uint32_t)(W * (wi + 1) / wpr) - L0;
            double b1[32], b2[32];
            uint64_t bj[32];
            for (int s = 0; s < 32; ++s) { b1[s] = 0.0; b2[s] = 0.0; bj[s] = 0; }
            uint64_t nj = 0;  /* jumpers of this part */
            if (!dead && nw > 0) {
                uint64_t pos = 0; /* next undecided part-local walker */
                for (uint32_t round = 0; pos < nw; ++round) {
                    for (uint32_t s = 0; s < 32 && pos < nw; ++s) {
                        const uint32_t ctr[4] = {0xfffffff0u | wi, 32u * round + s, i,
                                                 FM_TAG_ENTRY};
                        uint32_t wd[4];
                        fm_philox(ctr, k0, k1, wd);
                        for (int q = 0; q < 4 && pos < nw; ++q) {
                            const float E = fm_neg_ln_u(wd[q]);
                            float kf = floorf(E * ilam);
                            if (kf > 134217728.0f) kf = 134217728.0f;
                            float R = fmaf(-lamf, kf, E);
                            if (R < 0.0f) R = 0.0f;
                            pos += (uint64_t)kf;
                            if (pos >= nw) break;
                            uint64_t jl = 0;
                            const double dev =
                                fm_walker(rec, nbr, thr, alias, i, L0 + (uint32_t)pos, R, K,
                                          corr_i, dt, inv_dt, n_grid, N, strang, k0, k1, &jl);
                            const int ln = (int)(nj++ % 32);
                            b1[ln] = b1[ln] + dev;
                            b2[ln] = fma(dev, dev, b2[ln]);
                            bj[ln] += jl;
                            pos += 1;
                        }
                    }
                }
            }
            const uint32_t n0 = nw - (uint32_t)nj; /* never-jumpers of this part */
            for (int o = 16; o > 0; o >>= 1) {
                double c1[32], c2[32];
                uint64_t cj[32];
                for (int q = 0; q < 32; ++q) {
                    c1[q] = b1[q] + b1[q ^ o];
                    c2[q] = b2[q] + b2[q ^ o];
                    cj[q] = bj[q] + bj[q ^ o];
                }
                memcpy(b1, c1, sizeof(c1));
                memcpy(b2, c2, sizeof(c2));
                memcpy(bj, cj, sizeof(cj));
            }
            /* never-jumpers score f0: deviation f0 - K each, added after the
             * butterfly (exactly zero when K = f0) */
            const double cdev = f0 - K;
            if (n0 != 0 && cdev != 0.0) {
                b1[0] = fma((double)n0, cdev, b1[0]);
                b2[0] = fma((double)n0, cdev * cdev, b2[0]);
            }
            if (wi == 0) { w1 = b1[0]; w2 = b2[0]; wj = bj[0]; }
            else { w1 = w1 + b1[0]; w2 = w2 + b2[0]; wj += bj[0]; }
        }
        const double Wd = (double)W;
        value[r] = K + w1 / Wd;
        double sev = 0.0;
        if (W > 1) {
            double var = (w2 - (w1 * w1) / Wd) / (Wd - 1.0);
            if (var < 0.0) var = 0.0;
            sev = sqrt(var / Wd);
        }
        se[r] = sev;
        jumps[r] = wj;
    }
}
