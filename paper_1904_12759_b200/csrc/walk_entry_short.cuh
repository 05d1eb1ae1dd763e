// K3P — pipelined two-set shape of the K3 entry walker (included by
// walk_entry.cu, inside its anonymous namespace; shares TaskRec, the task
// stream and the combine pass with entry_walk_kernel).  EXPERIMENTAL: selected
// only by EXPMC_ENTRY_SHAPE=3 (A/B runs and the shape-parity test); measured
// slower than entry_walk_kernel on every configuration (profiles/r02/README.md).
//
// Same random-number and accumulation contract as entry_walk_kernel (gap
// rounds per (row, part), Philox counters (j, walker, row, 'ENTR'), ticket k
// of a task summed by lane k mod 32 in increasing k, xor butterfly, parts in
// index order), so oracle/fast_model.c pins it bit for bit and the two kernels
// are interchangeable on any input.  What changes is the schedule:
//
//  * Two walkers per lane (sets A and B), stepped alternately: a step of set
//    X is "sojourn of X's walkers at the state whose gather was issued one
//    step of the other set ago; refill idle lanes from the ticket ring; one
//    jump (Philox, pick, gather) for every lane".  X's gather is in flight
//    during the whole step of the other set, so each warp keeps two dependent
//    gathers outstanding instead of one.
//  * The gathered 32-byte Edge lands in registers (EPIPE_REGS=1, 87-90
//    registers, 5 blocks/SM; the slot's unused word is kept live by a store to
//    the sink slot — otherwise ptxas reuses its register right behind the load
//    and that write waits for the gather), or in shared memory by cp.async
//    (EPIPE_REGS=0, 76 registers, 6 blocks/SM; 14 shared-memory wavefronts per
//    gather instruction put the LSU data pipe at 70%).
//  * A finishing walker forms its deviation e^{Δt(S − corr)} v_end − K on the
//    spot and parks only that (8 B over its ticket) plus its jump count, so
//    the ticket ring is 12 B per ticket and the accumulation pass is a load
//    and two flops per ticket.
//  * Phases per warp instead of a per-iteration scheduler: gap rounds while a
//    round fits in the ring (G), steps while tickets remain (W), accumulation
//    of finished tickets (A).  Admission and the ready-ticket bound (a
//    min-reduction over the walkers in flight) run once per phase; walkers
//    stay in their lanes across phases.
//
// Why it loses: with 20-24 warps per SM instead of 32 the issue rate falls with
// the warp count — each warp's instruction stream is a serial dependency chain
// (stall reason `wait` ~2.7 warps per issue at every occupancy), and running
// two walkers' streams back to back in one warp adds no instruction-level
// parallelism.  Config 5: 54.0 ms (registers) / 50.1 ms (cp.async) against
// 43.7 ms; config 4: 3.27 s against 2.63 s.
#pragma once

#ifndef EPIPE_CAP
#define EPIPE_CAP 512  // tickets in the per-warp ring (power of 2, >= 256)
#endif
#ifndef EPIPE_REGS
#define EPIPE_REGS 1   // 1: the gathered Edge lands in registers (LDG.256); 0: in shared memory (cp.async)
#endif
#ifndef EPIPE_BL
#define EPIPE_BL (EPIPE_REGS ? 5 : 6)  // resident blocks per SM
#endif

template <uint32_t CAP>
struct PipeWarp {
#if !EPIPE_REGS
    uint4 land[2][2][32];  // [set][half][lane]: the lane's current Edge slot
                           //   half 0 = {j, off, deg|flags, 1/rate}, half 1 = {d, v}
#endif
    TaskRec task[ENTRY_TASKS];
    uint2 tk[CAP + 1];  // ticket: {first holding time R (fp32 bits), slot << 29 | walker};
                        // once its walker finished: the deviation (fp64); [CAP] = sink
    uint32_t tj[CAP];   // per finished ticket: its jump count
};

// A walker in flight (one per lane and set).
struct WalkP {
#if EPIPE_REGS
    unsigned long long ea, eb, ec, ed;  // the landing Edge slot: {j, off}, {deg|flags, 1/rate}, d, v
#endif
    double t, S, G;
    uint32_t tk, wl, jc, ew, off, degf;
    bool act;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint32_t src_bytes) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem),
                 "r"(src_bytes)
                 : "memory");
}

// Deviation of a finished walker (cold copy for the rare path that ends at
// the first sojourn; the hot path inlines the same operations).
__device__ __noinline__ double finish_dev_cold(double S, double G, double d, double v,
                                               double corr, double K, double dt, double n_grid1,
                                               int strang) {
    S = __fma_rn(d, __dsub_rn(n_grid1, G), S);
    if (strang) S = __dsub_rn(S, __dmul_rn(0.5, d));
    const double x = __dmul_rn(dt, __dsub_rn(S, corr));
    return __dsub_rn(__dmul_rn(exp_det(x), v), K);
}

template <int WPR, int BL>
__global__ void __launch_bounds__(128, BL)
entry_pipe_kernel(const RowRec* __restrict__ rec, const double* __restrict__ rate,
                  const Edge* __restrict__ adj, const uint32_t* __restrict__ thr,
                  const uint32_t* __restrict__ alias, const uint32_t* __restrict__ rows,
                  uint64_t nrows, FastParams p, double4* __restrict__ partial,
                  unsigned int* __restrict__ task_ctr) {
    constexpr int RT = ENTRY_TASKS;
    constexpr uint32_t CAP = EPIPE_CAP;
    static_assert((RT & (RT - 1)) == 0 && RT <= 8 && (CAP & (CAP - 1)) == 0 && CAP >= 2 * kRound,
                  "ring sizes");
    int warp = threadIdx.x >> 5;
    int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    __shared__ PipeWarp<CAP> states[4];
    // Opaque warp index, and the warp's state addressed as states[warp]
    // (no reference): otherwise the compiler rebuilds the state's address
    // from S2R SR_TID / SR_CgaCtaId at the top of every step, and the step
    // waits on those special-register reads (14% of the stall samples).
    asm volatile("" : "+r"(warp));
    asm volatile("" : "+r"(lane));
#define q states[warp]
    const uint32_t ntask = (uint32_t)(nrows * WPR);
    const uint32_t tstride = gridDim.x * 4u;

    // task ring and decision cursor: as in entry_walk_kernel
    uint32_t tw = 0, tf = 0;
    bool aopen = false;
    uint32_t oend = 0;
    bool ocl = false;
    uint32_t atask = blockIdx.x * 4u + warp;
    uint32_t apos = 0, around = 0, al0 = 0, anw = 0, atstart = 0;
    uint32_t head = 0, tail = 0;  // ticket counters: [head, tail) not yet popped
    uint32_t xc = 0;              // accumulation cursor
    double s1 = 0.0, s2 = 0.0;
    unsigned long long jsum = 0;

    auto next_task = [&]() -> uint32_t {
#if ENTRY_DYNAMIC
        uint32_t t = 0;
        if (lane == 0) t = tstride + atomicAdd(task_ctr, 1u);
        return __shfl_sync(FULL, t, 0);
#else
        return atask + tstride;
#endif
    };

    auto open_task = [&] {
        const int sl = (int)(tw & (RT - 1));
        const uint32_t i = rows ? rows[atask / WPR] : p.row0 + atask / WPR;
        const RowRec ri = load_rec(rec, i);
        const double lam = __dmul_rn(__ldg(rate + i), p.beta);
        const double ex = exp_det(lane == 0 ? -lam : __dmul_rn(p.beta, ri.d));
        const double e0 = __shfl_sync(FULL, ex, 0), e1 = __shfl_sync(FULL, ex, 1);
        const unsigned long long T0 = (unsigned long long)__dmul_rn(e0, 4294967296.0);
        const uint32_t part = atask % WPR;
        al0 = (uint32_t)(p.W * part / WPR);
        anw = (uint32_t)(p.W * (part + 1) / WPR) - al0;
        const bool dead = (T0 >> 32) != 0 || anw == 0;
        if (lane == 0) {
            TaskRec& a = q.task[sl];
            a.rr = RowRecU{ri.off, ri.deg_flags, ri.inv_rate,
                           dead ? 0u : __float_as_uint((float)__drcp_rn(lam)), ri.d, ri.v};
            a.i = i;
            a.n0 = anw;
            a.tend = tail;
            a.task = atask;
            a.closed = dead ? 1u : 0u;
            a.lam = (float)lam;
            const double f0 = __dmul_rn(e1, ri.v);
            a.f0 = f0;
            a.K = T0 >= (1ull << 31) ? f0 : 0.0;
            a.corr = p.strang ? __dmul_rn(0.5, ri.d) : ri.d;
        }
        if (tf == tw) {
            ocl = dead;
            oend = tail;
        }
        ++tw;
        apos = 0;
        around = 0;
        atstart = tail;
        if (dead) {
            atask = next_task();
        } else {
            aopen = true;
        }
        __syncwarp();
    };

    auto can_admit = [&] {
        return aopen ? tail + kRound - xc <= CAP : (atask < ntask && tw - tf < (uint32_t)RT);
    };
    // One gap round of the open task (see entry_walk_kernel::admit: same draws,
    // same ticket order).
    auto admit = [&] {
        if (!aopen) {
            open_task();
            return;
        }
        const uint32_t sl = (tw - 1) & (RT - 1);
        const TaskRec& a = q.task[sl];
        const float lamf = a.lam, ilam = __uint_as_float(a.rr.spare);
        const U4 D = philox4x32_10(
            U4{0xfffffff0u | (atask % WPR), 32u * around + (uint32_t)lane, a.i, kTagEntry}, p.rk);
        const uint32_t wd[4] = {D.x, D.y, D.z, D.w};
        uint32_t off[4];
        float R[4];
        uint32_t loc = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float E = neg_ln_u(wd[k]);
            const float kf = fminf(floorf(__fmul_rn(E, ilam)), 134217728.0f);
            R[k] = fmaxf(__fmaf_rn(-lamf, kf, E), 0.0f);
            off[k] = loc + (uint32_t)kf;
            loc = off[k] + 1u;
        }
        uint32_t inc = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc = min(inc + y, 0x7fffffffu);
        }
        const uint32_t exc = inc - loc;
        const uint32_t total = __shfl_sync(FULL, inc, 31);
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t P = apos + exc + off[k];
            const bool ok = P < anw;
            cnt += __popc(__ballot_sync(FULL, ok));
            const uint32_t pos = ok ? ((tail + 4u * lane + k) & (CAP - 1)) : CAP;
            q.tk[pos] = make_uint2(__float_as_uint(R[k]), (sl << 29) | (al0 + P));
        }
        tail += cnt;
        apos = min(apos + total, 0x7fffffffu);
        ++around;
        if (apos >= anw) {
            if (lane == 0) {
                q.task[sl].tend = tail;
                q.task[sl].closed = 1u;
                q.task[sl].n0 = anw - (tail - atstart);
            }
            if (tw - 1 == tf) {
                ocl = true;
                oend = tail;
            }
            aopen = false;
            atask = next_task();
        }
        __syncwarp();
    };

    // Park the deviation of a finished walker in its ticket.
    auto park = [&](WalkP& s, double dv) {
        const uint32_t pos = s.tk & (CAP - 1);
        *reinterpret_cast<double*>(&q.tk[pos]) = dv;
        q.tj[pos] = s.jc;
        s.act = false;
    };

    // One step of a walker set: sojourn at the landed state, refill, jump.
    auto step = [&](WalkP& s, const int set) {
        // this set's gather was committed before the other set's: landed
#if EPIPE_REGS
        if (s.act) {
            const uint4 e0 = make_uint4((uint32_t)s.ea, (uint32_t)(s.ea >> 32), (uint32_t)s.eb,
                                        (uint32_t)(s.eb >> 32));
            const double2 e1 = make_double2(__longlong_as_double((long long)s.ec),
                                            __longlong_as_double((long long)s.ed));
#else
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        if (s.act) {
            const uint4 e0 = q.land[set][0][lane];
            const double2 e1 = *reinterpret_cast<const double2*>(&q.land[set][1][lane]);
#endif
            const float h = __fmul_rn(neg_ln_u(s.ew), __uint_as_float(e0.w));
            const double tn = __dadd_rn(s.t, __dmul_rn((double)h, p.inv_dt));
            const double d = e1.x;
            if (tn >= p.n_grid) {
                // the path ends in this state: run_path's product
                // (estimator.cpp:26-39), Strang half weight at the end state
                double S = __fma_rn(d, __dsub_rn(p.n_grid1, s.G), s.S);
                if (p.strang) S = __dsub_rn(S, __dmul_rn(0.5, d));
                const TaskRec& m = q.task[s.wl >> 29];
                const double x = __dmul_rn(p.dt, __dsub_rn(S, m.corr));
                park(s, __dsub_rn(__dmul_rn(exp_det(x), e1.y), m.K));
#if EPIPE_REGS
                // The landing row id (word 0 of the slot) is not needed, and a
                // dead word's register is reused right behind the load: that
                // write then waits for the load to land (WAW) and serialises
                // the two sets.  Storing it to the sink slot on this path
                // keeps the register occupied while the gather is in flight.
                q.tk[CAP].x = e0.x;
#endif
            } else {
                const double kk = ceil(tn);
                s.S = __fma_rn(d, __dsub_rn(kk, s.G), s.S);
                s.G = kk;
                s.t = tn;
                s.off = e0.y;
                s.degf = e0.z;
            }
        }
        // idle lanes take the next tickets in order
        const unsigned idle = __ballot_sync(FULL, !s.act);
        const uint32_t avail = tail - head;
        if (idle != 0u && avail != 0u) {
            const uint32_t nidle = (uint32_t)__popc(idle);
            const uint32_t take = avail < nidle ? avail : nidle;
            const uint32_t rank = (uint32_t)__popc(idle & lt);
            if (!s.act && rank < take) {
                s.tk = head + rank;
                const uint2 t2 = q.tk[s.tk & (CAP - 1)];
                s.wl = t2.y;
                const TaskRec& m = q.task[t2.y >> 29];
                const uint4 r0 = *reinterpret_cast<const uint4*>(&m.rr);  // off, degf, ir, -
                const double d = m.rr.d;
                s.jc = 0;
                s.act = true;
                // a jumper's first sojourn (R < λ) ends in a jump, up to the
                // rounding of R / rate
                const float h = __fmul_rn(__uint_as_float(t2.x), __uint_as_float(r0.z));
                const double tn = __dadd_rn(0.0, __dmul_rn((double)h, p.inv_dt));
                if (tn >= p.n_grid) {
                    park(s, finish_dev_cold(0.0, 0.0, d, m.rr.v, m.corr, m.K, p.dt, p.n_grid1,
                                            p.strang));
                } else {
                    const double kk = ceil(tn);
                    s.S = __fma_rn(d, __dsub_rn(kk, 0.0), 0.0);
                    s.G = kk;
                    s.t = tn;
                    s.off = r0.x;
                    s.degf = r0.y;
                }
            }
            head += take;
        }
        // one jump for every walker in flight: Philox block (jumps so far,
        // walker, row), neighbour pick, alias correction on weighted rows,
        // and the gather of the landing Edge into the lane's slot
        {
            const uint32_t wi = q.task[s.wl >> 29].i;
            const U4 B = philox4x32_10(U4{s.jc, s.wl & 0x1fffffffu, wi, kTagEntry}, p.rk);
            uint32_t k = pick_index(B.y, B.w, s.degf & kDegMask);
            if (s.act && (s.degf & kNonUniform) && B.z >= __ldg(thr + s.off + k))
                k = __ldg(alias + s.off + k);
#if EPIPE_REGS
            ld256_gather(adj + (s.act ? s.off + k : 0u), s.ea, s.eb, s.ec, s.ed);
#else
            const char* src = reinterpret_cast<const char*>(adj + (s.act ? s.off + k : 0u));
            const uint32_t nb = s.act ? 16u : 0u;
            cp_async16(&q.land[set][0][lane], src, nb);
            cp_async16(&q.land[set][1][lane], src + 16, nb);
            asm volatile("cp.async.commit_group;" ::: "memory");
#endif
            s.ew = B.x;
            ++s.jc;
        }
    };

    // Phase A: sum the finished tickets in batches of 32 consecutive tickets
    // of the oldest task (lane = ticket - tstart mod 32) and finalize
    // completed tasks.  Tickets before `head` are finished except those of
    // the walkers in flight.
    auto accumulate = [&](const WalkP& a, const WalkP& b) {
        uint32_t rdy = head - xc;
        {
            const uint32_t oa = a.act ? a.tk - xc : ~0u, ob = b.act ? b.tk - xc : ~0u;
            const uint32_t m = __reduce_min_sync(FULL, oa < ob ? oa : ob);
            rdy = rdy < m ? rdy : m;
        }
        if (!(rdy >= 32u || (ocl && rdy >= oend - xc))) return;
        __syncwarp();
        while (tf != tw) {
            const TaskRec& m = q.task[tf & (RT - 1)];
            const uint32_t lim = ocl && oend - xc < rdy ? oend - xc : rdy;
            uint32_t nb;
            if (lim >= 32u) {
                nb = 32u;
            } else if (ocl && lim == oend - xc) {
                nb = lim;
            } else {
                break;
            }
            if (nb) {
                if ((uint32_t)lane < nb) {
                    const uint32_t pos = (xc + lane) & (CAP - 1);
                    const double dv = *reinterpret_cast<const double*>(&q.tk[pos]);
                    s1 = __dadd_rn(s1, dv);
                    s2 = __fma_rn(dv, dv, s2);
                    jsum += q.tj[pos];
                }
                xc += nb;
                rdy -= nb;
            }
            if (!ocl || xc != oend) continue;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                s1 = __dadd_rn(s1, __shfl_xor_sync(FULL, s1, o));
                s2 = __dadd_rn(s2, __shfl_xor_sync(FULL, s2, o));
                jsum += __shfl_xor_sync(FULL, jsum, o);
            }
            if (lane == 0) {
                const double f0 = m.f0, K = m.K;
                const uint32_t n0 = m.n0;
                const double c = __dsub_rn(f0, K);
                if (n0 != 0 && c != 0.0) {
                    s1 = __fma_rn((double)n0, c, s1);
                    s2 = __fma_rn((double)n0, __dmul_rn(c, c), s2);
                }
                partial[m.task] = make_double4(s1, s2, __longlong_as_double((long long)jsum), K);
            }
            s1 = 0.0;
            s2 = 0.0;
            jsum = 0;
            ++tf;
            __syncwarp();
            ocl = false;
            if (tf != tw) {
                const uint2 e = *reinterpret_cast<const uint2*>(&q.task[tf & (RT - 1)].tend);
                ocl = e.y != 0u;
                oend = e.x;
            }
        }
    };

    WalkP A;
#if EPIPE_REGS
    A.ea = A.eb = A.ec = A.ed = 0;
#endif
    A.t = A.S = A.G = 0.0;
    A.tk = A.wl = A.jc = A.ew = A.off = A.degf = 0;
    A.act = false;
    WalkP B = A;
    while (true) {
        // ---- G: gap rounds while a whole round's tickets fit in the ring
        // (the gathers of the walkers in flight land meanwhile)
        while (can_admit()) admit();
        // ---- W: steps of A and B while tickets remain; with nothing new
        // (ring or task slots blocked by walkers in flight, or the last
        // tasks) until every walker in flight has finished
        const bool drain = head == tail;
        for (;;) {
            step(A, 0);
            step(B, 1);
            if (head == tail && !(drain && __any_sync(FULL, A.act || B.act))) break;
        }
        __syncwarp();
        // ---- A
        accumulate(A, B);
        if (tf == tw && !aopen && atask >= ntask) break;
    }
#undef q
}
