// K3 entry walker — production kernel for the batched entry estimator
// (Theorem 1; reference entry_estimate, proj/src/estimator.cpp:169-206).
//
// Same law as the reference for every walker, re-designed for SIMT:
//
//  * Continuous clock (memorylessness): one exponential per
//    sojourn; a sojourn in state s over grid time [t, t') credits d_s to every
//    grid point k Δt inside it, half weights at k = 0 and k = N for Strang
//    (run_path, estimator.cpp:26-39).  Cost O(1 + jumps) per walker.
//  * Philox4x32-10 keyed by the seed.  Walkers are decided by gaps: part w
//    of row i owns walkers [wW/WPR, (w+1)W/WPR); gap round r draws counters
//    (0xfffffff0 | w, 32r + lane, i, 'ENTR'), and each of the 128 words gives
//    E = -ln u ~ Exp(1) = λK + R (λ = rate_i β): K = ⌊E/λ⌋ walkers that never
//    jump (Geometric), then one jumper whose first holding time is R/rate_i
//    (R ~ Exp(1) truncated to [0, λ), independent of K).  Jumper l's j-th
//    jump draws counter (j, l, i, 'ENTR'): words y,w = 64-bit neighbour pick,
//    z = alias coin, x = next holding time.  Randomness is a pure function of
//    (seed, row, part, walker).
//  * Walkers that never jump score the deterministic f0 = e^{β d_i} v_i; sums
//    are kept as deviations from a shift K (f0 when never-jumpers dominate),
//    so they contribute exact zeros, and cost nothing: decisions cost ~1.6
//    warp instructions per jumper instead of a quarter Philox per walker.
//  * One dependent 32-B gather per jump through the fat adjacency (Edge),
//    marked L1::no_allocate (no L1 line per gather in flight: the shared-
//    memory carveout no longer limits the gathers outstanding per SM).
//  * Warp-cooperative scheduling over a stream of tasks.  Task t = (row
//    t / WPR, part t % WPR).  A warp runs gap rounds (one Philox block per
//    lane, 128 gaps) and appends the jumpers as tickets (first holding time,
//    walker) to a shared-memory ring of CAP tickets (up to
//    ENTRY_TASKS tasks in flight); idle lanes pop tickets in order, across
//    chunk and row boundaries, so the sojourn code runs with (nearly) full
//    warps.  A finishing walker only parks its raw weight sum S, end value v
//    and jump count in its ticket.  Tickets of a task are contiguous, so they
//    are accumulated in batches of 32 consecutive tickets of the oldest task
//    (exponent, exp() and deviation convergent over the batch, ticket k of
//    the task on lane k mod 32, straight into that lane's running sums), and
//    a task is finalized once its last batch is in.
//  * One loop trip = jump (Philox, pick, gather issued, next -ln u) ->
//    accumulate / finalize -> sojourn at the gathered state -> admit / pop.
//    The gather is consumed in the trip that issued it, after the
//    accumulation work, in the registers it landed in (see the main loop).
//  * Fixed accumulation order (result contract, replayed by
//    oracle/fast_model.c): the jumpers of part w, numbered k = 0, 1, ... in
//    increasing l, are summed by lane k mod 32 in increasing k; lanes are
//    combined by an xor butterfly, parts in index order.  Independent of
//    scheduling, grid shape, GPU count and row sharding.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace expmc_b200 {

namespace {

constexpr int kRound = 128;  // gaps per warp round (4 per lane): at most kRound tickets
constexpr unsigned FULL = 0xffffffffu;

#ifndef ENTRY_TASKS
#define ENTRY_TASKS 8   // tasks in flight per warp (power of 2, <= 8: slot in 3 ticket bits)
#endif
#ifndef ENTRY_CAP
#define ENTRY_CAP 256   // jumper tickets in flight per warp (power of 2, >= 128)
#endif
#ifndef ENTRY_CARVE
#define ENTRY_CARVE 1     // size the smem carveout for the resident block count (max L1)
#endif
#ifndef ENTRY_DYNAMIC
#define ENTRY_DYNAMIC 1 // tasks after the first grid-full from a global counter (0: static stride)
#endif
#ifndef ENTRY_SWZ
#define ENTRY_SWZ 0 // 1: swizzle the ticket ring (measured 1.5% slower: the conflicts are not the limiter)
#endif
#ifndef ENTRY_TAB_SHARED
#define ENTRY_TAB_SHARED 1 // exp table in shared memory (8-block shape)
#endif
#ifndef ENTRY_LONG_WALK
#define ENTRY_LONG_WALK 8.0 // mean jumps per walker (β · mean rate) from which the long-walk gate applies
#endif
#ifndef ENTRY_GATE_MASK
#define ENTRY_GATE_MASK 15 // long walks: ready-ticket bound every 16th trip (cfg4: every trip 2628, 2nd 2648, 4th 2597, 8th 2577 ms; with the slim state 8th 2527, 16th 2519, 32nd ~2515)
#endif
#ifndef ENTRY_EXP_INRANGE
#define ENTRY_EXP_INRANGE 1 // clamp-free exp_det when the launch's exponents are provably within range
#endif
#ifndef ENTRY_POP_MIN
#define ENTRY_POP_MIN 3 // run the scheduler once this many lanes are idle (cfg4, slim state: 3 -> 2511, 4 -> 2527, 5 -> 2641 ms)
#endif

// Self-checking build (make variants VARIANTS="checks:-DEXPMC_CHECKS"): the
// invariants of the warp-synchronous ticket ring, asserted on the device.
// compute-sanitizer is closed on this pool (profiles/r02/sanitizer_closed_*),
// so this build, run under the bit-exact model tests with every launch shape
// and row sharding, is the race / bounds evidence (scripts/gpu_checks.sh).
#ifdef EXPMC_CHECKS
#define CHK(c)                                                                          \
    do {                                                                                \
        if (!(c)) {                                                                     \
            printf("K3 check failed: %s (line %d) block %d thread %d\n", #c, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                  \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
constexpr unsigned long long kUnfinished = 0x7ff8dead00000001ull;  // NaN: ticket popped, not parked
#else
#define CHK(c) ((void)0)
#endif

// Physical slot of ticket position `pos` in the tk ring.  A gap round
// stores ticket (lane, k) at tail + 4 lane + k: 8-byte slots 32 bytes apart
// hit 4 bank pairs (8-way conflicts).  XOR-ing bits 4-5 into bits 0-1
// spreads them over 16 bank pairs; consecutive positions (pops, batches)
// stay conflict-free, and the sink slot CAP maps to itself (CAP % 64 == 0).
__device__ __forceinline__ uint32_t tk_slot(uint32_t pos) {
#if ENTRY_SWZ
    return pos ^ ((pos >> 4) & 3u);
#else
    return pos;
#endif
}

struct RowRecU {     // RowRec without its 32-byte alignment (smem copy)
    uint32_t off, deg_flags;
    float inv_rate;
    uint32_t spare;
    double d, v;
};

// One task in flight (row, part): the start row's constants and the task's
// ticket range.  Tickets of a task are contiguous in ticket-counter space
// (chunks are admitted task by task), so the accumulation lane of a jumper
// is its part-local jumper index mod 32 = (ticket - tstart) mod 32.
struct __align__(16) TaskRec {
    RowRecU rr;      // record of the start row (rr.spare: 1/λ as fp32 bits)
    uint32_t i;      // matrix row
    uint32_t n0;     // walkers of the task part; once closed: its never-jumpers
    uint32_t tend;   // one past its last ticket (valid once closed)
    uint32_t closed; // all walkers decided (read with tend as one 8-byte word)
    float lam;       // λ = rate_i β (fp32), the never-jump exponent
    uint32_t task;   // task id (row index in the launch, times WPR, plus part)
    double f0;       // e^{β d_i} v_i (score of a walker that never jumps)
    double K;        // shift of the deviation sums: f0 when never-jumpers are the
                     // majority (T0 >= 2^31), else 0 (no cancellation against a
                     // huge f0 that no walker realises, e.g. BA hubs)
    double corr;     // weight correction at the start state (½ d_i Strang, d_i Lie)
};
static_assert(sizeof(TaskRec) == 80, "task layout");

template <int RT, int CAP>
struct WarpState {
    double S[CAP];      // per ticket: raw weight sum at finish
    double v[CAP];      // per ticket: v at the end state
    TaskRec task[RT];   // (16-byte aligned: the pop reads rr as one uint4)
    uint2 tk[CAP + 1];  // per ticket: {first holding time R·rate (fp32) until popped,
                        //   then the jump count; task slot << 29 | walker l}; the
                        //   last is the sink of the sweep's unconditional stores
                        //   (4 warps x 6800 B + the 512-B exp table: 8 blocks per
                        //   SM under the 228 KB carveout)
};

#ifdef ENTRY_STATS
// [0] iterations [1] idle lanes at pop [2] lanes left idle [3] ...while
// tasks remain (ring capacity) [4] jumping lanes [5] active lanes
#endif

// (WT = false: a matrix without weighted rows — every configuration of the
// benchmark — needs neither the flag bit nor the alias test in the jump.
// SPL = 0 / 1: the splitting (Lie / Strang) known at compile time, -1: read
// from the parameters; XS: the launch's exponents are known to be in range,
// else p.exp_safe decides per batch.  The launcher picks the instantiation;
// the operations on the data are the same in all of them.)
template <int WPR, int BL, int GM = 0, bool WT = true, int SPL = -1, bool XS = false>
__global__ void __launch_bounds__(128, BL)
entry_walk_kernel(const RowRec* __restrict__ rec, const double* __restrict__ rate,
                  const Edge* __restrict__ adj, const uint32_t* __restrict__ thr,
                  const uint32_t* __restrict__ alias, const uint32_t* __restrict__ rows,
                  uint64_t nrows, FastParams p, double4* __restrict__ partial,
                  unsigned int* __restrict__ task_ctr) {
    constexpr int RT = ENTRY_TASKS;
    constexpr uint32_t CAP = ENTRY_CAP;
    static_assert((RT & (RT - 1)) == 0 && RT <= 8 && (CAP & (CAP - 1)) == 0 && CAP >= kRound,
                  "ring sizes");
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const bool strang = SPL < 0 ? p.strang != 0 : SPL == 1;
    const bool xsafe = XS || p.exp_safe != 0;
    __shared__ WarpState<RT, CAP> states[4];
    // exp_det's 2^(j/32) table: a shared-memory copy for the 8-block shape
    // (the accumulation batches waited on its L1 lookups: 6.6% of the stall
    // samples).  The 7-block shape keeps the L1 table: 512 B more per block
    // would not fit its 196 KB carveout.
    constexpr bool kTabShared = ENTRY_TAB_SHARED && BL >= 8;
    __shared__ double2 s_tab[kTabShared ? 32 : 1];
    if (kTabShared) {
        if (threadIdx.x < 32) s_tab[threadIdx.x] = kExpTab[threadIdx.x];
        __syncthreads();
    }
    WarpState<RT, CAP>& q = states[warp];
    const uint32_t ntask = (uint32_t)(nrows * WPR);
    const uint32_t tstride = gridDim.x * 4u;

    // task ring (warp-uniform counters): tasks [tf, tw) are in flight, the
    // newest is being swept while `aopen`
    uint32_t tw = 0, tf = 0;
    bool aopen = false;
    // register copy of the oldest task's {tend, closed} (ocl false: none or open)
    uint32_t oend = 0;
    bool ocl = false;
    uint32_t atask = blockIdx.x * 4u + warp;  // next task to open / the open task
    // the open task's decision cursor: next undecided walker (part-local),
    // gap round, part walker range [al0, al0 + anw), first ticket
    uint32_t apos = 0, around = 0, al0 = 0, anw = 0, atstart = 0;
    uint32_t head = 0, tail = 0;  // ticket counters (positions mod CAP)
    uint32_t xc = 0;              // accumulation cursor: tickets before it are summed
    // lane-private walker state
    bool act = false;
    uint32_t tk = 0, wl = 0, wi = 0, jc = 0;
    float eh = 0.0f;  // Exp(1) variate of the next sojourn
    // G: grid points credited so far, kept as an exact integer-valued double
    // (ceil in fp64, no int conversions on the XU pipe)
    double t = 0.0, S = 0.0, G = 0.0;
    // The gathered slot {j, off | deg_flags, 1/rate | d | v} lives in la..ld,
    // registers that only the gather writes; of the state a walker needs for
    // its *next* jump only the row's offset and degree are kept (off_s,
    // degf_s).  An empty volatile asm with la..ld as in/out operands pins the
    // consumer: nothing that reads them can be scheduled above it.
    unsigned long long la = 0, lb = 0, lc = 0, ld = 0;
    uint32_t off_s = 0, degf_s = 0;
    // per-task accumulators of the oldest task (lane = jumper index mod 32)
    double s1 = 0.0, s2 = 0.0;
    unsigned long long jsum = 0;

    // One sojourn of the lane's walker from its current state: either the
    // path ends (park S', v, jumps in the ticket; lane becomes idle) or the
    // grid points are credited and the walker must jump (`jmp`).
    // (ir, d, vbits, jrow: the state's 1/rate, d, v bits and row id; off_n,
    // degf_n: its offset and degree, kept if the walker goes on)
    auto sojourn = [&](float E, float ir, double d, unsigned long long vbits, uint32_t jrow,
                       uint32_t off_n, uint32_t degf_n, bool& fin, bool& jmp) {  // E ~ Exp(1)
        const float h = __fmul_rn(E, ir);
        const double tn = __dadd_rn(t, __dmul_rn((double)h, p.inv_dt));
        if (tn >= p.n_grid) {
            // park the raw weight sum; the exponent is formed at accumulation
            S = __fma_rn(d, __dsub_rn(p.n_grid1, G), S);
            const uint32_t pos = tk & (CAP - 1);
            CHK(tk - xc < CAP && tail - tk - 1u < CAP);  // in the ring, not yet accumulated
#ifdef EXPMC_CHECKS
            CHK((unsigned long long)__double_as_longlong(q.S[pos]) == kUnfinished);  // parked once
#endif
            q.S[pos] = strang ? __dsub_rn(S, __dmul_rn(0.5, d)) : S;
            q.v[pos] = __longlong_as_double((long long)vbits);
            q.tk[tk_slot(pos)].x = jc;
            // (the landing row id, word 0 of the gathered slot, is not needed
            // by the walk: storing it to the sink slot keeps the word live,
            // so its register is not reused — and waited on — right behind
            // the load)
            q.tk[CAP].y = jrow;
            act = false;
            fin = true;
        } else {
            const double kk = ceil(tn);
            S = __fma_rn(d, __dsub_rn(kk, G), S);
            G = kk;
            t = tn;
            off_s = off_n;
            degf_s = degf_n;
            jmp = true;
        }
    };

    // Next task for this warp: static stride, or (ENTRY_DYNAMIC) the next
    // unclaimed task after the first grid-full.  The result contract does
    // not depend on which warp runs a task.
    auto next_task = [&]() -> uint32_t {
#if ENTRY_DYNAMIC
        uint32_t t = 0;
        if (lane == 0) t = tstride + atomicAdd(task_ctr, 1u);
        return __shfl_sync(FULL, t, 0);
#else
        return anext + tstride;
#endif
    };
    uint32_t anext = atask;
    auto advance_task = [&] {
        anext = atask;
        atask = next_task();
    };

    // Open task `atask` in slot tw: row constants computed by two lanes in
    // parallel (lane 0: e^{-λ}, lane 1: e^{β d}).  Part w of a row owns the
    // walkers [⌊wW/WPR⌋, ⌊(w+1)W/WPR⌋).
    auto open_task = [&] {
        const int sl = (int)(tw & (RT - 1));
        // listed rows, or (rows == nullptr) the contiguous range from p.row0
        const uint32_t i = rows ? rows[atask / WPR] : p.row0 + atask / WPR;
        const RowRec ri = load_rec(rec, i);
        const double lam = __dmul_rn(__ldg(rate + i), p.beta);
        const double ex = exp_det(lane == 0 ? -lam : __dmul_rn(p.beta, ri.d));
        const double e0 = __shfl_sync(FULL, ex, 0), e1 = __shfl_sync(FULL, ex, 1);
        const unsigned long long T0 = (unsigned long long)__dmul_rn(e0, 4294967296.0);
        const uint32_t part = atask % WPR;
        al0 = (uint32_t)(p.W * part / WPR);
        anw = (uint32_t)(p.W * (part + 1) / WPR) - al0;
        const bool dead = (T0 >> 32) != 0 || anw == 0;  // e^{-λ} rounds to 1: never jumps
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
            a.corr = strang ? __dmul_rn(0.5, ri.d) : ri.d;
        }
        if (tf == tw) {  // the new task is the oldest in flight
            ocl = dead;
            oend = tail;
        }
        ++tw;
        apos = 0;
        around = 0;
        atstart = tail;
        if (dead) {
            advance_task();
        } else {
            aopen = true;
        }
        __syncwarp();
    };

    // One gap round of the open task: 128 Exp(1) variates E (4 per lane, in
    // lane-major order) each decide a run of walkers.  E = λK + R with
    // K = ⌊E/λ⌋ ~ Geometric(1 - e^{-λ}) never-jumpers followed by one jumper
    // whose first holding time is R/rate, R ~ Exp(1) truncated to [0, λ) and
    // independent of K (memorylessness) — the law of W independent walkers,
    // at a cost per jumper instead of per walker.  Jumpers within the part
    // become tickets, in walker order.
    auto can_admit = [&] {
        return aopen ? tail + kRound - xc <= CAP : (atask < ntask && tw - tf < (uint32_t)RT);
    };
    auto admit = [&] {
        if (!aopen) {
            open_task();
            return;
        }
        const uint32_t sl = (tw - 1) & (RT - 1);
        const TaskRec& a = q.task[sl];
        CHK(tail + kRound - xc <= CAP && tw - tf >= 1u && tw - tf <= (uint32_t)RT);
        CHK(a.task == atask && a.closed == 0u);
        const float lamf = a.lam, ilam = __uint_as_float(a.rr.spare);
        const U4 D = philox4x32_10(
            U4{0xfffffff0u | (atask % WPR), 32u * around + (uint32_t)lane, a.i, kTagEntry}, p.rk);
        const uint32_t wd[4] = {D.x, D.y, D.z, D.w};
        uint32_t off[4];
        float R[4];
        uint32_t loc = 0;  // walkers decided by this lane's earlier gaps
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float E = neg_ln_u(wd[k]);
            const float kf = fminf(floorf(__fmul_rn(E, ilam)), 134217728.0f);  // 2^27 cap
            R[k] = fmaxf(__fmaf_rn(-lamf, kf, E), 0.0f);
            off[k] = loc + (uint32_t)kf;  // this gap's jumper, lane-relative
            loc = off[k] + 1u;
        }
        // exclusive scan of the lane totals, saturating at 2^31 - 1 (a
        // saturated prefix still exceeds any part, W < 2^29; no u32 wrap)
        uint32_t inc = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc = min(inc + y, 0x7fffffffu);
        }
        const uint32_t exc = inc - loc;  // exact below the cap
        const uint32_t total = __shfl_sync(FULL, inc, 31);
        // jumper positions increase in lane-major order, so the valid ones
        // are a prefix: ticket (lane, k) goes to tail + 4 lane + k
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t P = apos + exc + off[k];  // part-local walker
            const bool ok = P < anw;
            cnt += __popc(__ballot_sync(FULL, ok));
            const uint32_t pos = ok ? ((tail + 4u * lane + k) & (CAP - 1)) : CAP;
            // valid tickets form a prefix in (lane, k) order and stay inside the part
            CHK(!ok || (tail + 4u * lane + k - xc < CAP && al0 + P < (1u << 29)));
            q.tk[tk_slot(pos)] = make_uint2(__float_as_uint(R[k]), (sl << 29) | (al0 + P));
        }
#ifdef EXPMC_CHECKS
        {   // the valid tickets of the round are exactly positions [tail, tail + cnt)
            uint32_t mine = 0;
            for (int k = 0; k < 4; ++k) mine += (apos + exc + off[k] < anw) ? 1u : 0u;
            const uint32_t before = __reduce_add_sync(FULL, mine) - 0u;
            CHK(before == cnt);
            const bool prefix_ok = mine == 4u || (apos + exc + off[mine] >= anw);
            CHK(prefix_ok);
            const uint32_t full_before = __popc(__ballot_sync(FULL, mine == 4u) & lt);
            CHK(mine == 0u || full_before == (uint32_t)lane);  // every earlier lane is full
        }
#endif
        tail += cnt;
        apos = min(apos + total, 0x7fffffffu);
        ++around;
        if (apos >= anw) {  // every walker of the part decided
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
            advance_task();
        }
        __syncwarp();
    };

    uint32_t trip = 0;
    if (atask >= ntask) return;  // a warp without a task
    while (true) {
        // ---- one jump for every walker in flight.  The trip runs jump ->
        // accumulate / finalize -> sojourn -> admit / pop, so the gather issued
        // here is consumed in the same trip, after the accumulation work.  It
        // lands in registers (la..ld) that nothing else writes, and the
        // sojourn reads them in place behind an empty volatile asm that pins
        // the consumer; the only state carried to the next jump is the row's
        // offset and degree.  (With the gather landing in a loop-carried copy
        // of the whole slot, ptxas compacted the slot's dead word away by
        // register moves right behind the load, and every warp waited for its
        // gather *before* the accumulation work: 24.7% of the stall samples,
        // profiles/r02.)  Idle lanes gather too (a stale slot): no predicate
        // on the load or behind it.
        {
            const U4 B = philox4x32_10(U4{jc, wl, wi, kTagEntry}, p.rk);
            const uint32_t off = off_s, degf = degf_s;
            uint32_t k = pick_index(B.y, B.w, WT ? degf & kDegMask : degf);
            if (WT) {
                if (act && (degf & kNonUniform) && B.z >= __ldg(thr + off + k))
                    k = __ldg(alias + off + k);
            }
#ifdef EXPMC_CHECKS
            CHK(WT || (degf & kNonUniform) == 0u);
            CHK(!act || ((degf & kDegMask) != 0u && k < (degf & kDegMask)));
            // every lane gathers (idle lanes a stale but valid slot); p.stats: nnz
            CHK((uint64_t)(uintptr_t)p.stats == 0 ||
                (uint64_t)off + k < (uint64_t)(uintptr_t)p.stats);
#endif
            // (an idle lane's (off_s, degf_s) are those of a row some walker
            // stood on — or (0, 0) at the start — so off + k is a valid slot:
            // no select on the address)
            ld256_gather(adj + (off + k), la, lb, lc, ld);
            // the next holding-time variate, drawn here so that its polynomial
            // runs under the gather's latency instead of after the wait
            eh = neg_ln_u(B.x);
            ++jc;
        }
        // ---- accumulate finished tickets in batches of 32 (lane = ticket -
        // tstart mod 32) and finalize completed tasks, oldest first.  Tickets
        // [xc, xc + rdy) are popped and finished: the oldest ticket still
        // walking (or the first not popped) bounds them.
        // (long walks, GM = 2^k - 1: a look every 2^k trips — a walker takes
        // tens of trips, finished tickets can wait a few more)
        if (GM == 0 || ((++trip) & (uint32_t)GM) == 0u) {
        const uint32_t minoff = __reduce_min_sync(FULL, act ? tk - xc : ~0u);
        uint32_t rdy = head - xc < minoff ? head - xc : minoff;
        // (entry / continuation test: a full batch is ready, or every
        // remaining ticket of the closed oldest task is; it implies tf != tw)
        if (rdy >= 32u || (ocl && rdy >= oend - xc)) {
        __syncwarp();
        do {
            const TaskRec& m = q.task[tf & (RT - 1)];
            // a full batch, or the closed task's last (possibly empty) one
            const uint32_t rem = oend - xc;
            const uint32_t nb = ocl && rdy >= rem && rem < 32u ? rem : 32u;
            CHK(tf != tw && nb <= head - xc && nb <= rdy);
            if ((uint32_t)lane < nb) {
                const uint32_t pos = (xc + lane) & (CAP - 1);
#ifdef EXPMC_CHECKS
                // every ticket of the batch was popped and parked
                CHK((unsigned long long)__double_as_longlong(q.S[pos]) != kUnfinished);
                CHK((q.tk[tk_slot(pos)].y >> 29) == (tf & (RT - 1)));  // ...and is this task's
#endif
                const double x = __dmul_rn(p.dt, __dsub_rn(q.S[pos], m.corr));
                // (p.exp_safe: |x| <= 690 for every walker of this launch)
                const double ex = !kTabShared ? exp_det(x)
                                  : xsafe ? exp_det_inrange(x, s_tab)
                                               : exp_det_tab(x, s_tab, false);
                const double dv = __dsub_rn(__dmul_rn(ex, q.v[pos]), m.K);
                s1 = __dadd_rn(s1, dv);
                s2 = __fma_rn(dv, dv, s2);
                jsum += q.tk[tk_slot(pos)].x;
            }
            xc += nb;
            rdy -= nb;
            if (!ocl || xc != oend) continue;
            // task complete: butterfly, never-jumpers, output
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                s1 = __dadd_rn(s1, __shfl_xor_sync(FULL, s1, o));
                s2 = __dadd_rn(s2, __shfl_xor_sync(FULL, s2, o));
                jsum += __shfl_xor_sync(FULL, jsum, o);
            }
            if (lane == 0) {
                // never-jumpers score f0: deviation f0 - K each (0 when K = f0)
                const double f0 = m.f0, K = m.K;
                const uint32_t n0 = m.n0;
                const double c = __dsub_rn(f0, K);
                if (n0 != 0 && c != 0.0) {
                    s1 = __fma_rn((double)n0, c, s1);
                    s2 = __fma_rn((double)n0, __dmul_rn(c, c), s2);
                }
                // the divisions and sqrt of the estimate run in the
                // row-parallel combine pass, not on one lane here
                CHK(m.task < ntask && m.closed == 1u && m.tend == xc);
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
            // every task finalized: the kernel's exit.  (No task is in flight
            // only right after a finalize — tested here, not every trip: cfg5
            // 41.04 -> 40.68 ms — or from the start, tested before the loop.)
            else if (atask >= ntask) {
                goto finished;
            }
        } while (rdy >= 32u || (ocl && rdy >= oend - xc));
        }
        }
        // ---- sojourn of every walker in flight, at the state just gathered
        bool fin = false, jmp = false;
        if (act) {
            asm volatile("" : "+l"(la), "+l"(lb), "+l"(lc), "+l"(ld));
            sojourn(eh, __uint_as_float((uint32_t)(lb >> 32)), __longlong_as_double((long long)lc),
                    ld, (uint32_t)la, (uint32_t)(la >> 32), (uint32_t)lb, fin, jmp);
        }
        const unsigned idle = __ballot_sync(FULL, !act);
        // scheduler work only when enough lanes are free (batching pops
        // amortises the scheduler over several walkers)
        if (__popc(idle) >= ENTRY_POP_MIN) {
            // ---- admit: sweep chunks while queued tickets cannot feed the
            // idle lanes and a whole chunk's tickets fit in the ring
            while (tail - head < (uint32_t)__popc(idle) && can_admit()) admit();
            // ---- pop: idle lanes take tickets in order
            const uint32_t avail = tail - head;
            const uint32_t nidle = (uint32_t)__popc(idle);
            const uint32_t take = avail < nidle ? avail : nidle;
            // lanes left without tickets (ring or task slots held by work
            // that awaits accumulation): look at the next trip, not the 16th
            if (GM != 0 && avail < nidle) trip = (uint32_t)GM;
            const uint32_t rank = (uint32_t)__popc(idle & lt);
            if (!act && rank < take) {
                tk = head + rank;
                const uint2 t2 = q.tk[tk_slot(tk & (CAP - 1))];
                wl = t2.y & 0x1fffffffu;
                const TaskRec& m = q.task[t2.y >> 29];
                CHK(tk - xc < CAP && tail - tk - 1u < CAP);             // ticket is in the ring
                CHK((((t2.y >> 29) - tf) & (RT - 1)) < tw - tf);        // its task is in flight
#ifdef EXPMC_CHECKS
                q.S[tk & (CAP - 1)] = __longlong_as_double((long long)kUnfinished);
#endif
                const uint4 r0 = *reinterpret_cast<const uint4*>(&m.rr);  // off, degf, ir, -
                wi = m.i;
                t = 0.0; S = 0.0; G = 0.0; jc = 0;
                act = true;
                // a jumper's first sojourn (R < λ) ends in a jump, so it joins
                // the next trip's jump
                sojourn(__uint_as_float(t2.x), __uint_as_float(r0.z), m.rr.d,
                        (unsigned long long)__double_as_longlong(m.rr.v), 0u, r0.x, r0.y, fin, jmp);
            }
            head += take;
#ifdef ENTRY_STATS
            if (lane == 0) {
                atomicAdd(p.stats + 1, (unsigned long long)nidle);
                if (avail < nidle) {  // lanes left idle: why?
                    atomicAdd(p.stats + 2, (unsigned long long)(nidle - avail));
                    if (atask < ntask) atomicAdd(p.stats + 3, 1ull);  // ring full
                }
            }
#endif
        }
#ifdef ENTRY_STATS
        {
            const unsigned jb = __ballot_sync(FULL, jmp);
            const unsigned ab = __ballot_sync(FULL, act);
            if (lane == 0) {
                atomicAdd(p.stats + 0, 1ull);
                atomicAdd(p.stats + 4, (unsigned long long)__popc(jb));
                atomicAdd(p.stats + 5, (unsigned long long)__popc(ab));
            }
        }
#endif
    }
finished:;
}

#include "walk_entry_short.cuh"

// Combine the parts of each row in index order (same tree as the contract:
// part 0, then += part 1, ...) and form the estimate: mean K + Σdev / W,
// SE from the one-pass variance clamped at 0 (finalize, estimator.cpp:76-89).
template <int WPR>
__global__ void combine_parts_kernel(const double4* __restrict__ partial, uint64_t nrows,
                                     uint64_t W, double* __restrict__ out_value,
                                     double* __restrict__ out_se, uint64_t* __restrict__ out_jumps) {
    const uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const double4 a = partial[r * WPR];
    double s1 = a.x, s2 = a.y;
    unsigned long long js = (unsigned long long)__double_as_longlong(a.z);
    const double K = a.w;
#pragma unroll
    for (int k = 1; k < WPR; ++k) {
        const double4 b = partial[r * WPR + k];
        s1 = __dadd_rn(s1, b.x);
        s2 = __dadd_rn(s2, b.y);
        js += (unsigned long long)__double_as_longlong(b.z);
    }
    const double Wd = (double)W;
    out_value[r] = __dadd_rn(K, __ddiv_rn(s1, Wd));
    double se = 0.0;
    if (W > 1) {
        double var = __ddiv_rn(__dsub_rn(s2, __ddiv_rn(__dmul_rn(s1, s1), Wd)), __dsub_rn(Wd, 1.0));
        var = var > 0.0 ? var : 0.0;
        se = sqrt(__ddiv_rn(var, Wd));
    }
    out_se[r] = se;
    out_jumps[r] = js;
}

// Exactly BL resident blocks per SM with the smallest shared-memory carveout
// that holds them, so the rest of the SM's 256 KB is L1 for the edge
// gathers, and no more: padding each block with dynamic shared memory so
// that an extra block cannot fit pins the block count (when the driver
// sized the carveout for a register-limited occupancy above the target,
// config 4 ran 1.8x slower).  One-time configuration per instantiation (a
// function-local static, so concurrent first calls from several host
// threads initialise it once).
struct LaunchCfg {
    int nsm, pad;
};

using EntryKernel = void (*)(const RowRec*, const double*, const Edge*, const uint32_t*,
                             const uint32_t*, const uint32_t*, uint64_t, FastParams, double4*,
                             unsigned int*);

template <EntryKernel KERN, int BL>
const LaunchCfg& launch_cfg(const char* name) {
    static const LaunchCfg lc = [name] {
        int nsm = 0, pad = 0;
        int dev = 0, smem_sm = 0;
        cudaFuncAttributes fa;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            nsm = 148;
        int pct = -1;
        if (ENTRY_CARVE && cudaFuncGetAttributes(&fa, KERN) == cudaSuccess &&
            cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) ==
                cudaSuccess &&
            smem_sm > 0) {
            constexpr int kReserve = 1024;
            const long st = (long)fa.sharedSizeBytes;
            const int kb[] = {0, 8, 16, 32, 64, 100, 132, 164, 196, 228};
            long cap = smem_sm;
            for (int c : kb)
                if (c * 1024L >= BL * (st + kReserve) && c * 1024L <= smem_sm) {
                    cap = c * 1024L;
                    break;
                }
            const long tmin = smem_sm / (BL + 1) - kReserve + 1;  // BL+1 blocks must not fit
            const long tmax = cap / BL - kReserve;                 // BL blocks must fit in cap
            if (tmin <= tmax) pad = (int)(tmin > st ? tmin - st : 0);
            if (pad) cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
            // the driver rounds the percentage UP to a supported capacity
            pct = (int)floor(100.0 * cap / smem_sm);
            cudaFuncSetAttribute(KERN, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
        }
        int resident = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, KERN, 128, pad);
        cudaGetLastError();
        if (getenv("EXPMC_DEBUG"))
            fprintf(stderr,
                    "%s<BL=%d>: %d SMs, occupancy %d blocks/SM, pad %d B, carveout %d%%\n", name,
                    BL, nsm, resident, pad, pct);
        return LaunchCfg{nsm, pad};
    }();
    return lc;
}

template <int WPR, EntryKernel KERN, int BL>
int launch_t(const char* name, const DevSplit& m, const uint32_t* rows, uint64_t nrows,
             const FastParams& p, double* value, double* se, uint64_t* jumps, double4* partial,
             cudaStream_t s) {
    // Grid = one wave of resident blocks (the kernel strides over tasks).
    const LaunchCfg& lc = launch_cfg<KERN, BL>(name);
    const int nsm = lc.nsm, pad = lc.pad;
    const uint64_t warps = nrows * WPR;
    const uint64_t blocks = (warps + 3) / 4;
    const uint64_t cap = (uint64_t)nsm * BL;
    const unsigned grid = (unsigned)(blocks < cap ? blocks : cap);
    unsigned int* ctr = reinterpret_cast<unsigned int*>(partial + warps);
#if ENTRY_DYNAMIC
    cudaMemsetAsync(ctr, 0, sizeof(unsigned int), s);
#endif
#ifdef EXPMC_CHECKS
    FastParams pc = p;  // checks build: the gather bound (nnz) travels in the unused stats slot
    pc.stats = reinterpret_cast<unsigned long long*>((uintptr_t)m.nnz);
    KERN<<<grid, 128, pad, s>>>(m.rec, m.rate, m.adj, m.alias_thr, m.alias_idx, rows, nrows, pc,
                                partial, ctr);
#else
    KERN<<<grid, 128, pad, s>>>(m.rec, m.rate, m.adj, m.alias_thr, m.alias_idx, rows, nrows, p,
                                partial, ctr);
#endif
    combine_parts_kernel<WPR><<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(
        partial, nrows, p.W, value, se, jumps);
    return 2;
}

// Launch shapes; none changes a result bit.  With the gathers marked
// L1::no_allocate (common.cuh ld256_gather) the 8-block shape is the fastest
// on every configuration (config 4: 2.72 s, against 2.79 s at 7 blocks), so
// it is the only production shape.  EXPMC_ENTRY_SHAPE (A/B and tests only):
// 0 = entry_walk_kernel, 8 blocks/SM (32 warps); 1 = 7 blocks (28 warps, 60 KB
// of L1 — needed for long walks before the no-allocate gathers: 2.81 s vs
// 4.59 s on config 4); 3 = the pipelined two-set entry_pipe_kernel
// (walk_entry_short.cuh: bit-identical results, measured slower).
// Measured, profiles/r02/README.md.
// The production shape (8 blocks/SM).  An unweighted matrix whose exponents
// are in range for this launch — every configuration of the benchmark — runs
// the instantiation with the splitting, the range flag and "no weighted row"
// fixed at compile time (config 5: 39.29 -> 38.67 ms against the run-time
// tests); anything else the general one.
template <int WPR, int GM>
int launch_shape0(const DevSplit& m, const uint32_t* rows, uint64_t nrows, const FastParams& p,
                  double* value, double* se, uint64_t* jumps, double4* partial, cudaStream_t s) {
    if (!m.any_nonuniform && p.exp_safe) {
        if (p.strang)
            return launch_t<WPR, entry_walk_kernel<WPR, 8, GM, false, 1, true>, 8>(
                "entry_walk_kernel", m, rows, nrows, p, value, se, jumps, partial, s);
        return launch_t<WPR, entry_walk_kernel<WPR, 8, GM, false, 0, true>, 8>(
            "entry_walk_kernel", m, rows, nrows, p, value, se, jumps, partial, s);
    }
    return launch_t<WPR, entry_walk_kernel<WPR, 8, GM>, 8>("entry_walk_kernel", m, rows, nrows, p,
                                                           value, se, jumps, partial, s);
}

template <int WPR>
int launch_w(const DevSplit& m, const uint32_t* rows, uint64_t nrows, const FastParams& p,
             double* value, double* se, uint64_t* jumps, double4* partial, cudaStream_t s) {
    int shape = 0;
    if (const char* e = getenv("EXPMC_ENTRY_SHAPE")) shape = atoi(e);  // A/B and tests only
    switch (shape) {
        case 3:
            return launch_t<WPR, entry_pipe_kernel<WPR, EPIPE_BL>, EPIPE_BL>(
                "entry_pipe_kernel", m, rows, nrows, p, value, se, jumps, partial, s);
        case 0:
            // long walks (>= ENTRY_LONG_WALK jumps of a walker started at a
            // random row): ready-ticket look every 16th trip
            // (and enough walkers per task that task slots do not wait on
            // the look: measured 8-20% slower at 16-64 walkers per entry)
            if (p.beta * m.mean_rate >= ENTRY_LONG_WALK && p.W / WPR >= 512)
                return launch_shape0<WPR, ENTRY_GATE_MASK>(m, rows, nrows, p, value, se, jumps,
                                                           partial, s);
            return launch_shape0<WPR, 0>(m, rows, nrows, p, value, se, jumps, partial, s);
#ifdef EXPMC_EXPERIMENTS
        case 5:
            return launch_t<WPR, entry_walk_kernel<WPR, 5>, 5>("entry_walk_kernel", m, rows, nrows,
                                                               p, value, se, jumps, partial, s);
        case 6:
            return launch_t<WPR, entry_walk_kernel<WPR, 6>, 6>("entry_walk_kernel", m, rows, nrows,
                                                               p, value, se, jumps, partial, s);
#endif
        default:
            return launch_t<WPR, entry_walk_kernel<WPR, 7>, 7>("entry_walk_kernel", m, rows, nrows,
                                                               p, value, se, jumps, partial, s);
    }
}

}  // namespace

// Warps (parts) per row: a function of W only (part of the result contract).
int entry_fast_wpr(uint64_t W) {
    const uint64_t nch = (W + kRound - 1) / kRound;
    return nch >= 64 ? 4 : (nch >= 32 ? 2 : 1);
}

size_t entry_fast_scratch_bytes(uint64_t nrows, uint64_t W) {
    // per-task partials, then the task counter (ENTRY_DYNAMIC)
    return nrows * (size_t)entry_fast_wpr(W) * sizeof(double4) + 256;
}

int launch_entry_fast(const DevSplit& m, const uint32_t* rows, uint64_t nrows,
                      const FastParams& p_in, double* value, double* se, uint64_t* jumps,
                      void* scratch, cudaStream_t s) {
    if (nrows == 0) return 0;
    // Every exponent a walker forms is Δt (S - corr) with |S| <= (N + 1) max|d|
    // and |corr| <= max|d|: inside ±690 when β max|d| (N + 2) / N is.
    FastParams p = p_in;
    p.exp_safe = ENTRY_EXP_INRANGE &&
                 p.beta * m.dabs_max * ((double)p.N + 2.0) / (double)p.N < 690.0;
    double4* part = static_cast<double4*>(scratch);
#ifdef ENTRY_STATS
    static unsigned long long* st = nullptr;
    if (!st) cudaMallocManaged(&st, 64);
    cudaStreamSynchronize(s);
    for (int z = 0; z < 8; ++z) st[z] = 0;
    FastParams ps = p;
    ps.stats = st;
#define p ps
#endif
    int k;
    switch (entry_fast_wpr(p.W)) {
        case 4: k = launch_w<4>(m, rows, nrows, p, value, se, jumps, part, s); break;
        case 2: k = launch_w<2>(m, rows, nrows, p, value, se, jumps, part, s); break;
        default: k = launch_w<1>(m, rows, nrows, p, value, se, jumps, part, s); break;
    }
#ifdef ENTRY_STATS
#undef p
    cudaStreamSynchronize(s);
    fprintf(stderr,
            "ENTRY_STATS iters %llu idle@pop %.2f left_idle %.2f ring_full_iters %.3f "
            "jump_lanes %.2f active %.2f\n",
            st[0], (double)st[1] / st[0], (double)st[2] / st[0], (double)st[3] / st[0],
            (double)st[4] / st[0], (double)st[5] / st[0]);
#endif
    return k;
}

}  // namespace expmc_b200
