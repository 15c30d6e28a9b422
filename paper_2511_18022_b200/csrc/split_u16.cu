// split_u16.cu -- a5 (+ a3/a4 fused, a6 partials): the masked min-plus layer sweep of
// Eq. (3) with TWO scenarios per lane in packed 16-bit halves, fed by TMA.
//
// Same DP as split.cu (the separable route cost, g(i) = min_{p in window(i)} g(p) + Cg[i],
// f(n) = min g + B[n]), but every 32-bit register holds the pair {scenario 2l, scenario 2l+1}
// of lane l:
//
//  * loads: P = the tour-order prefix of the pair, one u16 per half (P <= 0x7FFF - Q for every
//    feasible scenario, kept there by a periodic rebase), so one 32-bit add updates both halves
//    with no carry between them.  A demand above Q (an infeasible scenario, DESIGN R4) can
//    carry out of the LOW half into the high one: such a pair's high scenario is recomputed by
//    split_finish_kernel (qmax, the largest raw demand of each half, tells).
//  * ring entry of split point p: Y = P(p) + Q + 0x8000 per half (a guard bit), G = g(p) -
//    base, 15 bits.  Candidate p of layer i (p in the window iff
//    P(i) - P(p) <= Q  <=>  Y >= P(i) + 0x8000):  d = Y - P(i) (one 32-bit IMAD on the FMA pipe:
//    no borrow, every half of Y is >= 0x7FFF >= P(i)) has bit 15 of a half set iff p is in that
//    scenario's window, and  key = G | (~d & 0x80008000)  (one LOP3) is G inside the window and
//    >= 0x8000 > every in-window G outside it.  Keys fold by 3-input u16x2 mins (VIMNMX3.U16x2).
//    Per candidate pair: IMAD (FMA pipe) + LOP3 + half a VIMNMX3 (ALU pipe), for 2 scenarios.
//  * values: g relative to a per-scenario int32 base.  g never falls more than NS below the
//    window minimum m(i) (NS = the tour's sum of negative Cg; m(i+1) >= min(m(i), g(i)) because
//    the window's left edge only moves right, DESIGN R5), so with base <= m - NS every value the
//    sweep forms is >= 0; every kU16Check layers a warp vote checks g and P against
//    TourInfo::thr16 / the load limit and, when needed, rebases both (subtract, saturating at
//    0 for values that are provably never in a window again).  tour_prep_kernel checks per
//    tour that values stay below 2^15 between checks (TourInfo::ok16); lanes of a tour that
//    fails it are deferred to split_finish_kernel, like ring overflows.
//  * the chain: g(i) = min(keys of age >= 2, g(i-1)) + Cg[i], the add as one 32-bit add of
//    the pair Cg * 0x10001 (no carry: both halves stay in [0, 0x7FFF]).
//  * LS = 4 layers per step: the candidates of age >= l + 1 of layer j + l (l = 0 .. 3) are split
//    points <= j, known before the step starts, so the four layers' unconditional groups run back
//    to back and ONE warp vote per deeper group of ages guards all four layers (the vote, its
//    branch and the branch-target fetch are paid once per 4 layers); the split points j + 1 ..
//    j + 3 made inside the step enter last, as keys whose window tests (loads only) were ready
//    early.  Measured (C2, 10^6 scenarios): two layers per step 84.0 us, four 79.8 us.
//
// Work decomposition (warp specialisation): a single wave of persistent CTAs of kU16Cons = 4
// consumer warps + 1 producer warp.  A tile is 256 scenarios (64 per consumer warp) of one tour;
// the producer of CTA k starts on tile k, takes later tiles from a global counter and fills an
// NS-stage shared-memory ring: per chunk of W layers, the chunk's W demand rows in W/4 16-byte
// loads of the tour's padded row table (one round trip), W/4 TMA gathers (cp.async.bulk.tensor.2d...tile::gather4: 4 tour-ordered
// demand rows x 256 scenarios, 512 B each, in one instruction; rows past n are outside the tensor
// and arrive as zeros) plus one bulk copy of the chunk's W Cg pairs, completing on the stage's
// "full" mbarrier; the consumers release the stage by arriving on its named hardware barrier
// (tma.cuh stage_release; the producer waits there in bar.sync, parked without polling), so a
// fast warp runs up to NS - 1 chunks ahead of the slowest.  The consumers carry no copy code:
// per chunk they wait on one barrier and arrive on another.
#include <climits>
#include <cstring>

#include "common.cuh"
#include "split_ws.cuh"
#include "tma.cuh"

namespace spdp {

#ifndef SPDP_U16_CONS
#define SPDP_U16_CONS 4
#define SPDP_U16_CONS_PER_BOX 4
#endif
constexpr int kU16Cons = SPDP_U16_CONS;           // consumer warps per CTA, one tile of NP * 64 kU16Cons scenarios
constexpr int kU16Threads = 32 * (kU16Cons + 1);  // + 1 producer warp
constexpr int kU16ConsPerBox = SPDP_U16_CONS_PER_BOX;  // consumer warps per TMA box
constexpr int kU16Box = kU16ConsPerBox * 64;           // columns of one TMA box (256 scenarios, 512 B per row)
constexpr int kU16BoxesPerTile = kU16Cons / kU16ConsPerBox;
static_assert(kU16Cons % kU16ConsPerBox == 0 && kU16Box <= 256, "TMA box: at most 256 columns");
constexpr uint32_t kGuard = 0x80008000u;

// Debug timeline (spdp_debug_timeline): when set, lane 0 of every consumer warp appends one record
// per tile {sm << 16 | warp slot, tile id, start ns, end ns} (global timer) after a u64 counter.
__device__ unsigned long long* g_timeline = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
// one record {sm << 16 | warp slot, tile (or 0xfffffff0 CTA start / 0xfffffff1 warp done), t0, now}
__device__ __forceinline__ void tl_record(unsigned slot, unsigned tile, unsigned long long t0) {
    const unsigned long long k = atomicAdd(g_timeline, 1ull);
    unsigned long long* r = g_timeline + 2 + 4 * k;
    r[0] = ((unsigned long long)smid() << 16) | slot;
    r[1] = tile;
    r[2] = t0;
    r[3] = gtimer();
}
static bool g_tl_on = false;  // host: a timeline buffer is set (launch the TL instantiation)

// NP = scenario pairs per lane (64 NP scenarios per consumer warp, NP TMA boxes per row and tile;
// shared memory per stage: [NP boxes][W rows][256 scenarios] u16, then the W Cg pairs, the header)
template <int W, int NP, int NST>
struct U16Cfg {
    static constexpr int NS = NST;                                          // stages
    static constexpr int kMaxReg = NP == 1 ? (W <= 24 ? 96 : 128) : 128;    // registers: 4 / 3 CTAs per SM
    static constexpr int kTile = NP * kU16Cons * 64;                       // scenarios per tile
    static constexpr int kWarp = NP * 64;                                   // scenarios per consumer warp
    static constexpr int kRowBytes = kU16Box * (int)sizeof(uint16_t);      // 512 B (one box row)
    static constexpr int kBoxBytes = W * kRowBytes;                         // W rows of one box
    static constexpr int kBoxes = NP * kU16BoxesPerTile;                   // boxes per tile
    static constexpr int kRowsBytes = kBoxes * kBoxBytes;                   // all boxes
    static constexpr int kCgOff = kRowsBytes;                               // W Cg pairs
    static constexpr int kHdrOff = kRowsBytes + W * (int)sizeof(int32_t);   // {tour, block, chunk, 0}
    static constexpr int kStageBytes = (kHdrOff + 16 + 127) / 128 * 128;    // (TMA: 128-B aligned)
    static constexpr int kStagesBytes = NS * kStageBytes;
    static constexpr size_t kSmem = (size_t)kStagesBytes + 2 * NS * sizeof(uint64_t);  // + barriers
    static_assert(W % 4 == 0 && (W * 4) % 16 == 0, "W must be a multiple of 4");
};

// Per-half constants, formed on the host (kernel parameters: uniform registers, so each use is
// one operand, not a re-materialised expression).  Host check: (kU16Check + 2)(Q + 1) <= 0x8000.
struct U16Consts {
    uint32_t m1;    // 0xffffffff (the IMAD multiplier)
    uint32_t one;   // 1 (the IMAD multiplier of an add that should issue on the FMA pipe)
    uint32_t qgp;   // (Q + 0x8000) per half: Y = P + Q + guard
    uint32_t nq1p;  // -(Q + 1) per half (16-bit two's complement)
    uint32_t padd;  // (0x7fff - pthr) per half, pthr = 0x7fff - Q - kU16Check (Q + 1): bit 15 of P + padd
                    // is set iff P > pthr (a load rebase is due)
};

// key = G | (~d & 0x80008000) as one LOP3 (an explicit lop3, so ptxas cannot split it around
// the vote branch that tests d)
__device__ __forceinline__ uint32_t key_of(uint32_t G, uint32_t d) {
    uint32_t k;
    asm("lop3.b32 %0, %1, %2, %3, 0xF2;" : "=r"(k) : "r"(G), "r"(d), "r"(kGuard));
    return k;
}

// g[r] for a warp-uniform runtime r < W, as a switch (an indexed branch, not W compare-selects)
template <int W>
__device__ __forceinline__ uint32_t ring_slot(const uint32_t (&g)[W], const int r) {
    switch (r) {
#define SPDP_RING_CASE(i) \
    case i:               \
        if constexpr (i < W) return g[i]; \
        break;
        SPDP_RING_CASE(0) SPDP_RING_CASE(1) SPDP_RING_CASE(2) SPDP_RING_CASE(3) SPDP_RING_CASE(4) SPDP_RING_CASE(5)
        SPDP_RING_CASE(6) SPDP_RING_CASE(7) SPDP_RING_CASE(8) SPDP_RING_CASE(9) SPDP_RING_CASE(10) SPDP_RING_CASE(11)
        SPDP_RING_CASE(12) SPDP_RING_CASE(13) SPDP_RING_CASE(14) SPDP_RING_CASE(15) SPDP_RING_CASE(16)
        SPDP_RING_CASE(17) SPDP_RING_CASE(18) SPDP_RING_CASE(19) SPDP_RING_CASE(20) SPDP_RING_CASE(21)
        SPDP_RING_CASE(22) SPDP_RING_CASE(23) SPDP_RING_CASE(24) SPDP_RING_CASE(25) SPDP_RING_CASE(26)
        SPDP_RING_CASE(27) SPDP_RING_CASE(28) SPDP_RING_CASE(29) SPDP_RING_CASE(30) SPDP_RING_CASE(31)
#undef SPDP_RING_CASE
        default: break;
    }
    return 0u;
}

// Minimum of N packed u16 pairs with ceil((N - 1) / 2) 3-input mins (VIMNMX3.U16x2).
template <int N>
__device__ __forceinline__ uint32_t umin_tree(const uint32_t* v) {
    if constexpr (N == 1) return v[0];
    else if constexpr (N == 2) return __vminu2(v[0], v[1]);
    else if constexpr (N == 3) return __vimin3_u16x2(v[0], v[1], v[2]);
    else if constexpr (N == 4) return __vimin3_u16x2(__vminu2(v[0], v[1]), v[2], v[3]);
    else return __vimin3_u16x2(umin_tree<N - 2>(v), v[N - 2], v[N - 1]);
}

// Minimum of v[lo .. N - 1] (lo a compile-time constant after unrolling).
template <int N>
__device__ __forceinline__ uint32_t umin_tree_from(const uint32_t* v, const int lo) {
    if (lo == 0) return umin_tree<N>(v);
    if constexpr (N > 1) return umin_tree_from<N - 1>(v + 1, lo - 1);
    return v[0];
}

// A0: ages scanned unconditionally (age 1 + A0 - 1 masked candidates); then groups of UG ages,
// each behind a warp vote on its youngest age; the scan of age W also tests for ring overflow.
// NP: scenario pairs per lane (independent DP chains; one vote and one range check serve all).
// TL: the debug-timeline instantiation (spdp_debug_timeline; never the production launch).
template <int W, int A0, int UG, int NP, int NST, int LS, bool TL = false>
__global__ void __launch_bounds__(kU16Threads) __maxnreg__((U16Cfg<W, NP, NST>::kMaxReg))
    split_sweep_u16_kernel(const __grid_constant__ CUtensorMap dmap, const int32_t* __restrict__ tours,
                           const int32_t* __restrict__ trows,
                           const int32_t* __restrict__ cgs, const int32_t* __restrict__ g0s,
                           const TourInfo* __restrict__ tinfo, int n, int T, int64_t S, uint32_t Q, U16Consts kc,
                           int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ slots,
                           unsigned long long* __restrict__ ovf_list, unsigned* __restrict__ hdr) {
    using Cfg = U16Cfg<W, NP, NST>;
    constexpr int NS = Cfg::NS;
    static_assert(A0 >= 2 && A0 <= W && UG >= 1 && NP >= 1 && (LS == 2 || LS == 4) && W % LS == 0 && kU16Check % LS == 0 && A0 >= LS + 1, "bad u16 sweep config");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + Cfg::kStagesBytes);  // [NS]: data landed
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t ntile_s = (uint32_t)((S + Cfg::kTile - 1) / Cfg::kTile);
    const uint32_t ntiles = ntile_s * (uint32_t)T;
    const int nchunks = (n + W - 1) / W;
    const int cgs_stride = cg_stride(n);
    if (tid == 0) {
        for (int k = 0; k < NS; ++k) {
            mbar_init(&full[k], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if constexpr (TL) {
        if (tid == 0) tl_record(blockIdx.x * kU16Cons, 0xfffffff0u, gtimer());  // CTA start
    }
    // (the dependent launch of split_finish_kernel is triggered by each producer once every tile is
    // claimed -- its CTAs then land on SMs the ramp-down frees: -0.6 us per C2 step, 3 interleaved
    // runs; a trigger at kernel start kept them resident through the whole sweep: +0.4 us)
    // (tables, counters and partial slots come from tour_prep_kernel: every role waits for it with
    // pdl_wait() before its first read of them; the demand matrix and the tours are inputs, complete
    // before tour_prep_kernel -- a plain launch -- started)

    // (a vote, not a plain branch on wid: the compiler then knows each role runs whole warps, and the
    // consumers' warp votes need no divergence checks, BRA.DIV)
    if (__any_sync(kFull, wid == kU16Cons)) {
        // ---------------- producer: one lane fills the stages in order -----------------------------
        // per chunk: NP W/4 gathers of 4 tour-ordered rows x 256 scenarios (box h of the tile), one
        // bulk copy of the W Cg pairs, the header; completion on the stage's full barrier.  The
        // whole warp runs the loop (lane 0 issues): no lane exits early, so the compiler keeps every
        // warp of the kernel provably converged.
        // the first tile of CTA k is tile k; later tiles come from the counter (starting at gridDim.x)
        int t = -1, b = 0, c = nchunks, st = 0;
        unsigned r = 0u, id = blockIdx.x;
        const int4* trow = nullptr;
        // Before the wait for tour_prep_kernel (it triggers this launch at its start): the first tile's
        // first min(NS, nchunks) chunks of demand rows, with the rows read from the tour itself (the
        // same clamp as the prep's row table), so the first data is in flight while the prep runs;
        // their Cg copies follow the wait (the stage's barrier expects both).
        int pre = 0;
        if (id < ntiles) {
            t = (int)(id / ntile_s);
            b = (int)lpt_block(id - (uint32_t)t * ntile_s, ntile_s, Cfg::kTile);
            pre = nchunks < NS ? nchunks : NS;
            // lane j loads the tour entries of rows k W + j of the pre chunks (one round trip for all)
            const int32_t* tr = tours + (int64_t)t * n;
            int myrow[NS];
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                const int i = k * W + lane;
                const int cst = (lane < W && k < pre && i < n) ? __ldg(tr + i) : 1;
                myrow[k] = i < n ? (cst < 1 ? 0 : (cst > n ? n - 1 : cst - 1)) : n;
            }
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                if (k >= pre) break;
                unsigned char* sb = smem_raw + (size_t)k * Cfg::kStageBytes;
                if (lane == 0) {
                    *reinterpret_cast<int4*>(sb + Cfg::kHdrOff) = make_int4(t, b, k, 0);
                    mbar_arrive_expect_tx(&full[k], (uint32_t)(Cfg::kRowsBytes + W * 4));
                }
#pragma unroll
                for (int g = 0; g < W / 4; ++g) {
                    const int r0 = __shfl_sync(kFull, myrow[k], 4 * g), r1 = __shfl_sync(kFull, myrow[k], 4 * g + 1);
                    const int r2 = __shfl_sync(kFull, myrow[k], 4 * g + 2), r3 = __shfl_sync(kFull, myrow[k], 4 * g + 3);
                    if (lane == 0)
#pragma unroll
                        for (int h = 0; h < Cfg::kBoxes; ++h)
                            tma_gather4(sb + h * Cfg::kBoxBytes + g * 4 * Cfg::kRowBytes, &dmap, b * Cfg::kTile + h * kU16Box,
                                        r0, r1, r2, r3, &full[k]);
                }
            }
            __syncwarp();
        }
        pdl_wait();
        if (pre > 0) {
            if (lane == 0)
                for (int k = 0; k < pre; ++k)
                    bulk_g2s_plain(smem_raw + (size_t)k * Cfg::kStageBytes + Cfg::kCgOff,
                                   cgs + (int64_t)t * kCgPlanes * cgs_stride + 2 * cgs_stride + k * W, W * 4, &full[k]);
            __syncwarp();
            trow = reinterpret_cast<const int4*>(trows + (int64_t)t * trow_stride(n));
            c = pre;
            st = pre % NS;
            r = (unsigned)(pre / NS);
        }
        for (;;) {
            if (r > 0) stage_acquire(st, 32 * (kU16Cons + 1));  // the consumers released the previous use (round r - 1)
            if (c == nchunks) {                           // the next tile
                if (t >= 0) {
                    if (lane == 0) id = atomicAdd(hdr + HDR_TILE, 1u) + gridDim.x;
                    id = __shfl_sync(kFull, id, 0);
                }
                t = id < ntiles ? (int)(id / ntile_s) : -1;
                b = id < ntiles ? (int)lpt_block(id - (uint32_t)t * ntile_s, ntile_s, Cfg::kTile) : 0;
                trow = reinterpret_cast<const int4*>(trows + (int64_t)(t < 0 ? 0 : t) * trow_stride(n));
                c = 0;
            }
            unsigned char* sb = smem_raw + (size_t)st * Cfg::kStageBytes;
            uint64_t* fb = &full[st];
            if (lane == 0) *reinterpret_cast<int4*>(sb + Cfg::kHdrOff) = make_int4(t, b, c, 0);
            if (__any_sync(kFull, t < 0)) {  // no tiles left: an arrival without data tells the consumers to stop
                if (lane == 0) mbar_arrive(fb);
                pdl_trigger();  // (every tile is claimed: split_finish_kernel may start launching)
                break;
            }
            if (lane == 0) {
                const int r0 = c * W;
                // the chunk's W rows, 4 per load (past n: row n, outside the tensor, reads as zeros)
                int4 rq[W / 4];
#pragma unroll
                for (int g = 0; g < W / 4; ++g) rq[g] = __ldg(trow + r0 / 4 + g);
                mbar_arrive_expect_tx(fb, (uint32_t)(Cfg::kRowsBytes + W * 4));
#pragma unroll
                for (int g = 0; g < W / 4; ++g)
#pragma unroll
                    for (int h = 0; h < Cfg::kBoxes; ++h)
                        tma_gather4(sb + h * Cfg::kBoxBytes + g * 4 * Cfg::kRowBytes, &dmap, b * Cfg::kTile + h * kU16Box,
                                    rq[g].x, rq[g].y, rq[g].z, rq[g].w, fb);
                bulk_g2s_plain(sb + Cfg::kCgOff, cgs + (int64_t)t * kCgPlanes * cgs_stride + 2 * cgs_stride + r0, W * 4,
                               fb);
            }
            __syncwarp();
            ++c;
            if (++st == NS) {
                st = 0;
                ++r;
            }
        }
    } else {
    // ---------------- consumer warp wid ---------------------------------------------------------
    __syncwarp();
    pdl_wait();
    const int slot = (blockIdx.x * kU16Cons + wid) % kSlots;
    unsigned* ovf_count = hdr + HDR_OVF_COUNT;
    const int rem = n % W;
    const uint32_t m1 = kc.m1, one = kc.one, QGP = kc.qgp, nQ1P = kc.nq1p, PADD = kc.padd;
    // pair k of lane l: scenarios 64 (NP wid + k) + 2 l + {0, 1} of the tile, i.e. box (NP wid + k) / 4,
    // columns 64 ((NP wid + k) % 4) + 2 l + {0, 1}
    int boff[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const int q = NP * wid + k;
        boff[k] = (q / kU16ConsPerBox) * Cfg::kBoxBytes + (q % kU16ConsPerBox) * 128 + 4 * lane;
    }

    uint32_t G[NP][W], Y[NP][W];
#pragma unroll
    for (int k = 0; k < NP; ++k)
#pragma unroll
        for (int a = 0; a < W; ++a) G[k][a] = 0u;

    struct LanePart {
        int nf, ni;
        long long sum, sqlo, sqhi;
    };
    __shared__ LanePart accs[kU16Cons * 32];
    LanePart* accp = &accs[tid];
    *accp = LanePart{0, 0, 0, 0, 0};
    int acc_t = -1;
    auto flush = [&]() {
        const LanePart a = *accp;
        const Part p = warp_sum(Part{a.nf, a.ni, a.sum, a.sqlo, a.sqhi});
        *accp = LanePart{0, 0, 0, 0, 0};
        if (lane == 0 && acc_t >= 0) {
            spdp_saa_partial* d = &slots[(int64_t)acc_t * kSlots + slot];
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_feas), (unsigned long long)p.n_feas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_infeas), (unsigned long long)p.n_infeas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sum), (unsigned long long)p.sum);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sumsq_lo), (unsigned long long)p.sq_lo);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sumsq_hi), (unsigned long long)p.sq_hi);
        }
    };

    // constants of tour acc_t, in shared memory (used a few times per chunk; registers are the ring's)
    struct TourConsts {
        uint32_t nsP, nNSP, GADD;  // NS, -NS per half; bit 15 of g + GADD set iff g > thr16
        int32_t base0, bn, ok;     // g = G + base, g(0) = NS + base0; B[n]; TourInfo::ok16
    };
    __shared__ TourConsts tcs[kU16Cons];
    TourConsts* tc = &tcs[wid];
    int cs = 0;         // stage
    unsigned cr = 0u;   // round (parity of the full barrier's phase)
    for (;;) {
        unsigned char* sb = smem_raw + (size_t)cs * Cfg::kStageBytes;
        mbar_wait_warp(&full[cs], cr & 1u);
        const int4 th = *reinterpret_cast<const int4*>(sb + Cfg::kHdrOff);
        if (__all_sync(kFull, th.x < 0)) break;  // (a vote: keeps the warp provably converged)
        const int t = th.x;
        const int64_t s0 = (int64_t)th.y * Cfg::kTile + wid * Cfg::kWarp;  // this warp's 64 NP scenarios
        unsigned long long tl0 = 0ull;
        if constexpr (TL) tl0 = gtimer();
        if (__any_sync(kFull, t != acc_t)) {  // a new tour: flush its predecessor's SAA sums, load its constants
            if (slots) flush();
            acc_t = t;
            const TourInfo ti = tinfo[t];
            const uint32_t ns = (uint32_t)ti.ns16;
            if (lane == 0)
                *tc = TourConsts{ns * 0x10001u, ((0x10000u - ns) & 0xffffu) * 0x10001u,
                                 (0x7fffu - (uint32_t)ti.thr16) * 0x10001u, g0s[t] - (int32_t)ns, ti.bn, ti.ok16};
            __syncwarp();
        }
        int32_t blo[NP], bhi[NP];
        uint32_t P[NP], gprev[NP], qmax[NP], ovfb[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            blo[k] = bhi[k] = tc->base0;
#pragma unroll
            for (int a = 0; a < W; ++a) Y[k][a] = 0x7fff7fffu;  // no window ever reaches an empty slot
            P[k] = 0u;
            gprev[k] = tc->nsP;
            qmax[k] = 0u;
            ovfb[k] = 0u;
        }

        for (int c = 0;;) {
            const uint32_t* cgc = reinterpret_cast<const uint32_t*>(sb + Cfg::kCgOff);
            const bool pad_chunk = (c + 1) * W > n;  // rows past n (zero demand): no overflow test there
            // the key of the candidate of age a (>= 2) at layer jj of pair k: G inside the window, >= 0x8000
            // outside; d (bit 15 of a half set iff inside) is returned for the votes
            auto cand = [&](const int k, const int jj, const uint32_t Pn, const int a, uint32_t& d) -> uint32_t {
                const int s = (jj - a + 1 + 2 * W) % W;
                d = imad_u32(Pn, m1, Y[k][s]);
                return key_of(G[k][s], d);
            };
            // the window of layer jj reaches the oldest ring age W: the ring may miss older candidates
            auto overflow = [&](const int k, const int jj, const uint32_t d) {
                if (!pad_chunk || c * W + jj < n) ovfb[k] |= d & kGuard;
            };
            // the unconditional ages lo..A0 of layer jj, folded (lo >= 2)
            auto first_group = [&](const int k, const int jj, const uint32_t Pn, const int lo) -> uint32_t {
                uint32_t key[A0 - 1];
#pragma unroll
                for (int a = 2; a <= A0; ++a) {
                    if (a < lo) {
                        key[a - 2] = 0xffffffffu;
                        continue;
                    }
                    uint32_t d;
                    key[a - 2] = cand(k, jj, Pn, a, d);
                    if (a == W) overflow(k, jj, d);
                }
                return umin_tree_from<A0 - 1>(key, lo - 2);
            };
            // the keys of a group (ages a0 + 1 .. a0 + UG - 1; age a0's key k0 done by the caller) folded into a
            auto group_rest = [&](const int k, const int jj, const uint32_t Pn, const int a0, uint32_t a,
                                  const uint32_t k0) {
                uint32_t key[UG + 1];
                key[0] = a;
                key[1] = k0;
#pragma unroll
                for (int u = 1; u < UG; ++u) {
                    if (a0 + u <= W) {
                        uint32_t d;
                        key[u + 1] = cand(k, jj, Pn, a0 + u, d);
                        if (a0 + u == W) overflow(k, jj, d);
                    } else {
                        key[u + 1] = 0xffffffffu;
                    }
                }
                return umin_tree<UG + 1>(key);
            };
            // every kU16Check layers: rebase values and loads if either approaches 2^15 (see the header);
            // one vote for all pairs (a rebase is valid at any layer, so pairs that do not need one may take it)
            auto range_check = [&](const uint32_t* gm) {
                uint32_t tv = 0u;
#pragma unroll
                for (int k = 0; k < NP; ++k) tv |= (gprev[k] + tc->GADD) | (P[k] + PADD);
                if (__any_sync(kFull, (tv & kGuard) != 0u)) {
#pragma unroll
                    for (int k = 0; k < NP; ++k) {
                        // values: base += b = max(gm - NS, 0); older values below it saturate at 0
                        const uint32_t b = __viaddmax_s16x2(gm[k], tc->nNSP, 0u);
                        const uint32_t nb = __vsub2(0u, b);
#pragma unroll
                        for (int a = 0; a < W; ++a) G[k][a] = __viaddmax_s16x2(G[k][a], nb, 0u);
                        gprev[k] = __viaddmax_s16x2(gprev[k], nb, 0u);
                        blo[k] += (int32_t)(b & 0xffffu);
                        bhi[k] += (int32_t)(b >> 16);
                        // loads: P -= bp = max(P - Q - 1, 0); a Y below bp is out of every window: 0x7fff
                        const uint32_t bp = __viaddmax_s16x2(P[k], nQ1P, 0u);
                        const uint32_t nbp = __vsub2(0u, bp);
#pragma unroll
                        for (int a = 0; a < W; ++a) Y[k][a] = __viaddmax_u16x2(Y[k][a], nbp, 0x7fff7fffu);
                        P[k] = __vadd2(P[k], nbp);
                    }
                }
            };
            // demands loaded two layers ahead (the LDS latency stays off the layer chain), Cg pairs
            // four at a time
            uint32_t qbuf[NP][2];
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                qbuf[k][0] = *reinterpret_cast<const uint32_t*>(sb + boff[k]);
                qbuf[k][1] = *reinterpret_cast<const uint32_t*>(sb + boff[k] + Cfg::kRowBytes);
            }
            uint4 cg4 = make_uint4(0u, 0u, 0u, 0u);
            auto cg_of = [&](const int j) -> uint32_t {
                if (j % 4 == 0) cg4 = *reinterpret_cast<const uint4*>(cgc + j);
                return (j % 4 == 0) ? cg4.x : (j % 4 == 1) ? cg4.y : (j % 4 == 2) ? cg4.z : cg4.w;
            };
            auto q_of = [&](const int k, const int j) -> uint32_t {
                const uint32_t q = qbuf[k][j % 2];
                if (j + 2 < W) qbuf[k][j % 2] = *reinterpret_cast<const uint32_t*>(sb + boff[k] + (j + 2) * Cfg::kRowBytes);
                return q;
            };
            // steps of LS layers: every candidate of age >= l + 2 of layer j + l (a split point <= j - 1) and
            // the age-(l + 1) one (split point j, the previous step's last value) are known when the step
            // starts, so all LS layers' first groups and voted groups run back to back, behind ONE vote per
            // group; the split points j + 1 .. j + LS - 1 produced inside the step are folded in last
            // (their loads, hence their window tests, are known early; only the LOP3 waits for the value)
#pragma unroll
            for (int j = 0; j < W; j += LS) {
                uint32_t cgv[LS];
#pragma unroll
                for (int l = 0; l < LS; ++l) cgv[l] = cg_of(j + l);
                uint32_t Pn[NP][LS], a[NP][LS];
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    uint32_t qv[LS];
#pragma unroll
                    for (int l = 0; l < LS; ++l) qv[l] = q_of(k, j + l);
#pragma unroll
                    for (int l = 0; l < LS; l += 2) qmax[k] = __vimax3_u16x2(qmax[k], qv[l], qv[l + 1]);
                    Y[k][j] = imad_u32(P[k], one, QGP);  // split point j (FMA pipe)
                    G[k][j] = gprev[k];
                    Pn[k][0] = P[k] + qv[0];
#pragma unroll
                    for (int l = 1; l < LS; ++l) Pn[k][l] = Pn[k][l - 1] + qv[l];
                }
#pragma unroll
                for (int k = 0; k < NP; ++k)
#pragma unroll
                    for (int l = 0; l < LS; ++l) a[k][l] = first_group(k, j + l, Pn[k][l], l + 1 > 2 ? l + 1 : 2);
#pragma unroll
                for (int gi = 0; gi < W; ++gi) {  // groups of UG ages behind one vote on their youngest
                    const int ag = A0 + 1 + gi * UG;
                    if (ag > W) break;
                    uint32_t dd[NP][LS], kk[NP][LS], dor = 0u;
#pragma unroll
                    for (int k = 0; k < NP; ++k)
#pragma unroll
                        for (int l = 0; l < LS; ++l) {
                            kk[k][l] = cand(k, j + l, Pn[k][l], ag, dd[k][l]);
                            dor |= dd[k][l];
                        }
                    if (!__any_sync(kFull, (dor & kGuard) != 0u)) break;
#pragma unroll
                    for (int k = 0; k < NP; ++k)
#pragma unroll
                        for (int l = 0; l < LS; ++l) {
                            if (ag == W) overflow(k, j + l, dd[k][l]);
                            a[k][l] = group_rest(k, j + l, Pn[k][l], ag, a[k][l], kk[k][l]);
                        }
                }
                uint32_t gmlast[NP];
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    // gn[m], yn[m]: split point j + m (m = 0: from the ring; 1 .. LS: produced here)
                    uint32_t gn[LS + 1], yn[LS + 1];
                    gn[0] = gprev[k];
                    yn[0] = Y[k][j];
#pragma unroll
                    for (int l = 0; l < LS; ++l) {
                        uint32_t m = a[k][l];
                        // in-step ages 2 .. l of layer j + l (split points j + 1 .. j + l - 1; LS <= 4: l <= 3)
                        if (l == 2) {
                            m = __vminu2(m, key_of(gn[1], imad_u32(Pn[k][l], m1, yn[1])));
                        } else if (l == 3) {
                            m = __vimin3_u16x2(m, key_of(gn[2], imad_u32(Pn[k][l], m1, yn[2])),
                                               key_of(gn[1], imad_u32(Pn[k][l], m1, yn[1])));
                        }
                        // age 1 (split point j + l) is always in the window when q <= Q (q > Q: qmax, DESIGN R4)
                        const uint32_t gm = __vminu2(m, gn[l]);
                        gn[l + 1] = gm + cgv[l];
                        yn[l + 1] = imad_u32(Pn[k][l], one, QGP);
                        if (l == LS - 1) gmlast[k] = gm;
                    }
#pragma unroll
                    for (int l = 1; l < LS; ++l) {  // (after every read of these slots' previous contents)
                        G[k][j + l] = gn[l];
                        Y[k][j + l] = yn[l];
                    }
                    gprev[k] = gn[LS];
                    P[k] = Pn[k][LS - 1];
                }
                if ((j + LS) % kU16Check == 0 || j + LS == W) range_check(gmlast);
            }
            stage_release(cs, 32 * (kU16Cons + 1));  // the stage may be refilled once every consumer is done
            if (++cs == NS) {
                cs = 0;
                ++cr;
            }
            if (++c >= nchunks) break;  // (c is warp-uniform: a plain branch, no vote -- measured faster)
            sb = smem_raw + (size_t)cs * Cfg::kStageBytes;
            mbar_wait_warp(&full[cs], cr & 1u);
        }
        if constexpr (TL) {
            if (lane == 0) tl_record(blockIdx.x * kU16Cons + wid, (unsigned)th.y, tl0);
        }
        const bool ok = tc->ok != 0;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            // rem == 0: the last layer computed position n; else position n sits in ring slot rem
            // (pushed by the first padded layer)
            const uint32_t val = rem == 0 ? gprev[k] : ring_slot<W>(G[k], rem);
            int dnf = 0, dni = 0;  // this pair's SAA terms, added to the lane's sums in one update
            long long dsum = 0, dlo = 0, dhi = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t s = s0 + 64 * k + 2 * lane + h;
                const bool live = s < S;
                const uint32_t sh = 16u * (uint32_t)h;
                const bool bad = ((qmax[k] >> sh) & 0xffffu) > Q;
                // (a demand above Q in the LOW half can carry into the high half: recompute the high one)
                const bool tainted = h == 1 && (qmax[k] & 0xffffu) > Q;
                const bool ovf = ((ovfb[k] >> sh) & 0x8000u) != 0u;
                const int fval = (int)((val >> sh) & 0xffffu) + (h ? bhi[k] : blo[k]) + tc->bn;
                const bool deferred = live && (ovf || !ok || tainted) && !bad;
                if (deferred) ovf_list[atomicAdd(ovf_count, 1u)] = ((unsigned long long)t << 40) | (unsigned long long)s;
                if (cost && live && !deferred) cost[(int64_t)t * S + s] = bad ? SPDP_INFEASIBLE : fval;
                if (live && !deferred) {
                    if (bad) {
                        dni += 1;
                    } else {
                        const unsigned long long sq = (unsigned long long)fval * (unsigned long long)fval;
                        dnf += 1;
                        dsum += fval;
                        dlo += (long long)(sq & 0xffffffffull);
                        dhi += (long long)(sq >> 32);
                    }
                }
            }
            if (dnf + dni > 0) {
                LanePart pa = *accp;
                pa.nf += dnf;
                pa.ni += dni;
                pa.sum += dsum;
                pa.sqlo += dlo;
                pa.sqhi += dhi;
                *accp = pa;
            }
        }
    }
    if (slots) flush();
    if constexpr (TL) {
        if (lane == 0) tl_record(blockIdx.x * kU16Cons + wid, 0xfffffff1u, gtimer());  // warp done
    }
    }  // (no early return in either role: the compiler keeps each warp provably converged)
}

spdp_status debug_timeline(void* p) {
    unsigned long long* q = static_cast<unsigned long long*>(p);
    g_tl_on = q != nullptr;
    return cuda_check(cudaMemcpyToSymbol(g_timeline, &q, sizeof(q)), "spdp_debug_timeline");
}

bool u16_loads_ok(int n, uint32_t Q) {
    (void)n;  // P is rebased, so only the per-check growth matters
    return ((int64_t)kU16Check + 2) * ((int64_t)Q + 1) <= 0x8000;
}

spdp_status make_demand_map(CUtensorMap* map, const uint16_t* demand, int64_t ld, int64_t S, int n, int box_cols) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return fail(SPDP_E_CUDA, "split_sweep_u16: cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)S, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(uint16_t)};
    const cuuint32_t box[2] = {(cuuint32_t)box_cols, 1u};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t*>(demand), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SPDP_E_CUDA, "split_sweep_u16: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SPDP_OK;
}

template <int W, int A0, int UG, int LS, bool TL = false>
static spdp_status launch_u16_t(cudaStream_t st, const SweepArgs& a) {
    constexpr int NP = 1, NST = 3;
    if constexpr (!TL && W == 20 && A0 == 6) {
        if (g_tl_on) return launch_u16_t<W, A0, UG, LS, true>(st, a);  // (C2's ordered-set variant only)
    }
    using Cfg = U16Cfg<W, NP, NST>;
    auto kern = split_sweep_u16_kernel<W, A0, UG, NP, NST, LS, TL>;
    int blocks_per_sm = 1;
    if (spdp_status e = kernel_setup((const void*)kern, (int)Cfg::kSmem, 100, kU16Threads, Cfg::kSmem, &blocks_per_sm,
                                     "split_sweep_u16 setup"))
        return e;
    CUtensorMap map;
    if (spdp_status e = make_demand_map(&map, a.demand, a.ld, a.S, a.n, kU16Box)) return e;
    const int64_t ntiles = ((a.S + Cfg::kTile - 1) / Cfg::kTile) * a.T;
    int64_t grid = (int64_t)blocks_per_sm * device_sms();  // (measured: 4-5 CTAs per SM saturate it)
    if (grid > ntiles) grid = ntiles;
    const uint32_t Q = a.Q, pthr = 0x7fffu - Q - (uint32_t)kU16Check * (Q + 1u);
    const U16Consts kc{0xffffffffu, 1u, (Q + 0x8000u) * 0x10001u, ((0x10000u - (Q + 1u)) & 0xffffu) * 0x10001u,
                       (0x7fffu - pthr) * 0x10001u};
    prof_begin(st);
    spdp_status rc = cuda_check(launch_pdl(kern, dim3((unsigned)grid), dim3(kU16Threads), Cfg::kSmem, st, map, a.tours, a.trows,
                                           a.cgs, a.g0, a.tinfo, a.n, a.T, a.S, a.Q, kc, a.cost, a.slots, a.ovf, a.hdr),
                                "split_sweep_u16_kernel");
    set_last_kernel("split_sweep_u16_kernel<%d,%d,%d,%d>", W, A0, UG, LS);
    prof_end(st);
    return rc;
}

template <int LS>
static spdp_status launch_u16_ls(int W, int A0, cudaStream_t st, const SweepArgs& a) {
    switch (W) {
        case 16: return A0 <= 6 ? launch_u16_t<16, 6, 2, LS>(st, a) : A0 <= 8 ? launch_u16_t<16, 8, 2, LS>(st, a)
                                                                              : launch_u16_t<16, 10, 2, LS>(st, a);
        case 20:
            switch (A0 < 5 ? 5 : (A0 > 16 ? 16 : A0)) {
                case 5: return launch_u16_t<20, 5, 2, LS>(st, a);
                case 6: return launch_u16_t<20, 6, 2, LS>(st, a);
                case 7: return launch_u16_t<20, 7, 2, LS>(st, a);
                case 8: return launch_u16_t<20, 8, 2, LS>(st, a);
                case 9: return launch_u16_t<20, 9, 2, LS>(st, a);
                case 10: return launch_u16_t<20, 10, 2, LS>(st, a);
                case 11:
                case 12: return launch_u16_t<20, 12, 2, LS>(st, a);
                case 13:
                case 14: return launch_u16_t<20, 14, 2, LS>(st, a);
                default: return launch_u16_t<20, 16, 2, LS>(st, a);
            }
        case 24: return A0 <= 8 ? launch_u16_t<24, 8, 2, LS>(st, a) : A0 <= 10 ? launch_u16_t<24, 10, 2, LS>(st, a)
                        : A0 <= 12 ? launch_u16_t<24, 12, 2, LS>(st, a) : A0 <= 14 ? launch_u16_t<24, 14, 2, LS>(st, a)
                                                                        : launch_u16_t<24, 16, 2, LS>(st, a);
        default: return A0 <= 8 ? launch_u16_t<32, 8, 2, LS>(st, a) : launch_u16_t<32, 12, 3, LS>(st, a);
    }
}

spdp_status launch_sweep_u16(int W, int mean_w, cudaStream_t st, const SweepArgs& a) {
    // unconditional ages (age 1 + A0 - 1 masked candidates) ~ the expected mean window + 4
    // (SPDP_F_MEAN_WINDOW; C2: mean 4 -> 8, C3: mean 8 -> 12), the rest in voted pairs
    const int A0 = mean_w <= 0 ? 8 : (mean_w + 4 < 5 ? 5 : mean_w + 4);
    return launch_u16_ls<4>(W, A0, st, a);
}

}  // namespace spdp
