// split_u16.cu -- a5 (+ a3/a4 fused, a6 partials): the masked min-plus layer sweep of
// Eq. (3) with TWO scenarios per lane in packed 16-bit halves.
//
// Same DP as split.cu (the separable route cost, g(i) = min_{p in window(i)} g(p) + Cg[i],
// f(n) = min g + B[n]), same copy side shape (per-warp cp.async stream of tour-ordered demand
// rows), but every 32-bit register holds the pair {scenario 2l, scenario 2l+1} of lane l:
//
//  * loads: P = the tour-order prefix of the pair, one u16 per half (P <= 0x7FFF - Q, kept
//    there by a periodic rebase), the demand q clamped to Q + 1 first (VIMNMX.U16x2), so one
//    32-bit add updates both halves with no carry between them.
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
//
// Work decomposition as split.cu's sweeps: one wave of persistent CTAs, each warp takes
// 64-scenario tiles from a global counter and streams W-row chunks (128 B per row) through a
// private NS-stage shared-memory ring with cp.async; candidate groups after the first run
// behind a warp vote on the group's youngest age (the window is a contiguous suffix of ages).
#include <climits>

#include "common.cuh"
#include "split_ws.cuh"

namespace spdp {

constexpr int kU16Warps = 8;
constexpr int kU16Threads = 32 * kU16Warps;
constexpr int kU16Tile = 64;   // scenarios per warp tile (two per lane)
constexpr int kU16Queue = 16;  // tile-id queue entries per warp
constexpr uint32_t kGuard = 0x80008000u;

template <int W, int MB = 0>
struct U16Cfg {
    // MB = 0: W = 16 -> 4 CTAs (32 warps) per SM within 64 registers and 2 stages; wider rings 3 / 2
    static constexpr int kMinBlocks = MB > 0 ? MB : (W <= 16 ? 4 : (W <= 24 ? 3 : 2));  // CTAs per SM
    static constexpr int NS = kMinBlocks >= 4 ? 2 : 3;                                  // stages per warp
    static constexpr int kRowsBytes = W * kU16Tile * (int)sizeof(uint16_t);  // W x 128 B
    static constexpr int kStageBytes = kRowsBytes + W * (int)sizeof(int32_t);
    static constexpr int kWarpBytes = kU16Queue * 8 + NS * kStageBytes;
    static constexpr size_t kSmem = (size_t)kU16Warps * kWarpBytes;
    static_assert(W % 4 == 0, "W must be a multiple of 4");
};

// d = a * b + c on the FMA pipe (b is the runtime value 0xffffffff, so ptxas cannot turn the
// multiply-add into an IADD3 on the ALU pipe, which the candidate LOP3 / VIMNMX3 already load)
__device__ __forceinline__ uint32_t imad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// key = G | (~d & 0x80008000) as one LOP3 (an explicit lop3, so ptxas cannot split it around
// the vote branch that tests d)
__device__ __forceinline__ uint32_t key_of(uint32_t G, uint32_t d) {
    uint32_t k;
    asm("lop3.b32 %0, %1, %2, %3, 0xF2;" : "=r"(k) : "r"(G), "r"(d), "r"(kGuard));
    return k;
}

// Minimum of N packed u16 pairs with ceil((N - 1) / 2) 3-input mins (VIMNMX3.U16x2): the first
// level folds triples, the rest chains (depth ~ N / 3; the layer chain does not wait on it).
template <int N>
__device__ __forceinline__ uint32_t umin_tree(const uint32_t* v) {
    if constexpr (N == 1) return v[0];
    else if constexpr (N == 2) return __vminu2(v[0], v[1]);
    else if constexpr (N == 3) return __vimin3_u16x2(v[0], v[1], v[2]);
    else if constexpr (N == 4) return __vimin3_u16x2(__vminu2(v[0], v[1]), v[2], v[3]);
    else return __vimin3_u16x2(umin_tree<N - 2>(v), v[N - 2], v[N - 1]);
}

// Per-half constants, formed on the host (kernel parameters: uniform registers, so each use is
// one operand, not a re-materialised expression).  Host check: (kU16Check + 2)(Q + 1) <= 0x8000.
struct U16Consts {
    uint32_t m1;    // 0xffffffff (the IMAD multiplier)
    uint32_t one;   // 1 (the IMAD multiplier of an add that should issue on the FMA pipe)
    uint32_t q1p;   // (Q + 1) per half: the demand clamp
    uint32_t qgp;   // (Q + 0x8000) per half: Y = P + Q + guard
    uint32_t nq1p;  // -(Q + 1) per half (16-bit two's complement)
    uint32_t nocopy;  // TUNING (temporary): 1 = skip the demand copies (timing of the compute side only)
    uint32_t padd;  // (0x7fff - pthr) per half, pthr = 0x7fff - Q - kU16Check (Q + 1): bit 15 of P + padd
                    // is set iff P > pthr (a load rebase is due)
};

template <int W, int MB>
struct U16Stream {  // copy cursor of one warp
    int c;                // next chunk of the copy tile (== nchunks: move to the next tile)
    int stage;            // next stage to fill
    unsigned qw;          // queue write index
    int ct;               // tour of the copy tile (-1: no more tiles)
    int64_t s0;           // first scenario of the copy tile
    int segs;             // 16-byte segments per row in the copy tile (8 unless ragged)
    unsigned nid;         // lane 0: the id of the tile after the copy tile (atomic issued one tile ahead)
    const uint16_t* src;  // lane < W: the source of this lane's row in the next chunk to issue

    // The tile-id counter and the row-pointer table are read one step ahead, so neither the
    // atomic's latency nor the pointer load stalls the warp (they were its top long-scoreboard
    // stalls).
    __device__ __forceinline__ void set_tile(unsigned id, uint32_t ntile_s, uint32_t ntiles, int64_t S) {
        ct = -1;
        if (id < ntiles) {
            const uint32_t t = id / ntile_s, b = id - t * ntile_s;
            ct = (int)t;
            s0 = (int64_t)b * kU16Tile;
            const int64_t left = S - s0;
            segs = left >= kU16Tile ? 8 : (int)((left + 7) >> 3);
        }
    }
    // the row pointer of this lane's row in chunk cc of a tile of tour t (s0 is added at use, so
    // the load's latency stays off the copy path)
    __device__ __forceinline__ const uint16_t* row_src(const uint16_t* const* __restrict__ rowp, int t, int cc, int n,
                                                       int lane) const {
        const int r = cc * W + lane;
        return (lane < W && r < n) ? rowp[(int64_t)t * (n + kTabPad) + r] : nullptr;
    }
    __device__ __forceinline__ void start(const uint16_t* const* __restrict__ rowp, int64_t S, uint32_t ntile_s,
                                          uint32_t ntiles, int n, int lane, unsigned* tile_ctr) {
        unsigned id = 0;
        if (lane == 0) id = atomicAdd(tile_ctr, 1u);
        id = __shfl_sync(kFull, id, 0);
        nid = 0;
        if (lane == 0) nid = atomicAdd(tile_ctr, 1u);
        set_tile(id, ntile_s, ntiles, S);
        c = 0;
        src = ct >= 0 ? row_src(rowp, ct, 0, n, lane) : nullptr;
    }

    // One chunk: lane r < W copies demand row r0 + r of the tile (8 x 16 B from its row pointer,
    // built by tour_prep_kernel), or fills it with the padding demand past row n; lanes W.. (or
    // 0.. when W = 32) copy the chunk's W Cg pairs.
    __device__ __forceinline__ void issue(unsigned char* stage_base, int2* tq, const uint16_t* const* __restrict__ rowp,
                                          const int32_t* __restrict__ cgp, int64_t S, uint32_t ntile_s, uint32_t ntiles,
                                          int n, int nchunks, int cgs_stride, int lane, unsigned* tile_ctr,
                                          uint32_t qpad2, uint32_t nocopy) {
        using Cfg = U16Cfg<W, MB>;
        // (every shuffle / vote here is executed by the whole warp at a point the compiler can prove
        // convergent; a shuffle under a lane-dependent branch would cost the layer loop's votes a
        // divergence check, BRA.DIV)
        const unsigned idn = __shfl_sync(kFull, nid, 0);  // the id of the tile after the copy tile
        if (c == nchunks) {  // the next tile (its id and first row pointers were fetched ahead)
            if (lane == 0) nid = atomicAdd(tile_ctr, 1u);
            set_tile(idn, ntile_s, ntiles, S);
            c = 0;
        }
        if (c == 0) {
            if (lane == 0) tq[qw & (kU16Queue - 1)] = ct >= 0 ? make_int2(ct, (int)(s0 / kU16Tile)) : make_int2(-1, 0);
            ++qw;
        }
        if (ct >= 0) {
            unsigned char* sb = stage_base + stage * Cfg::kStageBytes;
            const int r0 = c * W;
            if (lane < W && !nocopy) {
                unsigned char* dst = sb + lane * (kU16Tile * 2);
                if (r0 + lane < n) {
                    const uint16_t* sp = src + s0;
                    if (segs == 8) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) cp_async16(dst + 16 * k, sp + 8 * k);
                    } else {
                        for (int k = 0; k < segs; ++k) cp_async16(dst + 16 * k, sp + 8 * k);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        *reinterpret_cast<uint4*>(dst + 16 * k) = make_uint4(qpad2, qpad2, qpad2, qpad2);
                }
            }
            constexpr int kCgLane0 = W + W / 4 <= 32 ? W : 0;
            if (lane >= kCgLane0 && lane < kCgLane0 + W / 4) {
                const int cb = lane - kCgLane0;
                cp_async16(sb + Cfg::kRowsBytes + cb * 16, cgp + (int64_t)ct * kCgPlanes * cgs_stride + r0 + cb * 4);
            }
            // the next chunk's row sources: this tile's chunk c + 1, or the next tile's chunk 0
            // (c == nchunks - 1: the id read above is still the next tile's, its atomic long done)
            if (c + 1 < nchunks) {
                src = row_src(rowp, ct, c + 1, n, lane);
            } else if (idn < ntiles) {
                src = row_src(rowp, (int)(idn / ntile_s), 0, n, lane);
            }
        }
        cp_async_commit();
        ++c;
        stage = (stage + 1 == Cfg::NS) ? 0 : stage + 1;
    }
};

// A0: ages scanned unconditionally (age 1 + A0 - 1 masked candidates); then groups of UG ages,
// each behind a warp vote on its youngest age; the scan of age W also tests for ring overflow.
template <int W, int A0, int UG, bool PR, bool CL, int MB>
__global__ void __launch_bounds__(kU16Threads, U16Cfg<W, MB>::kMinBlocks)
    split_sweep_u16_kernel(const uint16_t* const* __restrict__ rowp, const int32_t* __restrict__ cgs,
                           const int32_t* __restrict__ g0s, const TourInfo* __restrict__ tinfo, int n, int T, int64_t S,
                           uint32_t Q, U16Consts kc, int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ slots,
                           unsigned long long* __restrict__ ovf_list, unsigned* __restrict__ hdr) {
    using Cfg = U16Cfg<W, MB>;
    constexpr int NS = Cfg::NS;
    static_assert(A0 >= 2 && A0 <= W && UG >= 0 && kU16Queue >= NS + 2, "bad u16 sweep config");
    pdl_wait();  // tables, counters and partial slots come from tour_prep_kernel
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned char* wbase = smem_raw + (size_t)wid * Cfg::kWarpBytes;
    int2* tq = reinterpret_cast<int2*>(wbase);
    unsigned char* stage_base = wbase + kU16Queue * 8;
    const uint32_t ntile_s = (uint32_t)((S + kU16Tile - 1) / kU16Tile);
    const uint32_t ntiles = ntile_s * (uint32_t)T;
    const int nchunks = (n + W - 1) / W;
    const int rem = n % W;
    const int cgs_stride = cg_stride(n);
    const uint32_t qpad = Q < 65535u ? Q : 65535u;
    const int slot = (blockIdx.x * kU16Warps + wid) % kSlots;
    unsigned* ovf_count = hdr + HDR_OVF_COUNT;

    const uint32_t m1 = kc.m1, one = kc.one, Q1P = kc.q1p, QGP = kc.qgp, nQ1P = kc.nq1p, PADD = kc.padd;

    U16Stream<W, MB> cs;
    cs.stage = 0;
    cs.qw = 0u;
    cs.start(rowp, S, ntile_s, ntiles, n, lane, hdr + HDR_TILE);
    auto issue = [&]() {
        cs.issue(stage_base, tq, rowp, cgs + 2 * cgs_stride, S, ntile_s, ntiles, n, nchunks, cgs_stride, lane,
                 hdr + HDR_TILE, qpad * 0x10001u, kc.nocopy);
    };
    for (int k = 0; k < NS; ++k) issue();

    uint32_t G[W], Y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) G[k] = 0u;

    struct LanePart {
        int nf, ni;
        long long sum, sqlo, sqhi;
    };
    __shared__ LanePart accs[kU16Threads];
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
    __shared__ TourConsts tcs[kU16Warps];
    TourConsts* tc = &tcs[wid];
    int cstage = 0;
    cp_async_wait<NS - 1>();
    __syncwarp();
    for (unsigned u = 0;; ++u) {
        const int2 tile = tq[u & (kU16Queue - 1)];
        if (__all_sync(kFull, tile.x < 0)) break;  // (a vote: keeps the warp provably converged)
        const int t = tile.x;
        const int64_t s0 = (int64_t)tile.y * kU16Tile;
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
        int32_t blo = tc->base0, bhi = blo;
#pragma unroll
        for (int k = 0; k < W; ++k) Y[k] = 0x7fff7fffu;  // no window ever reaches an empty slot
        uint32_t P = 0u, gprev = tc->nsP, qmax = 0u, ovfb = 0u;

        for (int c = 0;;) {
            const unsigned char* sb = stage_base + cstage * Cfg::kStageBytes;
            const uint32_t* bufw = reinterpret_cast<const uint32_t*>(sb) + lane;
            const uint32_t* cgc = reinterpret_cast<const uint32_t*>(sb + Cfg::kRowsBytes);
            // the key of the candidate of age a (>= 2) at layer jj: G inside the window, >= 0x8000 outside;
            // d (bit 15 of a half set iff inside) is returned for the votes
            auto cand = [&](const int jj, const uint32_t Pn, const int a, uint32_t& d) -> uint32_t {
                const int s = (jj - a + 1 + 2 * W) % W;
                d = imad_u32(Pn, m1, Y[s]);
                return key_of(G[s], d);
            };
            uint32_t qc_even = 0u;
            // demands loaded kQPf layers ahead (the LDS latency stays off the layer chain), Cg pairs
            // four at a time
            constexpr int kQPf = 2;
            uint32_t qbuf[kQPf];
#pragma unroll
            for (int k = 0; k < kQPf; ++k) qbuf[k] = bufw[k * 32];
            uint4 cg4 = make_uint4(0u, 0u, 0u, 0u);
            // the unconditional ages 2..A0 of layer jj, folded
            auto first_group = [&](const int jj, const uint32_t Pn) -> uint32_t {
                uint32_t key[A0 - 1];
#pragma unroll
                for (int k = 2; k <= A0; ++k) {
                    uint32_t d;
                    key[k - 2] = cand(jj, Pn, k, d);
                    if (k == W) ovfb |= d & kGuard;  // the window reaches the oldest ring age
                }
                return umin_tree<A0 - 1>(key);
            };
            // the keys of group gi (ages a0 + 1 .. a0 + UG - 1; age a0 done by the caller) folded into a
            auto group_rest = [&](const int jj, const uint32_t Pn, const int a0, uint32_t a, const uint32_t k0) {
                uint32_t key[UG + 1];
                key[0] = a;
                key[1] = k0;
#pragma unroll
                for (int k = 1; k < UG; ++k) {
                    if (a0 + k <= W) {
                        uint32_t d;
                        key[k + 1] = cand(jj, Pn, a0 + k, d);
                        if (a0 + k == W) ovfb |= d & kGuard;
                    } else {
                        key[k + 1] = 0xffffffffu;
                    }
                }
                return umin_tree<UG + 1>(key);
            };
            // every kU16Check layers: rebase values and loads if either approaches 2^15 (see the header)
            auto range_check = [&](const uint32_t gm) {
                const uint32_t tv = (gprev + tc->GADD) | (P + PADD);
                if (__any_sync(kFull, (tv & kGuard) != 0u)) {
                    // values: base += b = max(gm - NS, 0); older values below it saturate at 0
                    const uint32_t b = __viaddmax_s16x2(gm, tc->nNSP, 0u);
                    const uint32_t nb = __vsub2(0u, b);
#pragma unroll
                    for (int k = 0; k < W; ++k) G[k] = __viaddmax_s16x2(G[k], nb, 0u);
                    gprev = __viaddmax_s16x2(gprev, nb, 0u);
                    blo += (int32_t)(b & 0xffffu);
                    bhi += (int32_t)(b >> 16);
                    // loads: P -= bp = max(P - Q - 1, 0); a Y below bp is out of every window: 0x7fff
                    const uint32_t bp = __viaddmax_s16x2(P, nQ1P, 0u);
                    const uint32_t nbp = __vsub2(0u, bp);
#pragma unroll
                    for (int k = 0; k < W; ++k) Y[k] = __viaddmax_u16x2(Y[k], nbp, 0x7fff7fffu);
                    P = __vadd2(P, nbp);
                }
            };
            auto cg_of = [&](const int j) -> uint32_t {
                if (j % 4 == 0) cg4 = *reinterpret_cast<const uint4*>(cgc + j);
                return (j % 4 == 0) ? cg4.x : (j % 4 == 1) ? cg4.y : (j % 4 == 2) ? cg4.z : cg4.w;
            };
            auto q_of = [&](const int j) -> uint32_t {
                const uint32_t q = qbuf[j % kQPf];
                if (j + kQPf < W) qbuf[j % kQPf] = bufw[(j + kQPf) * 32];
                return q;
            };
            if constexpr (PR) {
                // Two layers per step: the candidates of age >= 2 of BOTH layers depend only on values
                // known before either (layer j + 1's age 2 is layer j's age 1), so both first groups run
                // back to back and one warp vote per group guards both layers' deeper candidates.
#pragma unroll
                for (int j = 0; j < W; j += 2) {
                    const uint32_t q0 = q_of(j), q1 = q_of(j + 1);
                    const uint32_t cg0 = cg_of(j), cg1 = cg_of(j + 1);
                    const uint32_t qc0 = CL ? __vminu2(q0, Q1P) : q0, qc1 = CL ? __vminu2(q1, Q1P) : q1;
                    qmax = __vimax3_u16x2(qmax, qc0, qc1);
                    Y[j] = imad_u32(P, one, QGP);  // split point of layer j's age 1 (FMA pipe)
                    G[j] = gprev;
                    const uint32_t Pn0 = P + qc0, Pn1 = Pn0 + qc1;
                    uint32_t a0 = first_group(j, Pn0), a1 = first_group(j + 1, Pn1);
#pragma unroll
                    for (int gi = 0; gi < W; ++gi) {
                        if (UG == 0) break;  // TUNING (temporary): no deep groups
                        const int ag = A0 + 1 + gi * UG;
                        if (ag > W) break;
                        uint32_t d0, d1;
                        const uint32_t k0 = cand(j, Pn0, ag, d0), k1 = cand(j + 1, Pn1, ag, d1);
                        if (__builtin_expect(!__any_sync(kFull, ((d0 | d1) & kGuard) != 0u), 1)) break;
                        if (ag == W) ovfb |= (d0 | d1) & kGuard;
                        a0 = group_rest(j, Pn0, ag, a0, k0);
                        a1 = group_rest(j + 1, Pn1, ag, a1, k1);
                    }
                    // age 1 (p = i - 1) is always in the window when q <= Q (q > Q: qmax, DESIGN R4)
                    const uint32_t g0 = __vminu2(a0, gprev) + cg0;
                    G[j + 1] = g0;  // (after layer j read slot j + 1 as its age W)
                    Y[j + 1] = imad_u32(Pn0, one, QGP);
                    const uint32_t gm1 = __vminu2(a1, g0);
                    gprev = gm1 + cg1;
                    P = Pn1;
                    if ((j + 1) % kU16Check == kU16Check - 1 || j + 1 == W - 1) range_check(gm1);
                }
            } else {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    const uint32_t q = q_of(j);
                    const uint32_t cg = cg_of(j);
                    const uint32_t qc = CL ? __vminu2(q, Q1P) : q;
                    if (j & 1) qmax = __vimax3_u16x2(qmax, qc_even, qc);  // (W is even)
                    else qc_even = qc;
                    Y[j] = imad_u32(P, one, QGP);  // split point i - 1 (age 1 of this layer)
                    G[j] = gprev;
                    const uint32_t Pn = P + qc;
                    uint32_t a = first_group(j, Pn);
#pragma unroll
                    for (int gi = 0; gi < W; ++gi) {  // groups of UG ages behind a vote on the youngest
                        const int ag = A0 + 1 + gi * UG;
                        if (ag > W) break;
                        uint32_t d0;
                        const uint32_t k0 = cand(j, Pn, ag, d0);
                        if (__builtin_expect(!__any_sync(kFull, (d0 & kGuard) != 0u), 1)) break;
                        if (ag == W) ovfb |= d0 & kGuard;
                        a = group_rest(j, Pn, ag, a, k0);
                    }
                    // age 1 (p = i - 1) is always in the window when q <= Q (q > Q: qmax, DESIGN R4)
                    const uint32_t gm = __vminu2(a, gprev);
                    gprev = gm + cg;
                    P = Pn;
                    if (j % kU16Check == kU16Check - 1 || j == W - 1) range_check(gm);
                }
            }
            __syncwarp();
            issue();
            cstage = (cstage + 1 == NS) ? 0 : cstage + 1;
            cp_async_wait<NS - 1>();
            __syncwarp();
            if (__all_sync(kFull, ++c >= nchunks)) break;
        }
        uint32_t val = gprev;  // rem == 0: the last layer computed position n
        if (rem != 0) {        // else position n sits in ring slot rem (pushed by the first padded layer)
#pragma unroll
            for (int k = 0; k < W; ++k)
                if (k == rem) val = G[k];
        }
        const bool ok = tc->ok != 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t s = s0 + 2 * lane + h;
            const bool live = s < S;
            const uint32_t sh = 16u * (uint32_t)h;
            const bool bad = ((qmax >> sh) & 0xffffu) > Q;
            // (unclamped loads: a demand above Q in the LOW half can carry into the high half, so the
            // high scenario of such a pair is recomputed by the finish kernel)
            const bool tainted = !CL && h == 1 && (qmax & 0xffffu) > Q;
            const bool ovf = ((ovfb >> sh) & 0x8000u) != 0u;
            const int fval = (int)((val >> sh) & 0xffffu) + (h ? bhi : blo) + tc->bn;
            const bool deferred = live && (ovf || !ok || tainted) && !bad;
            if (deferred) ovf_list[atomicAdd(ovf_count, 1u)] = ((unsigned long long)t << 40) | (unsigned long long)s;
            if (cost && live && !deferred) cost[(int64_t)t * S + s] = bad ? SPDP_INFEASIBLE : fval;
            if (live && !deferred) {
                LanePart pa = *accp;
                if (bad) {
                    pa.ni += 1;
                } else {
                    const unsigned long long sq = (unsigned long long)fval * (unsigned long long)fval;
                    pa.nf += 1;
                    pa.sum += fval;
                    pa.sqlo += (long long)(sq & 0xffffffffull);
                    pa.sqhi += (long long)(sq >> 32);
                }
                *accp = pa;
            }
        }
    }
    if (slots) flush();
    cp_async_wait<0>();
}

bool u16_loads_ok(int n, uint32_t Q) {
    (void)n;  // P is rebased, so only the per-check growth matters
    return ((int64_t)kU16Check + 2) * ((int64_t)Q + 1) <= 0x8000;
}

template <int W, int A0, int UG, bool PR = true, bool CL = false, int MB = 0>
static spdp_status launch_u16_t(cudaStream_t st, const SweepArgs& a, size_t pad = 0, uint32_t nocopy = 0) {
    using Cfg = U16Cfg<W, MB>;
    auto kern = split_sweep_u16_kernel<W, A0, UG, PR, CL, MB>;
    int blocks_per_sm = 1;
    if (spdp_status e = kernel_setup((const void*)kern, (int)(Cfg::kSmem + pad), 100, kU16Threads, Cfg::kSmem + pad, &blocks_per_sm,
                                     "split_sweep_u16 setup"))
        return e;
    const int64_t ntiles = ((a.S + kU16Tile - 1) / kU16Tile) * a.T;
    int64_t grid = (int64_t)blocks_per_sm * device_sms();
    const int64_t need = (ntiles + kU16Warps - 1) / kU16Warps;
    if (grid > need) grid = need;
    const uint32_t Q = a.Q, pthr = 0x7fffu - Q - (uint32_t)kU16Check * (Q + 1u);
    const U16Consts kc{0xffffffffu, 1u, (Q + 1u) * 0x10001u, (Q + 0x8000u) * 0x10001u,
                       ((0x10000u - (Q + 1u)) & 0xffffu) * 0x10001u, nocopy, (0x7fffu - pthr) * 0x10001u};
    prof_begin(st);
    spdp_status rc = cuda_check(launch_pdl(kern, dim3((unsigned)grid), dim3(kU16Threads), Cfg::kSmem + pad, st, a.rowp, a.cgs,
                                           a.g0, a.tinfo, a.n, a.T, a.S, a.Q, kc, a.cost, a.slots, a.ovf, a.hdr),
                                "split_sweep_u16_kernel");
    set_last_kernel("split_sweep_u16_kernel<%d,%d,%d,%d,%d>", W, A0, UG, PR ? 1 : 0, CL ? 1 : 0);
    prof_end(st);
    return rc;
}

spdp_status launch_sweep_u16(int W, int mean_w, cudaStream_t st, const SweepArgs& a) {
    // unconditional ages (age 1 + A0 - 1 masked candidates) ~ the expected mean window + 2
    // (SPDP_F_MEAN_WINDOW; C2: mean 4 -> 6, C3: mean 8 -> 10), the rest in voted pairs
    const bool pr = mean_w < 100;  // TUNING (temporary): mean_w >= 100 selects the clamped-load body
    if (!pr) mean_w -= 100;
    const int A0 = mean_w <= 0 ? 6 : (mean_w + 2 < 5 ? 5 : mean_w + 2);
    if (!pr) {  // TUNING (temporary) variants
        switch (mean_w) {
            case 1: return launch_u16_t<20, 6, 2, true, false, 3>(st, a, 40 * 1024);  // 2 CTAs per SM
            case 2: return launch_u16_t<20, 6, 2, true, false, 4>(st, a);             // 4 CTAs per SM, 64 regs
            case 3: return launch_u16_t<20, 6, 2, true, false, 3>(st, a, 150 * 1024); // 1 CTA per SM
            case 5: return launch_u16_t<20, 6, 2, true, false>(st, a, 0, 1u);         // no demand copies
            case 6: return launch_u16_t<20, 6, 0, true, false>(st, a);                // no deep groups (wrong)
            case 7: return launch_u16_t<20, 8, 0, true, false>(st, a);                // no deep groups (wrong)
            case 8: return launch_u16_t<20, 4, 0, true, false>(st, a);                // no deep groups (wrong)
            default: return launch_u16_t<20, 6, 2, true, true>(st, a);
        }
    }
    switch (W) {
        case 8: return launch_u16_t<8, 6, 2, true, false, 3>(st, a);  // TUNING (temporary)
        case 16: return A0 <= 6 ? launch_u16_t<16, 6, 2>(st, a) : A0 <= 8 ? launch_u16_t<16, 8, 2>(st, a)
                                                                          : launch_u16_t<16, 10, 2>(st, a);
        case 20:
            switch (A0) {
                case 5: return launch_u16_t<20, 5, 2>(st, a);
                case 6: return launch_u16_t<20, 6, 2>(st, a);
                case 7: return launch_u16_t<20, 7, 2>(st, a);
                case 8: return launch_u16_t<20, 8, 2>(st, a);
                case 9: return launch_u16_t<20, 9, 2>(st, a);
                case 12: return launch_u16_t<20, 12, 2>(st, a);
                case 20: return launch_u16_t<20, 20, 2>(st, a);
                default: return launch_u16_t<20, 10, 2>(st, a);
            }
        case 24: return A0 <= 6 ? launch_u16_t<24, 6, 2>(st, a) : A0 <= 8 ? launch_u16_t<24, 8, 2>(st, a)
                                                                          : launch_u16_t<24, 10, 2>(st, a);
        case 32: return A0 <= 6 ? launch_u16_t<32, 6, 2>(st, a) : launch_u16_t<32, 10, 3>(st, a);
        default: return launch_u16_t<64, 6, 2>(st, a);  // TUNING (temporary)
    }
}

}  // namespace spdp
