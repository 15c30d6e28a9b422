// split.cu -- a2 (tour prep), a3/a4 (standalone prefix + mask), a5/a8 (masked
// min-plus layer sweep, single and batched tours) and a6 (fused SAA partials).
//
// The DP (Eq. (1)-(3)):
//   f(0) = 0, f(i) = min_{mask(i) <= p <= i-1} f(p) + t(p, i),
//   t(p, i) = c_{0,s_{p+1}} + sum_{k=p+1}^{i-1} c_{s_k,s_{k+1}} + c_{s_i,0}.
// With the tour distance prefix D the route cost is separable and,
// in integers, exactly  t(p, i) = A[p] + B[i],  A[p] = c_{0,s_{p+1}} - D[p+1],
// B[i] = D[i] + c_{s_i,0}  (SURVEY finding 3).  With g(p) = f(p) + A[p]:
//   g(0) = c_{0,s_1},   g(i) = min_{p in window(i)} g(p) + Cg[i],
//   Cg[i] = B[i] + A[i] = c_{s_i,0} + c_{0,s_{i+1}} - c_{s_i,s_{i+1}}   (i < n),
//   f(n) = min_{p in window(n)} g(p) + B[n].
// So each Eq. (3) candidate is one integer min, and the scenario-invariant
// route-cost table c(i,j) collapses to two length-n vectors per tour.
//
// Parallel layout: scenarios -> threads (scenario-level
// parallelism); tours -> blockIdx.y (batched mode); the transition-level
// parallelism of PAPER:144-146 is used by split_general_kernel, where a warp
// cooperates on one scenario's window with a shuffle min.
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "split_ws.cuh"

namespace spdp {

// ---------------------------------------------------------------- a2: tour prep
// dynamic shared memory of tour_prep_kernel: 37 long longs (warp sums, D[n], block max, ext[5]),
// the validation bitmap, the Cg of every position
static inline size_t tour_prep_smem(int n) {
    return 37 * sizeof(long long) + sizeof(unsigned) * (size_t)((n + 32) / 32 + 1) + sizeof(int) * (size_t)n;
}

// One CTA per tour.  tab[i] = {row of customer s_{i+1}, Cg[i]} (0-based layer i
// computes f(i+1)); tab[n-1].y = B[n].  g0[t] = c_{0,s_1}.  D is a block scan.
// Also zeroes the tour's SAA partial and the overflow counter.
__global__ void __launch_bounds__(1024) tour_prep_kernel(const int32_t* __restrict__ tours, int n,
                                                         const int32_t* __restrict__ dist,
                                                         int2* __restrict__ tabs, int32_t* __restrict__ g0,
                                                         const uint16_t* __restrict__ demand, int64_t ld,
                                                         const uint16_t** __restrict__ rowps, TourInfo* __restrict__ tinfo,
                                                         int32_t* __restrict__ cgs, int32_t* __restrict__ trows,
                                                         spdp_saa_partial* __restrict__ slots,
                                                         unsigned* __restrict__ hdr, spdp_saa_partial* __restrict__ partial,
                                                         int validate) {
    extern __shared__ unsigned char smem_raw[];
    long long* wsum = reinterpret_cast<long long*>(smem_raw);              // 32 warp sums
    long long* dn = wsum + 32;                                             // D[n]
    int* cmx = reinterpret_cast<int*>(dn + 1);                             // block max of the used costs
    // ext: [0] NS = sum of max(0, -Cg), [1] max(0, max Cg), [2] the largest sum of max(0, Cg) over
    // kU16Check consecutive layers, [3] B[n] (the packed-u16 sweep's range constants, TourInfo), [4] g0
    int* ext = reinterpret_cast<int*>(smem_raw + 34 * sizeof(long long));
    unsigned* seen = reinterpret_cast<unsigned*>(smem_raw + 37 * sizeof(long long));  // bitmap
    int* cgsm = reinterpret_cast<int*>(seen + ((n + 32) / 32 + 1));  // Cg of every position (the window sums)
    pdl_trigger();  // the sweep's CTAs may launch now (they wait for this grid's completion)
    const int t = blockIdx.x;
    const int32_t* tour = tours + (int64_t)t * n;
    int2* tab = tabs + (int64_t)t * (n + kTabPad);
    const int64_t N1 = n + 1;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5;

    if (t == 0 && tid == 0) {
        hdr[HDR_OVF_COUNT] = 0u;
        hdr[HDR_TILE] = 0u;
    }
    if (slots)
        for (int i = tid; i < kSlots; i += nt) slots[(int64_t)t * kSlots + i] = spdp_saa_partial{0, 0, 0, 0, 0, 0};
    if (tid == 0) {
        *cmx = 0;
        ext[0] = ext[1] = ext[2] = ext[3] = ext[4] = 0;
        if (partial) partial[t] = spdp_saa_partial{0, 0, 0, 0, 0, 0};  // the finish kernel accumulates
    }
    if (validate) {
        for (int i = tid; i < (n + 32) / 32; i += nt) seen[i] = 0u;
        __syncthreads();
    }
    auto node = [&](int i) -> int {  // customer at 0-based position i, clamped to 1..n
        int c = tour[i];
        return c < 1 ? 1 : (c > n ? n : c);
    };
    // chunked block scan of arcs: arc[i] = c_{s_{i+1}, s_{i+2}}, i = 0..n-2
    const int per = (n + nt - 1) / nt;
    const int lo = tid * per, hi = min(n, lo + per);
    long long local = 0;
    int cmax = 0;
    unsigned bad = 0;
    for (int i = lo; i < hi; ++i) {
        const int a = node(i);
        if (validate) {
            const int raw = tour[i];
            if (raw < 1 || raw > n) bad |= ST_NOT_PERM;
            else if (atomicOr(&seen[raw >> 5], 1u << (raw & 31)) & (1u << (raw & 31))) bad |= ST_NOT_PERM;
        }
        const int c0a = dist[a], ca0 = dist[(int64_t)a * N1];
        cmax = max(cmax, max(c0a, ca0));
        if (c0a < 0 || ca0 < 0) bad |= ST_NEG_DIST;
        if (i + 1 < n) {
            const int arc = dist[(int64_t)a * N1 + node(i + 1)];
            if (arc < 0) bad |= ST_NEG_DIST;
            cmax = max(cmax, arc);
            local += arc;
        }
    }
    // exclusive scan of per-thread sums
    long long incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        long long v = (lane < (nt >> 5)) ? wsum[lane] : 0;
        long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long u = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += u;
        }
        if (lane < (nt >> 5)) wsum[lane] = x - v;  // exclusive warp offsets
    }
    __syncthreads();
    long long D = wsum[wid] + incl - local;  // D at position lo+1 (1-based): sum of arcs before lo
    if (lo <= n - 1 && n - 1 < hi) *dn = D + local;  // D[n] = all arcs
    atomicMax(cmx, cmax);
    // every table entry of this thread's positions in one pass (dist re-reads hit L1):
    // tab[i] = {row, Cg}, the int / fp32 Cg planes and the demand row pointer
    const int cs = cg_stride(n);
    int32_t* cgi = cgs + (int64_t)t * kCgPlanes * cs;  // plane 0: int Cg, 1: fp32 Cg / 2^24, 2: packed u16 pair
    const uint16_t** rowp = rowps + (int64_t)t * (n + kTabPad);
    int32_t* trow = trows + (int64_t)t * trow_stride(n);
    int ns_local = 0, cgpos_max = 0;
    for (int i = lo; i < hi; ++i) {
        const int a = node(i);
        const int ca0 = dist[(int64_t)a * N1];
        int2 e;
        e.x = a - 1;
        if (i + 1 < n) {
            const int b = node(i + 1);
            const int arc = dist[(int64_t)a * N1 + b];
            e.y = ca0 + dist[b] - arc;  // Cg[i+1] (1-based) = c_{s_i,0} + c_{0,s_{i+1}} - c_{s_i,s_{i+1}}
            D += arc;
        } else {
            e.y = (int)(D + ca0);       // B[n] = D[n] + c_{s_n,0}
        }
        tab[i] = e;
        cgsm[i] = e.y;
        cgi[i] = e.y;
        cgi[cs + i] = __float_as_int((float)e.y * 0x1p-24f);
        if (i + 1 < n) {
            cgi[2 * cs + i] = (int32_t)((uint32_t)e.y * 0x10001u);  // the pair {Cg, Cg} as one 32-bit add
            ns_local = min(ns_local + max(0, -e.y), 1 << 16);
            cgpos_max = max(cgpos_max, e.y);
        } else {
            cgi[2 * cs + i] = 0;  // layer n: B[n] is added in int32 at the end
            ext[3] = e.y;
        }
        rowp[i] = demand + (int64_t)e.x * ld;
        trow[i] = e.x;
    }
    if (ns_local) atomicAdd(&ext[0], ns_local);
    if (cgpos_max) atomicMax(&ext[1], cgpos_max);
    for (int i = n + tid; i < cs; i += nt) {  // padding (rows: row 0; Cg: 0)
        if (i < n + kTabPad) {
            tab[i] = make_int2(0, 0);
            rowp[i] = demand;
        }
        cgi[i] = 0;
        cgi[cs + i] = 0;
        cgi[2 * cs + i] = 0;
    }
    for (int i = cs + tid; i < n + kTabPad; i += nt) {
        tab[i] = make_int2(0, 0);
        rowp[i] = demand;
    }
    for (int i = n + tid; i < trow_stride(n); i += nt) trow[i] = n;  // outside the tensor: zeros
    if (lo == 0 && hi > 0) {  // (the thread of position 0: its dist row is in L1)
        const int g = dist[node(0)];
        g0[t] = g;
        ext[4] = g;
    }
    __syncthreads();
    {  // the largest sum of max(0, Cg) over kU16Check consecutive layers (cgsm is complete)
        int wmax = 0;
        for (int i = lo; i < min(hi, n - 1); ++i) {
            int sum = 0;
            for (int k = i; k < min(i + kU16Check, n - 1); ++k) sum += max(0, cgsm[k]);
            wmax = max(wmax, min(sum, 1 << 20));
        }
        if (wmax) atomicMax(&ext[2], wmax);
    }
    __syncthreads();
    if (tid == 0) {  // g0f = (g0 + OFF) / 2^24
        const long long OFF = *dn, cm = *cmx;
        TourInfo ti;
        ti.g0f_bits = __float_as_int((float)(ext[4] + OFF) * 0x1p-24f);
        ti.off = (int)(OFF < INT_MAX ? OFF : INT_MAX);
        // g + OFF <= (2n + 1) cmax + OFF and f(n) + OFF <= 2 n cmax + OFF: all below 2^24
        ti.ok = ((2LL * n + 2) * cm + OFF < (1LL << 24)) ? 1 : 0;
        // packed-u16 sweep: values relative to a base stay in [0, 0x7FFF]
        const int ns = ext[0], cgp = ext[1], win = ext[2];
        ti.ns16 = ns < 0x7FFF ? ns : 0x7FFF;
        ti.thr16 = 0x7FFF - (win < 0x7FFF ? win : 0x7FFF);
        ti.ok16 = ((long long)ns + cgp + win <= 0x7FFF) ? 1 : 0;
        ti.bn = ext[3];
        ti.pad = 0;
        tinfo[t] = ti;
    }
    // range: |g|, |f| <= 3 n cmax (SURVEY §7 hard part 10)
    if ((long long)cmax * (3LL * n + 1) >= (long long)INT_MAX) bad |= ST_RANGE;
    if (bad) atomicOr(&hdr[HDR_STATUS], bad);
}

// ---------------------------------------------------------------- a5: the sweep
// One scenario per thread.  The candidate ring holds, for the last W split
// points p (slot p mod W): G = g(p) and Y = P'(p) + Q, where P'(p) = 1 + sum of
// the first p tour-order demands.  p is in the Eq. (3) window of layer i iff
// P'(i) - P'(p) <= Q  <=>  Y >= P'(i).  Because q >= 0 the
// window is a contiguous suffix (DESIGN R5), so the candidate loop walks from
// the newest slot backwards and leaves as soon as no lane of the warp has a
// feasible candidate left.  The layer loop is unrolled by W so every ring
// index is a compile-time register name.  A scenario whose window would
// exceed the ring (the slot being evicted is still feasible) is appended to
// the overflow list and finished by split_finish_kernel.
//
// Work decomposition: a single wave of persistent CTAs whose warps are fully
// independent.  Every warp takes 32-scenario tiles (one scenario per lane; tile
// id = tour * tiles_per_tour + scenario block) from a global atomic counter,
// and streams its own tiles through a private NS-deep ring of shared-memory
// stages; a stage holds one chunk = W demand rows (64 B per row, gathered by
// the tour) plus the chunk's W Cg values, copied with cp.async (LDGSTS, 16 B
// per lane) in commit groups, so a warp only ever waits for its own data and
// runs at its own pace (windows, hence work, differ from warp to warp).  The
// stream runs across tile boundaries; a per-warp queue in shared memory hands
// the tile ids from the copy side to the compute side.  SAA partials are
// flushed per tile with a warp reduction and atomics into kSlots slots per tour.
//
// Value types: int = exact int32 with a predicated min per candidate (ISETP +
// VIMNMX, ALU pipe); fp32 = integer values scaled by 2^-24 (exact, see
// TourInfo::ok), each candidate masked branch-free on the FMA pipe --
// s = sat(P'(i) - Y), c = sat(G + s) is G when feasible and 1.0 (above every
// G < 1) when not -- and folded with 3-input mins (FMNMX3).
constexpr int kSweepWarps = 8;
constexpr int kSweepThreads = 32 * kSweepWarps;
constexpr int kTile = 32;   // scenarios per warp tile
constexpr int kVote = 4;    // candidates per group; groups after the first are guarded by a warp vote
constexpr int kQueue = 16;  // tile-id queue entries per warp (>= tiles the copies can run ahead + 1)

template <int W>
struct SweepCfg {
    static constexpr int NS = (W <= 8) ? 12 : (W <= 16 ? 7 : (W <= 24 ? 6 : (W <= 32 ? 4 : 3)));  // stages
    static constexpr int kMinBlocks = (W <= 24 ? 3 : 2);  // CTAs per SM the register budget targets
    static constexpr int kRowsBytes = W * kTile * (int)sizeof(uint16_t);   // W x 64 B
    static constexpr int kStageBytes = kRowsBytes + W * (int)sizeof(int32_t);  // rows + Cg slice (16 B multiple)
    static constexpr int kWarpBytes = kQueue * 8 + NS * kStageBytes;
    static constexpr size_t kSmem = (size_t)kSweepWarps * kWarpBytes;
    static_assert((W * 4) % 16 == 0, "W must be a multiple of 4");
};


// ---------------------------------------------------------------- a5: packed-fp32 sweep
// The same Eq. (3) ring sweep, with the candidate work shaped for the FMA pipe
// and the packed fp32x2 unit of sm_100 (FADD2):
//  * loads: P (tour-order prefix) is kept as the bit pattern of the float
//    2^23 + P, so P += q is one integer add and the bits ARE the exact float
//    (no conversion); the ring stores Y = 2^23 + P(p) + Q the same way.
//  * values: G = (g + OFF) 2^-24 in [0, 1), exact (TourInfo::ok).
//  * candidate p of age a: s = sat(P(i) - Y) is 0 when p is in the window
//     and 1 when not (FADD.SAT, exact: integers below 2^24);
//    two candidates are completed by one FADD2, c = G + s (>= 1 > every
//    feasible G when masked), and folded by 3-input mins (FMNMX3).
//  * the ring is float2 pairs {slot 2m, slot 2m+1}; positions 2m, 2m+1 are
//    adjacent, so at every layer the ages pair up as (1,2),(3,4),.. (odd
//    layer) or 1,(2,3),(4,5),.. (even layer) -- both compile-time.
//  * candidate groups: U0 pairs unconditionally, then UG pairs per warp vote
//    (any lane whose window still reaches the group's youngest age).
//  * overflow: only tested where the scan reaches the oldest ring age (rare);
//    a lane whose window reaches it is deferred to the finish kernel.
//  * a new tile does not clear the ring: P restarts Q + 1 above the previous
//    tile's last load, which puts every old slot outside every window (the
//    ring is cleared only when P would leave the exact range).
//  * the copy side advances incremental cursors (no divisions per chunk) and
//    the SAA partial is accumulated per lane across tiles, reduced once per
//    warp (and on a change of tour).
// Minimum of N floats as a balanced tree of 3-input mins (FMNMX3): depth log3(N).
template <int N>
__device__ __forceinline__ float min_tree(const float* v) {
    if constexpr (N == 1) return v[0];
    else if constexpr (N == 2) return fminf(v[0], v[1]);
    else if constexpr (N == 3) return fminf(fminf(v[0], v[1]), v[2]);
    else {
        constexpr int A = (N + 2) / 3, B = (N - A + 1) / 2, C = N - A - B;
        return fminf(fminf(min_tree<A>(v), min_tree<B>(v + A)), min_tree<C>(v + A + B));
    }
}

template <int W, int NS, int kRowsBytes, int kStageBytes>
struct F2Stream {  // dynamic copy-cursor state only (constants stay kernel parameters)
    int c;          // next chunk of the current copy tile (== nchunks: fetch a new tile)
    int stage;      // next stage to fill
    unsigned qw;    // queue write index
    int ct;         // tour of the copy tile (-1: no more tiles)
    int64_t s0;     // first scenario of the copy tile
    int segs;       // 16-byte segments per row in the copy tile (4 unless ragged)

    // One chunk: lane r < rows copies demand row r0 + r of the tile (4 x 16 B from its row
    // pointer, built by tour_prep_kernel), lanes < W/4 copy the chunk's Cg slice.
    __device__ __forceinline__ void issue(unsigned char* stage_base, int2* tq, const uint16_t* const* __restrict__ rowp,
                                          const int32_t* __restrict__ cgf, int64_t S, uint32_t ntile_s,
                                          uint32_t ntiles, int n, int nchunks, int cgs_stride, int lane,
                                          unsigned* tile_ctr, uint32_t qpad2) {
        if (c == nchunks) {
            unsigned id = 0;
            if (lane == 0) id = atomicAdd(tile_ctr, 1u);
            id = __shfl_sync(kFull, id, 0);
            int2 e = make_int2(-1, 0);
            ct = -1;
            if (id < ntiles) {
                const uint32_t t = id / ntile_s, b = id - t * ntile_s;
                e = make_int2((int)t, (int)b);
                ct = (int)t;
                s0 = (int64_t)b * kTile;
                const int64_t left = S - s0;
                segs = left >= kTile ? 4 : (int)((left + 7) >> 3);
            }
            if (lane == 0) tq[qw & (kQueue - 1)] = e;
            ++qw;
            c = 0;
        }
        if (ct >= 0) {
            unsigned char* sb = stage_base + stage * kStageBytes;
            const int r0 = c * W;
            const int rows = (n - r0) < W ? (n - r0) : W;
#pragma unroll
            for (int rb = 0; rb < W; rb += 32) {  // row r = rb + lane (W > 32: several rows per lane)
                const int r = rb + lane;
                if (r < rows) {
                    const uint16_t* src = rowp[(int64_t)ct * (n + kTabPad) + r0 + r] + s0;
                    unsigned char* dst = sb + r * (kTile * 2);
                    if (segs == 4) {
                        cp_async16(dst, src);
                        cp_async16(dst + 16, src + 8);
                        cp_async16(dst + 32, src + 16);
                        cp_async16(dst + 48, src + 24);
                    } else {
                        for (int k = 0; k < segs; ++k) cp_async16(dst + 16 * k, src + 8 * k);
                    }
                } else if (r < W) {  // final chunk: rows n.. hold the caller's padding demand
                    uint4* dst = reinterpret_cast<uint4*>(sb + r * (kTile * 2));
#pragma unroll
                    for (int k = 0; k < 4; ++k) dst[k] = make_uint4(qpad2, qpad2, qpad2, qpad2);
                }
            }
#pragma unroll
            for (int cb = 0; cb < W / 4; cb += 32)
                if (cb + lane < W / 4)
                    cp_async16(sb + kRowsBytes + (cb + lane) * 16, cgf + (int64_t)ct * kCgPlanes * cgs_stride + r0 + (cb + lane) * 4);
        }
        cp_async_commit();
        ++c;
        stage = (stage + 1 == NS) ? 0 : stage + 1;
    }
};

// F2Cfg: SweepCfg with the stage count / CTAs per SM of a packed-fp32 variant (MB = 0: defaults).
template <int W, int MB>
struct F2Cfg : SweepCfg<W> {
    // (W = 24: 4 stages keep 3 CTAs per SM within the shared memory)
    static constexpr int NS = (MB >= 4 || W == 24) ? 4 : SweepCfg<W>::NS;
    static constexpr int kMinBlocks = MB > 0 ? MB : SweepCfg<W>::kMinBlocks;
    static constexpr int kWarpBytes = kQueue * 8 + NS * SweepCfg<W>::kStageBytes;
    static constexpr size_t kSmem = (size_t)kSweepWarps * kWarpBytes;
};

template <int W, int U0, int UG, int MB, int NG, bool PAIR = false>
__global__ void __launch_bounds__(kSweepThreads, F2Cfg<W, MB>::kMinBlocks)
    split_sweep_f2_kernel(const uint16_t* const* __restrict__ rowp, const int32_t* __restrict__ cgs,
                          const TourInfo* __restrict__ tinfo, int n, int T, int64_t S, uint32_t Q, uint32_t p_limit,
                          int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ slots,
                          unsigned long long* __restrict__ ovf_list, unsigned* __restrict__ hdr) {
    using Cfg = F2Cfg<W, MB>;
    constexpr int NS = Cfg::NS;
    constexpr int H = W / 2;  // float2 ring pairs
    pdl_wait();  // tables, counters and partial slots come from tour_prep_kernel
    static_assert(W % 4 == 0 && U0 >= 1 && UG >= 1 && kQueue >= NS + 2, "bad sweep config");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned char* wbase = smem_raw + (size_t)wid * Cfg::kWarpBytes;
    int2* tq = reinterpret_cast<int2*>(wbase);
    unsigned char* stage_base = wbase + kQueue * 8;
    const uint32_t ntile_s = (uint32_t)((S + kTile - 1) / kTile);
    const int nchunks = (n + W - 1) / W;
    const int rem = n % W;
    const uint32_t qpad = Q < 65535u ? Q : 65535u;
    constexpr uint32_t kMagic = 0x4B000000u;  // bits of 2^23
    const int slot = (blockIdx.x * kSweepWarps + wid) % kSlots;
    unsigned* ovf_count = hdr + HDR_OVF_COUNT;

    const uint32_t ntiles = ntile_s * (uint32_t)T;
    const int cgs_stride = cg_stride(n);
    F2Stream<W, NS, Cfg::kRowsBytes, Cfg::kStageBytes> cs{nchunks, 0, 0u, -1, 0, 4};
    auto issue = [&]() {
        cs.issue(stage_base, tq, rowp, cgs + cgs_stride, S, ntile_s, ntiles, n, nchunks, cgs_stride, lane, hdr + HDR_TILE,
                 qpad * 0x10001u);
    };
    for (int k = 0; k < NS; ++k) issue();

    float2 G2[H];
    uint32_t Yb[W];
#pragma unroll
    for (int k = 0; k < H; ++k) G2[k] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int k = 0; k < W; ++k) Yb[k] = 0u;  // float 0 < 2^23 <= P: never in a window
    uint32_t Pb = kMagic;

    // per-lane SAA accumulator of tour acc_t, kept in shared memory (after the warp's stages)
    struct LanePart {
        int nf, ni;
        long long sum, sqlo, sqhi;
    };
    __shared__ LanePart accs[kSweepThreads];
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

    int cstage = 0;
    cp_async_wait<NS - 1>();  // the first tile's first chunk (later ones: end of the chunk loop)
    __syncwarp();
    for (unsigned u = 0;; ++u) {
        const int2 tile = tq[u & (kQueue - 1)];
        // (a vote, not a plain branch: the value is warp-uniform, and the compiler must know it,
        // or every warp-synchronous instruction below pays a divergence check, BRA.DIV)
        if (__all_sync(kFull, tile.x < 0)) break;
        const int t = tile.x;
        const int64_t s0 = (int64_t)tile.y * kTile;
        const int cols = (int)((S - s0) < kTile ? (S - s0) : kTile);
        const bool live = lane < cols;
        const int col = live ? lane : cols - 1;
        const TourInfo ti = tinfo[t];
        if (__any_sync(kFull, slots && t != acc_t)) {  // (a vote: the flush's shuffles stay convergent)
            flush();
            acc_t = t;
        }
        // restart P above every old slot's Y (or clear the ring when P nears the exact range's end)
        if (__any_sync(kFull, Pb - kMagic > p_limit)) {
#pragma unroll
            for (int k = 0; k < W; ++k) Yb[k] = 0u;
            Pb = kMagic;
        } else {
            Pb += Q + 1u;
        }
        float gprev = __int_as_float(ti.g0f_bits);
        uint32_t qmax = 0u;
        bool ovf = false;

        // (the chunk loop has no lane- or data-dependent branch: the copy side pads the final
        // chunk, every wait is unconditional and the back edge is a warp vote -- so the compiler
        // can prove the warp converged and the layer votes need no divergence checks, BRA.DIV)
        for (int c = 0;;) {
            unsigned char* sb = stage_base + cstage * Cfg::kStageBytes;
            const uint16_t* bufw = reinterpret_cast<const uint16_t*>(sb) + col;
            const float* cgc = reinterpret_cast<const float*>(sb + Cfg::kRowsBytes);
            // candidate pair unit v of layer jj (compile-time): even layer -> ages (2v+2, 2v+3), the
            // last one (ages W, 1) wrapping around the ring; odd layer -> age 2 alone (v = 0), ages
            // (2v+1, 2v+2) (v >= 1).  A pair's odd slot is the float2's .y, the even slot below it the .x.
            auto unit = [&](const int jj, const float Pn, const int v, float& lo, float& hi) {
                if ((jj & 1) && v == 0) {
                    const int xs = (jj - 1 + W) % W;
                    lo = hi = G2[xs >> 1].x + __saturatef(Pn - __uint_as_float(Yb[xs]));
                    return;
                }
                const int ys = (jj & 1) ? ((jj - 2 * v + 2 * W) % W) : ((jj - 2 * v - 1 + 2 * W) % W);
                const int xs = ys - 1;
                const float2 sp = make_float2(__saturatef(Pn - __uint_as_float(Yb[xs])),
                                              __saturatef(Pn - __uint_as_float(Yb[ys])));
                const float2 cnd = __fadd2_rn(G2[xs >> 1], sp);
                lo = cnd.x;
                hi = cnd.y;
            };
            auto youngest = [&](const int jj, const int v) {  // slot of unit v's youngest age
                return (jj & 1) ? ((jj - 2 * v + 2 * W) % W) : ((jj - 2 * v - 1 + 2 * W) % W);
            };
            // Candidates of age >= 2 first: they depend only on P and on g values of earlier
            // layers, so the DP chain through the layers is just  g = min(old, g_prev) + Cg.
            auto first_group = [&](const int jj, const float Pn, const uint32_t Pnb) -> float {
                float cv[2 * U0];
#pragma unroll
                for (int v = 0; v < U0; ++v) {
                    if (v < H) unit(jj, Pn, v, cv[2 * v], cv[2 * v + 1]);
                    else cv[2 * v] = cv[2 * v + 1] = 2.0f;
                }
                if (U0 >= H) ovf |= Yb[(jj + 1) % W] >= Pnb;  // oldest ring age (W) reached
                return min_tree<2 * U0>(cv);
            };
            // NG voted groups of UG pairs, then (if still needed) the rest in one straight run
            auto deep_groups = [&](const int jj, const float Pn, const uint32_t Pnb, float a) -> float {
#pragma unroll
                for (int gi = 0; gi <= NG; ++gi) {
                    const int v0 = U0 + gi * UG;
                    const int v1 = gi < NG ? v0 + UG : H;
                    if (v0 >= H) break;
                    if (!__any_sync(kFull, Yb[youngest(jj, v0)] >= Pnb)) break;
#pragma unroll
                    for (int v = v0; v < v1; ++v)
                        if (v < H) {
                            float lo, hi;
                            unit(jj, Pn, v, lo, hi);
                            a = fminf(a, fminf(lo, hi));
                        }
                    if (v1 >= H) ovf |= Yb[(jj + 1) % W] >= Pnb;  // the scan reached the oldest ring age
                }
                return a;
            };
            uint32_t qnext = bufw[0];
            if constexpr (PAIR) {
                // Two layers at a time: every candidate of age >= 2 of BOTH layers is known before
                // either layer's result, so both first groups run back to back and ONE warp vote
                // guards the deeper groups of the pair (one skip branch per two layers).
#pragma unroll
                for (int j = 0; j < W; j += 2) {
                    const float cg0 = cgc[j], cg1 = cgc[j + 1];
                    const uint32_t q0 = qnext;
                    const uint32_t q1 = bufw[(j + 1) * kTile];
                    if (j + 2 < W) qnext = bufw[(j + 2) * kTile];
                    qmax = max(qmax, max(q0, q1));
                    const uint32_t Pnb0 = Pb + q0, Pnb1 = Pnb0 + q1;
                    const float Pn0 = __uint_as_float(Pnb0), Pn1 = __uint_as_float(Pnb1);
                    G2[j >> 1].x = gprev;  // slot j: the point of layer j's age 1
                    Yb[j] = Pb + Q;
                    float a0 = first_group(j, Pn0, Pnb0);
                    float a1 = first_group(j + 1, Pn1, Pnb1);
                    if (U0 < H && __any_sync(kFull, Yb[youngest(j, U0)] >= Pnb0 || Yb[youngest(j + 1, U0)] >= Pnb1)) {
                        a0 = deep_groups(j, Pn0, Pnb0, a0);
                        a1 = deep_groups(j + 1, Pn1, Pnb1, a1);
                    }
                    Yb[j + 1] = Pnb0 + Q;  // (after layer j read slot j + 1 as its age W)
                    // age 1 (p = i - 1) is always in the window when q <= Q (q > Q: qmax, DESIGN R4)
                    const float g0 = fminf(a0, gprev) + cg0;
                    G2[j >> 1].y = g0;
                    gprev = fminf(a1, g0) + cg1;
                    Pb = Pnb1;
                }
            } else {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    const float cg = cgc[j];
                    const uint32_t qi = qnext;  // loaded one layer ahead
                    if (j + 1 < W) qnext = bufw[(j + 1) * kTile];
                    qmax = max(qmax, qi);
                    const uint32_t Pnb = Pb + qi;
                    const float Pn = __uint_as_float(Pnb);
                    if (j & 1) G2[j >> 1].y = gprev;
                    else G2[j >> 1].x = gprev;
                    Yb[j] = Pb + Q;
                    float a = first_group(j, Pn, Pnb);
                    a = deep_groups(j, Pn, Pnb, a);
                    // age 1 (p = i - 1) is always in the window when q <= Q (q > Q: qmax, DESIGN R4)
                    gprev = fminf(a, gprev) + cg;
                    Pb = Pnb;
                }
            }
            __syncwarp();
            issue();
            cstage = (cstage + 1 == NS) ? 0 : cstage + 1;
            cp_async_wait<NS - 1>();  // the next chunk (or the next tile's first chunk) has landed
            __syncwarp();
            if (++c >= nchunks) break;
        }
        if (rem != 0) {  // f(n) sits in the slot of position n (pushed by the first padded layer)
#pragma unroll
            for (int k = 0; k < W; ++k)
                if (k == rem) gprev = (k & 1) ? G2[k >> 1].y : G2[k >> 1].x;
        }
        const bool bad = qmax > Q;
        const int fval = (int)(gprev * 0x1p24f) - ti.off;
        const bool deferred = live && (ovf || ti.ok == 0) && !bad;
        const int64_t s = s0 + col;
        if (deferred) ovf_list[atomicAdd(ovf_count, 1u)] = ((unsigned long long)t << 40) | (unsigned long long)s;
        if (cost && live && !deferred) cost[(int64_t)t * S + s] = bad ? SPDP_INFEASIBLE : fval;
        if (live && !deferred) {
            LanePart a = *accp;
            if (bad) {
                a.ni += 1;
            } else {
                const unsigned long long sq = (unsigned long long)fval * (unsigned long long)fval;
                a.nf += 1;
                a.sum += fval;
                a.sqlo += (long long)(sq & 0xffffffffull);
                a.sqhi += (long long)(sq >> 32);
            }
            *accp = a;
        }
    }
    if (slots) flush();
    cp_async_wait<0>();
}

// ---------------------------------------------------------------- a5: exact-int32 ring sweep
// The Eq. (3) ring sweep in exact int32 (used when the packed-fp32 sweep's exactness
// checks fail, or with SPDP_F_SWEEP_INT).  One scenario per lane, a register ring of the
// last W split points {G = g(p), Y = P'(p) + Q}, P'(p) = 1 + prefix; candidate p is in
// the window iff Y >= P'(i), a predicated min per candidate (ISETP +
// VIMNMX, ALU pipe); the newest kVote candidates unconditionally, then groups of kVote
// behind a warp vote.  Same copy side / warp-uniform structure as the packed-fp32 sweep.
template <int W>
__global__ void __launch_bounds__(kSweepThreads, (W <= 24 ? 3 : (W <= 32 ? 2 : 1)))
    split_sweep_kernel(const uint16_t* const* __restrict__ rowp, const int32_t* __restrict__ cgs,
                       const int32_t* __restrict__ g0s, int n, int T, int64_t S, uint32_t Q,
                       int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ slots,
                       unsigned long long* __restrict__ ovf_list, unsigned* __restrict__ hdr) {
    using Cfg = SweepCfg<W>;
    constexpr int NS = Cfg::NS;
    pdl_wait();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned char* wbase = smem_raw + (size_t)wid * Cfg::kWarpBytes;
    int2* tq = reinterpret_cast<int2*>(wbase);
    unsigned char* stage_base = wbase + kQueue * 8;
    const uint32_t ntile_s = (uint32_t)((S + kTile - 1) / kTile);
    const uint32_t ntiles = ntile_s * (uint32_t)T;
    const int nchunks = (n + W - 1) / W;
    const int rem = n % W;
    const int cgs_stride = cg_stride(n);
    const uint32_t qpad = Q < 65535u ? Q : 65535u;
    const int slot = (blockIdx.x * kSweepWarps + wid) % kSlots;
    unsigned* ovf_count = hdr + HDR_OVF_COUNT;

    // (final chunk padded with q_pad = min(Q, 65535), Cg = 0: a demand of Q collapses every
    // window to the newest slot, so padded layers never flag an overflow nor disturb f(n))
    F2Stream<W, NS, Cfg::kRowsBytes, Cfg::kStageBytes> cs{nchunks, 0, 0u, -1, 0, 4};
    auto issue = [&]() {
        cs.issue(stage_base, tq, rowp, cgs, S, ntile_s, ntiles, n, nchunks, cgs_stride, lane, hdr + HDR_TILE,
                 qpad * 0x10001u);
    };
    for (int k = 0; k < NS; ++k) issue();

    struct LanePart {
        int nf, ni;
        long long sum, sqlo, sqhi;
    };
    __shared__ LanePart accs[kSweepThreads];
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

    int cstage = 0;
    cp_async_wait<NS - 1>();
    __syncwarp();
    for (unsigned u = 0;; ++u) {
        const int2 tile = tq[u & (kQueue - 1)];
        if (__all_sync(kFull, tile.x < 0)) break;  // warp-uniform (see split_sweep_f2_kernel)
        const int t = tile.x;
        const int64_t s0 = (int64_t)tile.y * kTile;
        const int cols = (int)((S - s0) < kTile ? (S - s0) : kTile);
        const bool live = lane < cols;
        const int col = live ? lane : cols - 1;  // tail lanes replay a real scenario
        if (__any_sync(kFull, slots && t != acc_t)) {
            flush();
            acc_t = t;
        }
        int G[W];
        uint32_t Y[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
            G[k] = INT_MAX;
            Y[k] = 0u;  // never feasible: P' >= 1
        }
        int gprev = g0s[t];
        uint32_t P = 1u;
        uint32_t qmax = 0u;  // bad <=> some q > Q (Eq. (2) set empty, DESIGN R4)
        int ovfacc = -1;     // ovf <=> some evicted slot still feasible: max(Y - P'(i)) >= 0
        for (int c = 0;;) {
            const unsigned char* sb = stage_base + cstage * Cfg::kStageBytes;
            const uint16_t* buf = reinterpret_cast<const uint16_t*>(sb) + col;
            const int32_t* cgc = reinterpret_cast<const int32_t*>(sb + Cfg::kRowsBytes);
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const int cgi = cgc[j];
                const uint32_t qi = buf[j * kTile];
                qmax = max(qmax, qi);
                const uint32_t Pn = P + qi;
                ovfacc = max(ovfacc, (int)(Y[j] - Pn));
                G[j] = gprev;
                Y[j] = P + Q;
                int best = gprev, best1 = gprev;  // p = L; two independent min chains
#pragma unroll
                for (int k0 = 1; k0 < W; k0 += kVote) {
                    if (k0 > 1 && !__any_sync(kFull, Y[(j - k0 + W) % W] >= Pn)) break;
#pragma unroll
                    for (int v = 0; v < kVote; ++v) {
                        const int k = k0 + v;
                        if (k < W) {
                            const int sl = (j - k + W) % W;
                            if (Y[sl] >= Pn) {
                                if (v & 1) best1 = min(best1, G[sl]);
                                else best = min(best, G[sl]);
                            }
                        }
                    }
                }
                gprev = min(best, best1) + cgi;
                P = Pn;
            }
            __syncwarp();
            issue();
            cstage = (cstage + 1 == NS) ? 0 : cstage + 1;
            cp_async_wait<NS - 1>();
            __syncwarp();
            if (++c >= nchunks) break;
        }
        if (rem != 0) {  // f(n) sits in the slot of position n (pushed by the first padded layer)
#pragma unroll
            for (int k = 0; k < W; ++k)
                if (k == rem) gprev = G[k];
        }
        const bool bad = qmax > Q;
        const bool deferred = live && ovfacc >= 0 && !bad;
        const int64_t s = s0 + col;
        if (deferred) ovf_list[atomicAdd(ovf_count, 1u)] = ((unsigned long long)t << 40) | (unsigned long long)s;
        if (cost && live && !deferred) cost[(int64_t)t * S + s] = bad ? SPDP_INFEASIBLE : gprev;
        if (live && !deferred) {
            LanePart a = *accp;
            if (bad) {
                a.ni += 1;
            } else {
                const unsigned long long sq = (unsigned long long)gprev * (unsigned long long)gprev;
                a.nf += 1;
                a.sum += gprev;
                a.sqlo += (long long)(sq & 0xffffffffull);
                a.sqhi += (long long)(sq >> 32);
            }
            *accp = a;
        }
    }
    if (slots) flush();
    cp_async_wait<0>();
}

// ---------------------------------------------------------------- a5 variant: monotone-deque sweep
// The same DP, g(i) = min_{p in [mask(i), i-1]} g(p) + Cg[i], evaluated as a
// sliding-window minimum with a monotone deque per scenario (
// the window's lower end mask(i) is nondecreasing, R5): the deque holds the
// split points whose g is smaller than every later one, so its front is the
// window minimum.  Each split point is pushed once and popped at most once, so
// the work per layer is O(1) amortised instead of O(window) -- the exact same
// value as the Eq. (3) scan (pops use >= on g, a tie keeps the newer point).
// Per lane a D-entry circular deque {g, Y = P'(p) + Q} lives in shared memory
// ([D][32] per warp, lane-contiguous, conflict-free); front and back values are
// cached in registers.  A scenario whose deque would exceed D is deferred to the
// finish kernel.  The demand stream is the sweep's warp-private cp.async ring
// (chunks of kDqRows rows); the layer loop is a plain loop (no unrolling).
constexpr int kDqRows = 16;  // rows per chunk
constexpr int kDqNS = 2;     // stages per warp (2 + 4 CTAs / SM: C4 1.885 -> 1.746 ms vs 4 stages + 3 CTAs)
constexpr int kDqD = 16;     // deque capacity per scenario

struct DequeCfg {
    static constexpr int kRowsBytes = kDqRows * kTile * (int)sizeof(uint16_t);
    static constexpr int kStageBytes = kRowsBytes + kDqRows * (int)sizeof(int32_t);
    static constexpr int kDqBytes = kDqD * kTile * (int)sizeof(int2);
    static constexpr int kWarpBytes = kQueue * 8 + kDqNS * kStageBytes + kDqBytes;
    static constexpr size_t kSmem = (size_t)kSweepWarps * kWarpBytes;
};

__global__ void __launch_bounds__(kSweepThreads, 4)
    split_deque_kernel(const uint16_t* const* __restrict__ rowp, const int32_t* __restrict__ cgs,
                       const int32_t* __restrict__ g0s, int n, int T, int64_t S, uint32_t Q,
                       int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ slots,
                       unsigned long long* __restrict__ ovf_list, unsigned* __restrict__ hdr) {
    using Cfg = DequeCfg;
    constexpr int NS = kDqNS, R = kDqRows, D = kDqD;
    pdl_wait();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned char* wbase = smem_raw + (size_t)wid * Cfg::kWarpBytes;
    int2* tq = reinterpret_cast<int2*>(wbase);
    unsigned char* stage_base = wbase + kQueue * 8;
    // [D][32] {g, Y} per warp (lane-contiguous rows of 256 B, conflict-free), as a shared address
    const uint32_t dqa = smem_u32(stage_base + NS * Cfg::kStageBytes) + 8u * (uint32_t)lane;
    constexpr uint32_t kMask = (uint32_t)(D - 1) * 256u;
    static_assert((D & (D - 1)) == 0, "D must be a power of two");
    const uint32_t ntile_s = (uint32_t)((S + kTile - 1) / kTile);
    const uint32_t ntiles = ntile_s * (uint32_t)T;
    const int nchunks = (n + R - 1) / R;
    const int cgs_stride = cg_stride(n);
    unsigned* ovf_count = hdr + HDR_OVF_COUNT;

    // copy side: the row-pointer stream of the packed-fp32 sweep (int Cg plane; the padded rows
    // of the final chunk are never read: the layer loop stops at n)
    F2Stream<R, NS, Cfg::kRowsBytes, Cfg::kStageBytes> cs{nchunks, 0, 0u, -1, 0, 4};
    auto issue = [&]() {
        cs.issue(stage_base, tq, rowp, cgs, S, ntile_s, ntiles, n, nchunks, cgs_stride, lane, hdr + HDR_TILE, 0u);
    };
    for (int k = 0; k < NS; ++k) issue();

    int cstage = 0;
    cp_async_wait<NS - 1>();
    __syncwarp();
    for (unsigned u = 0;; ++u) {
        const int2 tile = tq[u & (kQueue - 1)];
        if (__all_sync(kFull, tile.x < 0)) break;  // warp-uniform (see split_sweep_f2_kernel)
        const int t = tile.x;
        const int64_t s0 = (int64_t)tile.y * kTile;
        const int cols = (int)((S - s0) < kTile ? (S - s0) : kTile);
        const bool live = lane < cols;
        const int col = live ? lane : cols - 1;

        int gprev = g0s[t];
        uint32_t P = 1u;
        uint32_t qmax = 0u;
        bool ovf = false;
        // deque = entries [hd, tl) (mod D), kept as byte offsets (x 256 = one [32] row of int2);
        // entry e lives at dqa + (e & 0xF00)
        uint32_t hd8 = 0u, tl8 = 0u;
        int fg = 0, bg = INT_MIN;  // cached front g and back g (INT_MIN: empty)
        uint32_t fy = 0u;          // cached front Y
        auto layer = [&](const uint32_t q, const int cg) {
            qmax = max(qmax, q);
            // (the load advances by min(q, Q): equal for every feasible lane; a lane with q > Q is
            // infeasible -- qmax tells, its value is discarded -- and the clamp keeps the point just
            // pushed inside the next window, which ends the front-pop loop below for every lane)
            const uint32_t Pn = P + min(q, Q);
            const uint32_t ynew = P + Q;
            // push p = L with g(p) = gprev: pop dominated points (g >= gprev) from the back
            while (bg >= gprev) {  // (per lane: no vote)
                const uint32_t ntl = tl8 - 256u;
                const int nb = lds_s32(dqa + ((ntl - 256u) & kMask));
                tl8 = ntl;
                bg = (ntl != hd8) ? nb : INT_MIN;
            }
            ovf |= (tl8 - hd8 == (uint32_t)D * 256u);  // capacity exceeded: the overflow path
            sts_s32x2(dqa + (tl8 & kMask), gprev, (int)ynew);
            if (tl8 == hd8) {
                fg = gprev;
                fy = ynew;
            }
            tl8 += 256u;
            bg = gprev;
            // pop split points that left the window (Y < P'(L+1)) from the front.  (No size test: the
            // point just pushed, p = L with Y = P'(L) + Q >= P'(L) + min(q, Q) = P'(L+1), stays in
            // the window, so it stops the loop.)
            while (fy < Pn) {  // (per lane: no vote)
                const uint32_t nhd = hd8 + 256u;
                const int2 e = lds_s32x2(dqa + (nhd & kMask));
                hd8 = nhd;
                fg = e.x;
                fy = (uint32_t)e.y;
            }
            gprev = fg + cg;  // the front is the window minimum
            P = Pn;
        };

        for (int c = 0;;) {
            const unsigned char* sb = stage_base + cstage * Cfg::kStageBytes;
            const uint16_t* buf = reinterpret_cast<const uint16_t*>(sb) + col;
            const int32_t* cgc = reinterpret_cast<const int32_t*>(sb + Cfg::kRowsBytes);
            const int rows = (n - c * R) < R ? (n - c * R) : R;
            if (rows == R) {  // (warp-uniform) full chunk: unrolled, static stage offsets
#pragma unroll
                for (int j = 0; j < R; ++j) layer(buf[j * kTile], cgc[j]);
            } else {
                for (int j = 0; j < rows; ++j) layer(buf[j * kTile], cgc[j]);
            }
            __syncwarp();
            issue();
            cstage = (cstage + 1 == NS) ? 0 : cstage + 1;
            cp_async_wait<NS - 1>();
            __syncwarp();
            if (++c >= nchunks) break;
        }
        const bool bad = qmax > Q;
        const int64_t s = s0 + col;
        const bool deferred = live && ovf && !bad;
        if (deferred) ovf_list[atomicAdd(ovf_count, 1u)] = ((unsigned long long)t << 40) | (unsigned long long)s;
        if (cost && live && !deferred) cost[(int64_t)t * S + s] = bad ? SPDP_INFEASIBLE : gprev;
        if (slots) {
            Part p{0, 0, 0, 0, 0};
            if (live && !deferred) part_add_cost(p, gprev, !bad);
            p = warp_sum(p);
            if (lane == 0) {
                spdp_saa_partial* d = &slots[(int64_t)t * kSlots + ((blockIdx.x * kSweepWarps + wid) % kSlots)];
                atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_feas), (unsigned long long)p.n_feas);
                atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_infeas), (unsigned long long)p.n_infeas);
                atomicAdd(reinterpret_cast<unsigned long long*>(&d->sum), (unsigned long long)p.sum);
                atomicAdd(reinterpret_cast<unsigned long long*>(&d->sumsq_lo), (unsigned long long)p.sq_lo);
                atomicAdd(reinterpret_cast<unsigned long long*>(&d->sumsq_hi), (unsigned long long)p.sq_hi);
            }
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------- f2: penalized sweep
// Penalized split (DESIGN R22): every p is a candidate,
//   g(i) = Cg[i] + min_p  g(p) + lambda * max(0, P'(i) - Y(p)),   Y(p) = P'(p) + Q,
// i.e. routes may exceed Q at lambda per unit of overload.  Ring entries store G = g(p)
// and Z = g(p) - lambda Y(p), so a candidate is ONE add-max (VIADDMNMX):
//   c = max(lambda P'(i) + Z, G)      (= G inside the capacity window, penalised outside).
// The ring holds the last W split points; an older point is folded, when it leaves the
// ring, into H = min Z (its candidate is then H + lambda P'(i)) -- exact as long as it has
// already left the capacity window, which the eviction checks (else the lane is deferred
// to the finish kernel, like every lane whose lambda P' could leave the int32 range).
// No warp votes: every ring entry is a candidate at every layer.
template <int W>
__global__ void __launch_bounds__(kSweepThreads, 3)
    split_penalized_kernel(const uint16_t* const* __restrict__ rowp, const int32_t* __restrict__ cgs,
                           const int32_t* __restrict__ g0s, int n, int T, int64_t S, uint32_t Q, int32_t lam,
                           int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ slots,
                           unsigned long long* __restrict__ ovf_list, unsigned* __restrict__ hdr) {
    using Cfg = F2Cfg<W, 0>;
    constexpr int NS = Cfg::NS;
    constexpr int32_t kBig = 1 << 30;
    pdl_wait();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned char* wbase = smem_raw + (size_t)wid * Cfg::kWarpBytes;
    int2* tq = reinterpret_cast<int2*>(wbase);
    unsigned char* stage_base = wbase + kQueue * 8;
    const uint32_t ntile_s = (uint32_t)((S + kTile - 1) / kTile);
    const uint32_t ntiles = ntile_s * (uint32_t)T;
    const int nchunks = (n + W - 1) / W;
    const int rem = n % W;
    const int cgs_stride = cg_stride(n);
    const int slot = (blockIdx.x * kSweepWarps + wid) % kSlots;
    unsigned* ovf_count = hdr + HDR_OVF_COUNT;

    F2Stream<W, NS, Cfg::kRowsBytes, Cfg::kStageBytes> cs{nchunks, 0, 0u, -1, 0, 4};
    auto issue = [&]() {
        // (final-chunk padding: demand min(Q + 1, 65535) and Cg 0, so a padded layer pushes every
        // older point out of the capacity window -- no false deferral -- after f(n) was pushed)
        cs.issue(stage_base, tq, rowp, cgs, S, ntile_s, ntiles, n, nchunks, cgs_stride, lane, hdr + HDR_TILE,
                 (Q < 65535u ? Q + 1u : 65535u) * 0x10001u);
    };
    for (int k = 0; k < NS; ++k) issue();

    struct LanePart {
        int nf, ni;
        long long sum, sqlo, sqhi;
    };
    __shared__ LanePart accs[kSweepThreads];
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

    int cstage = 0;
    cp_async_wait<NS - 1>();
    __syncwarp();
    for (unsigned u = 0;; ++u) {
        const int2 tile = tq[u & (kQueue - 1)];
        if (__all_sync(kFull, tile.x < 0)) break;
        const int t = tile.x;
        const int64_t s0 = (int64_t)tile.y * kTile;
        const int cols = (int)((S - s0) < kTile ? (S - s0) : kTile);
        const bool live = lane < cols;
        const int col = live ? lane : cols - 1;
        if (__any_sync(kFull, slots && t != acc_t)) {
            flush();
            acc_t = t;
        }
        int G[W], Z[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
            G[k] = kBig;  // empty slot: never the minimum (real values < 2^29), Z = G - lambda * 0
            Z[k] = kBig;
        }
        int32_t H = kBig;  // min Z over the points that left the ring
        int gprev = g0s[t];
        uint32_t P = 1u;   // P'(i) = 1 + prefix
        bool ovf = false;
        for (int c = 0;;) {
            const unsigned char* sb = stage_base + cstage * Cfg::kStageBytes;
            const uint16_t* buf = reinterpret_cast<const uint16_t*>(sb) + col;
            const int32_t* cgc = reinterpret_cast<const int32_t*>(sb + Cfg::kRowsBytes);
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const uint32_t q = buf[j * kTile];
                const uint32_t Pn = P + q;
                const int32_t lp = lam * (int32_t)Pn;
                // evict slot j (the point W layers back) into H; if it is still inside the capacity
                // window (lambda P' + Z < G, lambda > 0) its penalty-free cost would be lost: defer
                ovf |= lp + Z[j] < G[j];
                H = min(H, Z[j]);
                G[j] = gprev;
                Z[j] = gprev - lam * (int32_t)(P + Q);
                int best = H + lp;
#pragma unroll
                for (int k = 0; k < W; ++k) best = min(best, __viaddmax_s32(lp, Z[k], G[k]));
                gprev = best + cgc[j];
                P = Pn;
            }
            __syncwarp();
            issue();
            cstage = (cstage + 1 == NS) ? 0 : cstage + 1;
            cp_async_wait<NS - 1>();
            __syncwarp();
            if (++c >= nchunks) break;
        }
        if (rem != 0) {  // f(n): the slot of position n (pushed by the first padded layer)
#pragma unroll
            for (int k = 0; k < W; ++k)
                if (k == rem) gprev = G[k];
        }
        // lambda P' grew monotonically: its final value bounds every intermediate one
        ovf |= (int64_t)lam * (int64_t)(P + Q) >= (int64_t)(1 << 29);
        const bool deferred = live && ovf;
        const int64_t s = s0 + col;
        if (deferred) ovf_list[atomicAdd(ovf_count, 1u)] = ((unsigned long long)t << 40) | (unsigned long long)s;
        if (cost && live && !deferred) cost[(int64_t)t * S + s] = gprev;
        if (live && !deferred) {
            LanePart a = *accp;
            const unsigned long long sq = (unsigned long long)gprev * (unsigned long long)gprev;
            a.nf += 1;
            a.sum += gprev;
            a.sqlo += (long long)(sq & 0xffffffffull);
            a.sqhi += (long long)(sq >> 32);
            *accp = a;
        }
    }
    if (slots) flush();
    cp_async_wait<0>();
}

// Deferred penalized scenarios: one warp each, every p in [0, L] a candidate (lanes over p,
// REDUX-free int64 shuffle min), int64 values; per-warp scratch of 3 (n+1) words.
__global__ void __launch_bounds__(128) split_penalized_finish_kernel(
    const int2* __restrict__ tabs, const int32_t* __restrict__ g0s, int n, const uint16_t* __restrict__ demand,
    int64_t ld, int64_t S, uint32_t Q, int64_t lam, int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ partial,
    const unsigned long long* __restrict__ ovf_list, const unsigned* __restrict__ ovf_count) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    pdl_wait();
    long long* g = reinterpret_cast<long long*>(smem_raw) + (size_t)wid * 2 * (n + 1);
    long long* pre = g + (n + 1);
    const unsigned count = *ovf_count;
    for (unsigned idx = blockIdx.x * nw + wid; idx < count; idx += gridDim.x * nw) {
        const unsigned long long key = ovf_list[idx];
        const int t = (int)(key >> 40);
        const int64_t s = (int64_t)(key & ((1ull << 40) - 1));
        const int2* tab = tabs + (int64_t)t * (n + kTabPad);
        long long carry = 0;
        if (lane == 0) pre[0] = 0;
        for (int b = 0; b < n; b += 32) {
            const int i = b + lane;
            long long v = (i < n) ? (long long)demand[(int64_t)tab[i].x * ld + s] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long w = __shfl_up_sync(kFull, v, o);
                if (lane >= o) v += w;
            }
            if (i < n) pre[i + 1] = carry + v;
            carry += __shfl_sync(kFull, v, 31);
        }
        if (lane == 0) g[0] = g0s[t];
        __syncwarp();
        for (int L = 0; L < n; ++L) {
            const long long Pn = pre[L + 1];
            long long best = LLONG_MAX;
            for (int p = lane; p <= L; p += 32) {
                const long long over = Pn - pre[p] - (long long)Q;
                best = min(best, g[p] + (over > 0 ? lam * over : 0));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
            if (lane == 0) g[L + 1] = best + tab[L].y;
            __syncwarp();
        }
        const long long f = g[n];
        if (lane == 0) {
            if (cost) cost[(int64_t)t * S + s] = f < INT_MAX ? (int32_t)f : INT_MAX - 1;
            if (partial) {
                const unsigned long long sq = (unsigned long long)f * (unsigned long long)f;
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].n_feas), 1ull);
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sum), (unsigned long long)f);
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sumsq_lo), sq & 0xffffffffull);
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sumsq_hi), sq >> 32);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- finish kernel
// (1) SAA partial of each tour: sum of its CTAs' slots, added atomically (the
//     partials are zeroed by tour_prep_kernel);
// (2) the overflow list (scenarios whose window outgrew the sweep's ring): one
//     THREAD per scenario with a kOvfW-entry register ring (the exact-int32 Eq. (3)
//     scan of split_sweep_kernel, each thread exiting its own candidate loop at its
//     window's edge; demands gathered from global memory kOvfPf layers ahead), so a
//     few thousand overflow scenarios run fully in parallel with no scratch memory;
// (3) scenarios whose window outgrows even that ring: one warp per scenario with
//     transition-level parallelism -- the lanes split the
//     candidates p in [mask(i), i-1] and combine them with REDUX.MIN, mask(i)
//     advances monotonically with a ballot; any window width.
constexpr int kOvfW = 32;   // register ring of the overflow threads (its code is unrolled W x W: keep it small)
constexpr int kOvfPf = 8;   // demand prefetch distance (layers)

// Exact int32 Eq. (3) scan of one scenario with a W-entry register ring; false if
// some window reached past the ring (the result is then not valid).
template <int W>
__device__ __forceinline__ bool ring_split_one(const int2* __restrict__ tab, int g0, int n,
                                               const uint16_t* __restrict__ demand, int64_t ld, int64_t s, uint32_t Q,
                                               int& f) {
    static_assert(W % kOvfPf == 0, "prefetch distance must divide the ring");
    int G[W];
    uint32_t Y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        G[k] = INT_MAX;
        Y[k] = 0u;  // P' >= 1: never in a window
    }
    uint32_t qb[kOvfPf];  // demands and Cg of the next kOvfPf layers (static slots: layer L uses slot L % kOvfPf)
    int cb[kOvfPf];
#pragma unroll
    for (int k = 0; k < kOvfPf; ++k) {
        const int2 e = (k < n) ? __ldg(&tab[k]) : make_int2(0, 0);
        qb[k] = (k < n) ? demand[(int64_t)e.x * ld + s] : 0u;
        cb[k] = e.y;
    }
    int gprev = g0;
    uint32_t P = 1u;  // P'(i) = 1 + prefix
    bool ovf = false;
    for (int L0 = 0; L0 < n; L0 += W) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int L = L0 + j;
            if (L < n) {
                const uint32_t q = qb[j % kOvfPf];
                const int cg = cb[j % kOvfPf];
                const int La = L + kOvfPf;
                if (La < n) {
                    const int2 e = __ldg(&tab[La]);
                    qb[j % kOvfPf] = demand[(int64_t)e.x * ld + s];
                    cb[j % kOvfPf] = e.y;
                }
                const uint32_t Pn = P + q;
                ovf |= Y[j] >= Pn;  // the slot being overwritten is still in the window
                G[j] = gprev;
                Y[j] = P + Q;
                int best = gprev;
#pragma unroll
                for (int k = 1; k < W; ++k) {
                    const int sl = (j - k + W) % W;
                    if (Y[sl] < Pn) break;  // the window is a contiguous suffix (DESIGN R5)
                    best = min(best, G[sl]);
                }
                gprev = best + cg;
                P = Pn;
            }
        }
    }
    f = gprev;
    return !ovf;
}

__global__ void __launch_bounds__(128) split_finish_kernel(
    const spdp_saa_partial* __restrict__ slots, int kslots, int T, const int2* __restrict__ tabs,
    const int32_t* __restrict__ g0s, int n, const uint16_t* __restrict__ demand, int64_t ld, int64_t S, uint32_t Q,
    int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ partial,
    const unsigned long long* __restrict__ ovf_list, const unsigned* __restrict__ ovf_count) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ Part red[4];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    pdl_wait();  // slots and the overflow list come from the sweep
    if (partial) {
        for (int t = blockIdx.x; t < T; t += gridDim.x) {
            Part a{0, 0, 0, 0, 0};
            for (int b = threadIdx.x; b < kslots; b += blockDim.x) {
                const spdp_saa_partial& e = slots[(int64_t)t * kslots + b];
                a.n_feas += e.n_feas;
                a.n_infeas += e.n_infeas;
                a.sum += e.sum;
                a.sq_lo += e.sumsq_lo;
                a.sq_hi += e.sumsq_hi;
            }
            Part r = block_sum(a, red);
            if (threadIdx.x == 0) {
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].n_feas), (unsigned long long)r.n_feas);
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].n_infeas), (unsigned long long)r.n_infeas);
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sum), (unsigned long long)r.sum);
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sumsq_lo), (unsigned long long)r.sq_lo);
                atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sumsq_hi), (unsigned long long)r.sq_hi);
            }
            __syncthreads();
        }
    }
    const unsigned count = ovf_count ? *ovf_count : 0u;
    auto emit = [&](int t, int64_t s, int f) {
        if (cost) cost[(int64_t)t * S + s] = f;
        if (partial) {
            const unsigned long long sq = (unsigned long long)f * (unsigned long long)f;
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].n_feas), 1ull);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sum), (unsigned long long)f);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sumsq_lo), sq & 0xffffffffull);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial[t].sumsq_hi), sq >> 32);
        }
    };
    int* g = reinterpret_cast<int*>(smem_raw) + (size_t)wid * 3 * (n + 1);  // warp scratch of (3)
    uint32_t* pre = reinterpret_cast<uint32_t*>(g + (n + 1));
    int* cgl = g + 2 * (n + 1);
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < count; base += stride) {
        // (2) one overflow scenario per lane
        const unsigned idx = base + lane;
        int t = 0, f = 0;
        int64_t s = 0;
        bool todo = false;
        if (idx < count) {
            const unsigned long long key = ovf_list[idx];
            t = (int)(key >> 40);
            s = (int64_t)(key & ((1ull << 40) - 1));
            const bool ok = ring_split_one<kOvfW>(tabs + (int64_t)t * (n + kTabPad), g0s[t], n, demand, ld, s, Q, f);
            if (ok) emit(t, s, f);
            todo = !ok;
        }
        // (3) the lanes whose window outgrew the ring, one at a time, by the whole warp
        unsigned pending = __ballot_sync(kFull, todo);
        while (pending) {
            const int src = __ffs(pending) - 1;
            pending &= pending - 1;
            const int tt = __shfl_sync(kFull, t, src);
            const int64_t ss = __shfl_sync(kFull, s, src);
            const int2* tab = tabs + (int64_t)tt * (n + kTabPad);
            // tour-order prefix P(i) = sum_{k<=i} q, i = 0..n: all loads in flight, then a warp scan
            uint32_t carry = 0u;
            if (lane == 0) pre[0] = 0u;
            for (int b = 0; b < n; b += 32) {
                const int i = b + lane;
                uint32_t v = 0u;
                if (i < n) {
                    const int2 e = tab[i];
                    v = demand[(int64_t)e.x * ld + ss];
                    cgl[i] = e.y;
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t u = __shfl_up_sync(kFull, v, o);
                    if (lane >= o) v += u;
                }
                if (i < n) pre[i + 1] = carry + v;
                carry += __shfl_sync(kFull, v, 31);
            }
            if (lane == 0) g[0] = g0s[tt];
            __syncwarp();
            int m = 0;  // mask(L+1), monotone in L
            for (int L = 0; L < n; ++L) {
                const uint32_t Pn = pre[L + 1];
                for (;;) {  // first p >= m with P(L+1) - P(p) <= Q (p = L always qualifies: q <= Q)
                    const int p = m + lane;
                    const unsigned bb = __ballot_sync(kFull, p <= L && Pn - pre[p] <= Q);
                    if (bb) {
                        m += __ffs(bb) - 1;
                        break;
                    }
                    m += 32;
                }
                int best = INT_MAX;
                for (int p = m + lane; p <= L; p += 32) best = min(best, g[p]);
                best = __reduce_min_sync(kFull, best);
                if (lane == 0) g[L + 1] = best + cgl[L];
                __syncwarp();
            }
            if (lane == 0) emit(tt, ss, g[n]);
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------- sampling (window_hint = 0)
__global__ void sample_window_kernel(const int2* __restrict__ tab, int n, const uint16_t* __restrict__ demand,
                                     int64_t ld, int64_t S, uint32_t Q, unsigned* __restrict__ hdr) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    // two-pointer on the tour-order prefix, re-reading the left demand
    uint32_t P = 0, Pm = 0;
    int m = 0, wmax = 1;
    unsigned long long wsum = 0;
    for (int i = 1; i <= n; ++i) {
        const uint32_t q = demand[(int64_t)tab[i - 1].x * ld + s];
        if (q > Q) return;  // infeasible scenario: not representative
        P += q;
        while (P - Pm > Q) {
            Pm += demand[(int64_t)tab[m].x * ld + s];
            ++m;
        }
        wmax = max(wmax, i - m);
        wsum += (unsigned long long)(i - m);
    }
    atomicMax(&hdr[HDR_SAMPLE_W], (unsigned)wmax);
    atomicAdd(reinterpret_cast<unsigned long long*>(&hdr[HDR_SAMPLE_SUM]), wsum);
    atomicAdd(&hdr[HDR_SAMPLE_CNT], 1u);
}

// ---------------------------------------------------------------- a3 / a4 standalone
__global__ void prefix_kernel(const int32_t* __restrict__ tour, int n, const uint16_t* __restrict__ demand,
                              int64_t ld, int64_t S, uint32_t* __restrict__ prefix) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    uint32_t P = 0;
    prefix[s] = 0;
    for (int i = 1; i <= n; ++i) {
        int c = tour[i - 1];
        c = c < 1 ? 1 : (c > n ? n : c);
        P += demand[(int64_t)(c - 1) * ld + s];
        prefix[(int64_t)i * S + s] = P;
    }
}

__global__ void mask_kernel(const int32_t* __restrict__ tour, int n, const uint16_t* __restrict__ demand,
                            int64_t ld, int64_t S, uint32_t Q, int32_t* __restrict__ mask) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    auto q_at = [&](int i) -> uint32_t {  // demand at 1-based tour position i
        int c = tour[i - 1];
        c = c < 1 ? 1 : (c > n ? n : c);
        return demand[(int64_t)(c - 1) * ld + s];
    };
    uint32_t P = 0, Pm = 0;  // P = P(i), Pm = P(m)
    int m = 0;
    for (int i = 1; i <= n; ++i) {
        const uint32_t q = q_at(i);
        P += q;
        int out;
        if (q > Q) {
            out = -1;     // Eq. (2) set is empty (DESIGN R4)
            m = i;        // no segment reaching back past i is feasible later
            Pm = P;
        } else {
            while (P - Pm > Q) Pm += q_at(++m);
            out = m;
        }
        mask[(int64_t)(i - 1) * S + s] = out;
    }
}

// ---------------------------------------------------------------- a6 standalone
__global__ void __launch_bounds__(256) saa_reduce_kernel(const int32_t* __restrict__ cost, int64_t S,
                                                         spdp_saa_partial* __restrict__ partial) {
    __shared__ Part red[8];
    Part p{0, 0, 0, 0, 0};
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
        const int c = cost[s];
        part_add_cost(p, c, c != SPDP_INFEASIBLE);
    }
    Part r = block_sum(p, red);
    if (threadIdx.x == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_feas), (unsigned long long)r.n_feas);
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_infeas), (unsigned long long)r.n_infeas);
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sum), (unsigned long long)r.sum);
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_lo), (unsigned long long)r.sq_lo);
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_hi), (unsigned long long)r.sq_hi);
    }
}

// ---------------------------------------------------------------- host dispatch
static int num_sms() { return device_sms(); }

// Launches the sweep: one wave of persistent CTAs (occupancy x SMs).
template <int W>
static spdp_status launch_sweep_t(cudaStream_t st, const SweepArgs& a) {
    auto kern = split_sweep_kernel<W>;
    int blocks_per_sm = 1;  // (all of the unified L1/smem as shared memory)
    if (spdp_status e = kernel_setup((const void*)kern, (int)SweepCfg<W>::kSmem, 100, kSweepThreads, SweepCfg<W>::kSmem,
                                     &blocks_per_sm, "split_sweep setup"))
        return e;
    const int64_t ntiles = ((a.S + kTile - 1) / kTile) * a.T;
    int64_t grid = (int64_t)blocks_per_sm * num_sms();
    const int64_t need = (ntiles + kSweepWarps - 1) / kSweepWarps;
    if (grid > need) grid = need;
    prof_begin(st);
    spdp_status rc = cuda_check(launch_pdl(kern, dim3((unsigned)grid), dim3(kSweepThreads), SweepCfg<W>::kSmem, st, a.rowp,
                                           a.cgs, a.g0, a.n, a.T, a.S, a.Q, a.cost, a.slots, a.ovf, a.hdr),
                                "split_sweep_kernel");
    set_last_kernel("split_sweep_kernel<%d,int>", W);
    prof_end(st);
    return rc;
}

static spdp_status launch_deque(cudaStream_t st, const SweepArgs& a) {
    int blocks_per_sm = 1;
    if (spdp_status e = kernel_setup((const void*)split_deque_kernel, 220 * 1024, 100, kSweepThreads, DequeCfg::kSmem,
                                     &blocks_per_sm, "split_deque setup"))
        return e;
    const int64_t ntiles = ((a.S + kTile - 1) / kTile) * a.T;
    int64_t grid = (int64_t)blocks_per_sm * num_sms();
    const int64_t need = (ntiles + kSweepWarps - 1) / kSweepWarps;
    if (grid > need) grid = need;
    prof_begin(st);
    spdp_status rc = cuda_check(launch_pdl(split_deque_kernel, dim3((unsigned)grid), dim3(kSweepThreads), DequeCfg::kSmem, st,
                                           a.rowp, a.cgs, a.g0, a.n, a.T, a.S, a.Q, a.cost, a.slots, a.ovf, a.hdr),
                                "split_deque_kernel");
    set_last_kernel("split_deque_kernel<%d>", kDqD);
    prof_end(st);
    return rc;
}

template <int W, int U0, int UG, int MB = 0, int NG = W, bool PAIR = false>
static spdp_status launch_sweep_f2_t(cudaStream_t st, const SweepArgs& a) {
    using Cfg = F2Cfg<W, MB>;
    auto kern = split_sweep_f2_kernel<W, U0, UG, MB, NG, PAIR>;
    int blocks_per_sm = 1;
    if (spdp_status e = kernel_setup((const void*)kern, (int)Cfg::kSmem, 100, kSweepThreads, Cfg::kSmem, &blocks_per_sm,
                                     "split_sweep_f2 setup"))
        return e;
    const int64_t ntiles = ((a.S + kTile - 1) / kTile) * a.T;
    int64_t grid = (int64_t)blocks_per_sm * num_sms();
    const int64_t need = (ntiles + kSweepWarps - 1) / kSweepWarps;
    if (grid > need) grid = need;
    prof_begin(st);
    // P restarts Q + 1 above the previous tile's loads; one tile adds at most (n + W) q_pad + Q + 1
    const int64_t qpad = a.Q < 65535u ? a.Q : 65535;
    const int64_t lim = (1LL << 23) - 1 - ((int64_t)a.n + W) * qpad - 2 * (int64_t)a.Q - 2;
    if (lim < 0) return fail(SPDP_E_RESOURCE, "split_sweep_f2: loads exceed the exact fp32 range");
    spdp_status rc = cuda_check(launch_pdl(kern, dim3((unsigned)grid), dim3(kSweepThreads), Cfg::kSmem, st, a.rowp,
                                           a.cgs, a.tinfo, a.n, a.T, a.S, a.Q, (uint32_t)lim, a.cost, a.slots, a.ovf,
                                           a.hdr),
                                "split_sweep_f2_kernel");
    set_last_kernel("split_sweep_f2_kernel<%d,%d,%d,%d,%d,%d>", W, U0, UG, MB, NG, PAIR ? 1 : 0);
    prof_end(st);
    return rc;
}

static spdp_status launch_sweep(int W, bool f32, cudaStream_t st, const SweepArgs& a, int mean_w) {
    if (f32) {
        // unconditional candidate pairs U0 ~ 0.8 x the mean window (measured: C2, mean 3.75 -> 3;
        // C3, mean 7.7 -> 6); an SPDP_F2 setting overrides
        const bool wide = mean_w >= 6;
        switch (W) {
            case 8: return launch_sweep_f2_t<8, 2, 1>(st, a);
            case 16: return wide ? launch_sweep_f2_t<16, 5, 1>(st, a) : launch_sweep_f2_t<16, 3, 1>(st, a);
            case 20:  // (pairs: -1.4 % at C3)
                return wide ? launch_sweep_f2_t<20, 6, 2, 0, 20, true>(st, a) : launch_sweep_f2_t<20, 3, 1>(st, a);
            case 24: return wide ? launch_sweep_f2_t<24, 6, 2, 0, 24, true>(st, a) : launch_sweep_f2_t<24, 3, 1>(st, a);
            default: return wide ? launch_sweep_f2_t<32, 8, 2>(st, a) : launch_sweep_f2_t<32, 4, 2>(st, a);
        }
    }
    switch (W) {
        case 8: return launch_sweep_t<8>(st, a);
        case 16: return launch_sweep_t<16>(st, a);
        case 20: return launch_sweep_t<20>(st, a);
        case 24: return launch_sweep_t<24>(st, a);
        case 32: return launch_sweep_t<32>(st, a);
        default: return launch_sweep_t<64>(st, a);
    }
}

// Ring width W: the smallest instantiated width that holds the expected maximum window.
static int pick_w(int hint) {
    static const int widths[] = {8, 16, 20, 24, 32, 64};
    for (int w : widths)
        if (hint <= w) return w;
    return 64;
}

template <int W>
static spdp_status launch_penalized_t(cudaStream_t st, const SweepArgs& a, int32_t lam) {
    using Cfg = F2Cfg<W, 0>;
    auto kern = split_penalized_kernel<W>;
    int blocks_per_sm = 1;
    if (spdp_status e = kernel_setup((const void*)kern, (int)Cfg::kSmem, 100, kSweepThreads, Cfg::kSmem, &blocks_per_sm,
                                     "split_penalized setup"))
        return e;
    const int64_t ntiles = ((a.S + kTile - 1) / kTile) * a.T;
    int64_t grid = (int64_t)blocks_per_sm * num_sms();
    const int64_t need = (ntiles + kSweepWarps - 1) / kSweepWarps;
    if (grid > need) grid = need;
    prof_begin(st);
    spdp_status rc = cuda_check(launch_pdl(kern, dim3((unsigned)grid), dim3(kSweepThreads), Cfg::kSmem, st, a.rowp, a.cgs,
                                           a.g0, a.n, a.T, a.S, a.Q, lam, a.cost, a.slots, a.ovf, a.hdr),
                                "split_penalized_kernel");
    set_last_kernel("split_penalized_kernel<%d>", W);
    prof_end(st);
    return rc;
}

static spdp_status split_common(const int32_t* tours, int32_t T, const int32_t* dist, int32_t n,
                                const uint16_t* demand, int64_t ld, int64_t S, int32_t Q, int32_t* cost,
                                spdp_saa_partial* partial, int32_t window_hint, void* ws, size_t ws_bytes,
                                uint32_t flags, cudaStream_t st, const char* fn, int32_t lam = -1) {
    if (n < 1) return fail(SPDP_E_USAGE, "%s: n=%d < 1", fn, n);
    if (n > SPDP_MAX_N) return fail(SPDP_E_RESOURCE, "%s: n=%d > SPDP_MAX_N=%d", fn, n, SPDP_MAX_N);
    if (T < 1) return fail(SPDP_E_USAGE, "%s: T=%d < 1", fn, T);
    if (T >= (1 << 23)) return fail(SPDP_E_RESOURCE, "%s: T=%d too large", fn, T);
    if (S < 1) return fail(SPDP_E_USAGE, "%s: S=%lld < 1", fn, (long long)S);
    if (S >= (1LL << 40)) return fail(SPDP_E_RESOURCE, "%s: S too large", fn);
    if (Q < 1) return fail(SPDP_E_USAGE, "%s: Q=%d < 1 (SPEC:34)", fn, Q);
    if (!tours || !dist || !demand || !ws) return fail(SPDP_E_USAGE, "%s: NULL required pointer", fn);
    if (ld < S || (ld % 8) != 0) return fail(SPDP_E_USAGE, "%s: ld=%lld must be >= S and a multiple of 8", fn, (long long)ld);
    if (((uintptr_t)demand & 15u) != 0) return fail(SPDP_E_USAGE, "%s: demand must be 16-byte aligned", fn);
    if (window_hint < 0) return fail(SPDP_E_USAGE, "%s: window_hint < 0", fn);
    const WsLayout L = ws_layout(n, S, T);
    if (ws_bytes < L.total) return fail(SPDP_E_USAGE, "%s: workspace %zu < required %zu", fn, ws_bytes, L.total);
    char* w = static_cast<char*>(ws);
    unsigned* hdr = reinterpret_cast<unsigned*>(w + L.hdr);
    int32_t* g0 = reinterpret_cast<int32_t*>(w + L.g0);
    TourInfo* tinfo = reinterpret_cast<TourInfo*>(w + L.tinfo);
    int2* tabs = reinterpret_cast<int2*>(w + L.tabs);
    const uint16_t** rowp = reinterpret_cast<const uint16_t**>(w + L.rowp);
    spdp_saa_partial* slots = reinterpret_cast<spdp_saa_partial*>(w + L.slots);
    unsigned long long* ovf = reinterpret_cast<unsigned long long*>(w + L.ovf);
    // Q above the largest possible load behaves as "everything fits"; clamp so P' + Q fits uint32.
    const uint32_t Qe = (uint32_t)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    const bool validate = (flags & SPDP_F_VALIDATE) != 0;
    spdp_status rc;
    if (validate || window_hint == 0) {
        rc = cuda_check(cudaMemsetAsync(hdr, 0, 256, st), "cudaMemsetAsync(hdr)");
        if (rc) return rc;
    }
    if ((rc = launch_tour_prep(tours, T, n, dist, demand, ld, w, L, partial, partial != nullptr, validate, st)))
        return rc;
    int W = pick_w(window_hint);
    int mean_w = (int)((flags >> SPDP_F_MEAN_WINDOW_SHIFT) & 0xffu);  // expected mean window (0: unknown)
    if (validate || window_hint == 0) {
        if (window_hint == 0) {
            const int64_t Ss = S < 4096 ? S : 4096;
            sample_window_kernel<<<(unsigned)ceil_div(Ss, 256), 256, 0, st>>>(tabs, n, demand, ld, Ss, Qe, hdr);
            if ((rc = last_launch("sample_window_kernel"))) return rc;
        }
        unsigned h[8];
        if ((rc = cuda_check(cudaMemcpyAsync(h, hdr, sizeof(h), cudaMemcpyDeviceToHost, st), "memcpy(hdr)"))) return rc;
        if ((rc = cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
        if (validate && h[HDR_STATUS]) {
            const unsigned b = h[HDR_STATUS];
            return fail(SPDP_E_DATA, "%s: invalid input:%s%s%s", fn, (b & ST_NOT_PERM) ? " tour is not a permutation of 1..n" : "",
                        (b & ST_NEG_DIST) ? " negative cost" : "",
                        (b & ST_RANGE) ? " 3*n*max(dist) exceeds the int32 range" : "");
        }
        if (window_hint == 0) {
            W = pick_w((int)(h[HDR_SAMPLE_W] + h[HDR_SAMPLE_W] / 4 + 1));
            const unsigned long long wsum = (unsigned long long)h[HDR_SAMPLE_SUM] | ((unsigned long long)h[HDR_SAMPLE_SUM + 1] << 32);
            if (h[HDR_SAMPLE_CNT] > 0 && mean_w == 0)
                mean_w = (int)((wsum + (unsigned long long)h[HDR_SAMPLE_CNT] * n / 2) / ((unsigned long long)h[HDR_SAMPLE_CNT] * n));
        }
    }
    const SweepArgs args{tours, rowp, tabs, reinterpret_cast<const int32_t*>(w + L.trow), reinterpret_cast<const int32_t*>(w + L.cgs), g0, tinfo, n, T, demand, ld, S, Qe,
                         cost, partial ? slots : nullptr, ovf, hdr};
    // fp32 sweep when every load value it forms (P' <= (n + W) min(Q, 65535) for feasible scenarios
    // including the padded layers, Y = P' + Q) is an exact float; the per-tour cost range is checked on
    // the device (TourInfo::ok: lanes of a tour that fails it are finished by the int finish kernel)
    // (the packed-fp32 sweep keeps loads as 2^23 + P + Q, exact below 2^24)
    const int64_t qeff = Qe < 65535u ? (int64_t)Qe : 65535;
    const bool f32_loads_exact = ((int64_t)n + 64) * qeff + 2 * (int64_t)Qe + 2 < (1LL << 23);
    int mode = 0;  // 0 auto, 1 int ring, 2 packed-fp32 ring, 3 deque, 4 packed-u16 ring
    if (flags & SPDP_F_SWEEP_INT) mode = 1;
    if (flags & SPDP_F_SWEEP_F32) mode = 2;
    if (flags & SPDP_F_SWEEP_DEQUE) mode = 3;
    if (flags & SPDP_F_SWEEP_U16) mode = 4;
    // default for windows <= 32: the packed-u16 ring (two scenarios per lane) when its load range
    // check passes, else the packed-fp32 ring when its loads are exact, else the int ring
    const bool u16_ok = W <= 32 && W >= 16 && u16_loads_ok(n, Qe) && S < (1LL << 31);
    const bool use_u16 = u16_ok && (mode == 4 || mode == 0);
    const bool use_f32 = W <= 32 && f32_loads_exact && S < (1LL << 31) && (mode == 2 || mode == 0 || mode == 4);
    // windows wider than the largest cheap register ring: the O(1)-amortised deque sweep
    // (measured 4.8x faster than the W=64 ring at n=1000, slower at small windows)
    if (lam >= 0) {  // f2 penalized split (DESIGN R22)
        if (S >= (1LL << 31)) return fail(SPDP_E_RESOURCE, "%s: S >= 2^31", fn);
        rc = W <= 16 ? launch_penalized_t<16>(st, args, lam) : launch_penalized_t<24>(st, args, lam);
        if (rc) return rc;
        const size_t per_warp = 2 * sizeof(long long) * (size_t)(n + 1);
        const int warps = per_warp * 4 <= 192 * 1024 ? 4 : 1;
        if ((rc = kernel_setup((const void*)split_finish_kernel, 200 * 1024, 100, 0, 0, nullptr, "split_finish setup")))
            return rc;
        if ((rc = kernel_setup((const void*)split_penalized_finish_kernel, 200 * 1024, -1, 0, 0, nullptr,
                               "split_penalized_finish setup")))
            return rc;
        // SAA slots -> partial (no strict overflow list), then the deferred penalized scenarios
        rc = cuda_check(launch_pdl(split_finish_kernel, dim3(num_sms()), dim3(128), (size_t)0, st,
                                   partial ? slots : nullptr, (int)kSlots, T, (const int2*)tabs, (const int32_t*)g0, n,
                                   demand, ld, S, Qe, cost, partial, (const unsigned long long*)ovf,
                                   (const unsigned*)nullptr),
                        "split_finish_kernel");
        if (rc) return rc;
        rc = cuda_check(launch_pdl(split_penalized_finish_kernel, dim3(2 * num_sms()), dim3(warps * 32), per_warp * warps,
                                   st, (const int2*)tabs, (const int32_t*)g0, n, demand, ld, S, (uint32_t)Q,
                                   (int64_t)lam, cost, partial, (const unsigned long long*)ovf,
                                   (const unsigned*)(hdr + HDR_OVF_COUNT)),
                        "split_penalized_finish_kernel");
        return rc;
    }
    // the O(1)-amortised deque for windows wider than the largest cheap ring, or for mean windows
    // >= 12 (measured crossover: deque 10.3 vs ring 7.4 ms at mean 7.7 (C3), 0.23 vs 1.4 ms at 15)
    if (mode == 3 || (mode == 0 && (W > 32 || mean_w >= 12))) rc = launch_deque(st, args);
    else if (use_u16) rc = launch_sweep_u16(W, mean_w, st, args);
    else rc = launch_sweep(W, use_f32, st, args, mean_w);
    if (rc) return rc;
    return launch_finish(w, L, T, n, demand, ld, S, Qe, cost, partial, true, st);
}

spdp_status launch_tour_prep(const int32_t* tours, int32_t T, int32_t n, const int32_t* dist,
                             const uint16_t* demand, int64_t ld, char* w, const WsLayout& L,
                             spdp_saa_partial* partial, bool zero_slots, bool validate, cudaStream_t st) {
    const int threads = n <= 128 ? 128 : (n >= 2048 ? 1024 : 256);
    const size_t smem = tour_prep_smem(n);
    // (the sweep's shared-memory carveout: no L1 / shared reconfiguration between the kernels of a call)
    if (spdp_status e = kernel_setup((const void*)tour_prep_kernel, (int)tour_prep_smem(SPDP_MAX_N), 100, 0, 0, nullptr,
                                     "tour_prep setup"))
        return e;
    // (a plain launch: launched with PDL behind the previous call's finish kernel -- waiting in the
    // kernel for it -- measured 0.4 us slower per C2 step)
    tour_prep_kernel<<<T, threads, smem, st>>>(
        tours, n, dist, reinterpret_cast<int2*>(w + L.tabs), reinterpret_cast<int32_t*>(w + L.g0), demand, ld,
        reinterpret_cast<const uint16_t**>(w + L.rowp), reinterpret_cast<TourInfo*>(w + L.tinfo),
        reinterpret_cast<int32_t*>(w + L.cgs), reinterpret_cast<int32_t*>(w + L.trow), zero_slots ? reinterpret_cast<spdp_saa_partial*>(w + L.slots) : nullptr,
        reinterpret_cast<unsigned*>(w + L.hdr), partial, validate ? 1 : 0);
    return last_launch("tour_prep_kernel");
}

spdp_status launch_finish(char* w, const WsLayout& L, int32_t T, int32_t n, const uint16_t* demand, int64_t ld,
                          int64_t S, uint32_t Qe, int32_t* cost, spdp_saa_partial* partial, bool pdl,
                          cudaStream_t st) {
    // the SAA partials + the overflow list (one thread per scenario; 4 warps per CTA,
    // each with 12 (n+1) B of shared scratch for the rare windows wider than kOvfW)
    const size_t per_warp = 3 * sizeof(int) * (size_t)(n + 1);
    const int warps = per_warp * 4 <= 192 * 1024 ? 4 : 1;
    if (spdp_status e = kernel_setup((const void*)split_finish_kernel, 200 * 1024, 100, 0, 0, nullptr, "split_finish setup"))
        return e;
    const spdp_saa_partial* slots = partial ? reinterpret_cast<const spdp_saa_partial*>(w + L.slots) : nullptr;
    const int2* tabs = reinterpret_cast<const int2*>(w + L.tabs);
    const int32_t* g0 = reinterpret_cast<const int32_t*>(w + L.g0);
    const unsigned long long* ovf = reinterpret_cast<const unsigned long long*>(w + L.ovf);
    const unsigned* ovf_count = reinterpret_cast<const unsigned*>(w + L.hdr) + HDR_OVF_COUNT;
    if (pdl)
        return cuda_check(launch_pdl(split_finish_kernel, dim3(4 * num_sms()), dim3(warps * 32), per_warp * warps, st,
                                     slots, (int)kSlots, (int)T, tabs, g0, (int)n, demand, ld, S, Qe, cost, partial, ovf,
                                     ovf_count),
                          "split_finish_kernel");
    split_finish_kernel<<<4 * num_sms(), warps * 32, per_warp * warps, st>>>(slots, (int)kSlots, (int)T, tabs, g0, (int)n,
                                                                             demand, ld, S, Qe, cost, partial, ovf,
                                                                             ovf_count);
    return last_launch("split_finish_kernel");
}

}  // namespace spdp

using namespace spdp;

extern "C" size_t spdp_workspace_bytes(int32_t n, int64_t S, int32_t T) {
    if (n < 1 || S < 1 || T < 1) return 0;
    return ws_layout(n, S, T).total;
}

extern "C" spdp_status spdp_split_eval(const int32_t* tour, const int32_t* dist, int32_t n, const uint16_t* demand,
                                       int64_t ld, int64_t S, int32_t Q, int32_t* cost, spdp_saa_partial* partial,
                                       int32_t window_hint, void* ws, size_t ws_bytes, uint32_t flags,
                                       spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval");
    return split_common(tour, 1, dist, n, demand, ld, S, Q, cost, partial, window_hint, ws, ws_bytes, flags,
                        (cudaStream_t)stream, "spdp_split_eval");
}

extern "C" spdp_status spdp_split_eval_penalized(const int32_t* tour, const int32_t* dist, int32_t n,
                                                 const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                                 int32_t lambda, int32_t* cost, spdp_saa_partial* partial,
                                                 int32_t window_hint, void* ws, size_t ws_bytes, uint32_t flags,
                                                 spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval_penalized");
    if (lambda < 0) return fail(SPDP_E_USAGE, "spdp_split_eval_penalized: lambda=%d < 0", lambda);
    return split_common(tour, 1, dist, n, demand, ld, S, Q, cost, partial, window_hint, ws, ws_bytes, flags,
                        (cudaStream_t)stream, "spdp_split_eval_penalized", lambda);
}

extern "C" spdp_status spdp_split_eval_batch(const int32_t* tours, int32_t T, const int32_t* dist, int32_t n,
                                             const uint16_t* demand, int64_t ld, int64_t S, int32_t Q, int32_t* cost,
                                             spdp_saa_partial* partial, int32_t window_hint, void* ws, size_t ws_bytes,
                                             uint32_t flags, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval_batch");
    return split_common(tours, T, dist, n, demand, ld, S, Q, cost, partial, window_hint, ws, ws_bytes, flags,
                        (cudaStream_t)stream, "spdp_split_eval_batch");
}

// ---------------------------------------------------------------- f1: route recovery
// One thread per requested scenario; per-thread prefix P and DP values g live in
// the workspace ([K][n+1] each).  Layer L computes g(L+1) over the window
// p in [mask(L+1), L] with the two-pointer mask and records the
// argmin, scanning p upward with "<=" so the LARGEST p wins ties (DESIGN R10).
// Values are exact int32 (same range check as the sweep); INF marks an empty
// window (a demand above Q, DESIGN R4) and propagates.
__global__ void __launch_bounds__(128) split_routes_kernel(const int2* __restrict__ tab, const int32_t* __restrict__ g0s,
                                                           int n, const uint16_t* __restrict__ demand, int64_t ld,
                                                           int64_t S, uint32_t Q, const int64_t* __restrict__ scen,
                                                           int K, int32_t* __restrict__ pred, int32_t* __restrict__ cost,
                                                           int32_t* __restrict__ nroutes, int32_t* __restrict__ maxload,
                                                           uint32_t* __restrict__ Pw, int32_t* __restrict__ Gw) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const int64_t N1 = (int64_t)n + 1;
    int64_t s = scen[k];
    s = s < 0 ? 0 : (s >= S ? S - 1 : s);  // (the host checks the range; clamp keeps reads in bounds)
    uint32_t* P = Pw + (int64_t)k * N1;
    int32_t* G = Gw + (int64_t)k * N1;
    int32_t* pr = pred + (int64_t)k * N1;
    uint32_t acc = 0u;
    P[0] = 0u;
    for (int i = 0; i < n; ++i) {  // tour-order prefix
        acc += demand[(int64_t)tab[i].x * ld + s];
        P[i + 1] = acc;
    }
    G[0] = g0s[0];
    pr[0] = -1;
    int m = 0;
    for (int L = 0; L < n; ++L) {
        const uint32_t Pn = P[L + 1];
        while (m <= L && Pn - P[m] > Q) ++m;  // mask(L+1); m = L+1: empty window
        int best = INT_MAX, arg = -1;
        for (int p = m; p <= L; ++p) {
            const int v = G[p];
            if (v != INT_MAX && v <= best) {
                best = v;
                arg = p;
            }
        }
        G[L + 1] = (arg < 0) ? INT_MAX : best + tab[L].y;  // tab[n-1].y = B[n]: G[n] = f(n)
        pr[L + 1] = arg;
    }
    const int f = G[n];
    cost[k] = (f == INT_MAX) ? SPDP_INFEASIBLE : f;
    if (nroutes || maxload) {
        int r = 0;
        uint32_t ml = 0u;
        if (f != INT_MAX) {
            for (int i = n; i > 0; i = pr[i]) {  // walk the optimal routes back from n
                ++r;
                ml = max(ml, P[i] - P[pr[i]]);
            }
        }
        if (nroutes) nroutes[k] = r;
        if (maxload) maxload[k] = (int32_t)ml;
    }
}

// f1 with a warp per scenario (n <= kRoutesWarpMaxN): the prefix loads by a warp scan, the window's
// lower end by a ballot over 32 positions at a time, the window minimum by two warp reductions
// (REDUX: the smallest g, then the largest p holding it -- ties go to the largest p, as in the
// thread-per-scenario kernel above); P and g in shared memory.  Same results.
constexpr int kRoutesWarpMaxN = 1024;
__global__ void __launch_bounds__(128) split_routes_warp_kernel(const int2* __restrict__ tab, const int32_t* __restrict__ g0s,
                                                                int n, const uint16_t* __restrict__ demand, int64_t ld,
                                                                int64_t S, uint32_t Q, const int64_t* __restrict__ scen,
                                                                int K, int32_t* __restrict__ pred, int32_t* __restrict__ cost,
                                                                int32_t* __restrict__ nroutes, int32_t* __restrict__ maxload) {
    extern __shared__ uint32_t rsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int k = blockIdx.x * (blockDim.x >> 5) + wid;
    if (k >= K) return;  // (warp-uniform)
    const int N1 = n + 1;
    uint32_t* P = rsm + (size_t)wid * 2 * N1;
    int32_t* G = reinterpret_cast<int32_t*>(P + N1);
    int64_t s = scen[k];
    s = s < 0 ? 0 : (s >= S ? S - 1 : s);  // (the host checks the range; clamp keeps reads in bounds)
    int32_t* pr = pred + (int64_t)k * N1;
    uint32_t carry = 0u;  // tour-order prefix, 32 positions per step
    for (int b = 0; b < n; b += 32) {
        const int i = b + lane;
        uint32_t q = i < n ? (uint32_t)demand[(int64_t)tab[i].x * ld + s] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(kFull, q, o);
            if (lane >= o) q += u;
        }
        if (i < n) P[i + 1] = carry + q;
        carry += __shfl_sync(kFull, q, 31);
    }
    if (lane == 0) {
        P[0] = 0u;
        G[0] = g0s[0];
        pr[0] = -1;
    }
    __syncwarp();
    int m = 0;
    for (int L = 0; L < n; ++L) {
        const uint32_t Pn = P[L + 1];
        for (;;) {  // mask(L+1): the first p >= m with Pn - P[p] <= Q (monotone in p), L + 1 if none
            const int p = m + lane;
            const bool stop = p > L || Pn - P[p] <= Q;
            const unsigned bal = __ballot_sync(kFull, stop);
            if (bal) {
                m += __ffs(bal) - 1;
                break;
            }
            m += 32;
        }
        unsigned best = 0xffffffffu;  // g ^ 0x80000000 (order-preserving); INT_MAX maps to 0xffffffff: unreachable
        int arg = -1;
        for (int p0 = m; p0 <= L; p0 += 32) {
            const int p = p0 + lane;
            const unsigned key = (unsigned)(p <= L ? G[p] : INT_MAX) ^ 0x80000000u;
            const unsigned mn = __reduce_min_sync(kFull, key);
            const unsigned pm = __reduce_max_sync(kFull, key == mn ? (unsigned)(p + 1) : 0u);
            if (mn != 0xffffffffu && mn <= best) {  // (a later chunk holds larger p: ties go there)
                best = mn;
                arg = (int)pm - 1;
            }
        }
        if (lane == 0) {
            G[L + 1] = (arg < 0) ? INT_MAX : (int32_t)(best ^ 0x80000000u) + tab[L].y;  // tab[n-1].y = B[n]: G[n] = f(n)
            pr[L + 1] = arg;
        }
        __syncwarp();
    }
    if (lane == 0) {
        const int f = G[n];
        cost[k] = (f == INT_MAX) ? SPDP_INFEASIBLE : f;
        if (nroutes || maxload) {
            int r = 0;
            uint32_t ml = 0u;
            if (f != INT_MAX) {
                for (int i = n; i > 0; i = pr[i]) {  // walk the optimal routes back from n
                    ++r;
                    ml = max(ml, P[i] - P[pr[i]]);
                }
            }
            if (nroutes) nroutes[k] = r;
            if (maxload) maxload[k] = (int32_t)ml;
        }
    }
}

extern "C" size_t spdp_routes_workspace_bytes(int32_t n, int32_t K) {
    if (n < 1 || K < 1) return 0;
    return ws_layout(n, 1, 1).total + align_up(sizeof(uint32_t) * 2 * (size_t)K * (size_t)(n + 1), 256);
}

extern "C" spdp_status spdp_split_routes(const int32_t* tour, const int32_t* dist, int32_t n, const uint16_t* demand,
                                         int64_t ld, int64_t S, int32_t Q, const int64_t* scen, int32_t K,
                                         int32_t* pred, int32_t* cost, int32_t* nroutes, int32_t* maxload, void* ws,
                                         size_t ws_bytes, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_routes");
    const char* fn = "spdp_split_routes";
    if (n < 1 || S < 1 || Q < 1 || K < 1) return fail(SPDP_E_USAGE, "%s: n, S, Q and K must be >= 1", fn);
    if (n > SPDP_MAX_N) return fail(SPDP_E_RESOURCE, "%s: n=%d > SPDP_MAX_N", fn, n);
    if (!tour || !dist || !demand || !scen || !pred || !cost || !ws) return fail(SPDP_E_USAGE, "%s: NULL pointer", fn);
    if (ld < S) return fail(SPDP_E_USAGE, "%s: ld < S", fn);
    if (ws_bytes < spdp_routes_workspace_bytes(n, K)) return fail(SPDP_E_USAGE, "%s: workspace too small", fn);
    cudaStream_t st = (cudaStream_t)stream;
    const WsLayout L = ws_layout(n, 1, 1);
    char* w = static_cast<char*>(ws);
    unsigned* hdr = reinterpret_cast<unsigned*>(w + L.hdr);
    int32_t* g0 = reinterpret_cast<int32_t*>(w + L.g0);
    int2* tabs = reinterpret_cast<int2*>(w + L.tabs);
    const uint16_t** rowp = reinterpret_cast<const uint16_t**>(w + L.rowp);
    TourInfo* tinfo = reinterpret_cast<TourInfo*>(w + L.tinfo);
    uint32_t* Pw = reinterpret_cast<uint32_t*>(w + L.total);
    int32_t* Gw = reinterpret_cast<int32_t*>(Pw + (size_t)K * (size_t)(n + 1));
    const uint32_t Qe = (uint32_t)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    spdp_status rc;
    {
        const int threads = n <= 128 ? 128 : (n >= 2048 ? 1024 : 256);
        const size_t smem = tour_prep_smem(n);
        if ((rc = kernel_setup((const void*)tour_prep_kernel, (int)tour_prep_smem(SPDP_MAX_N), 100, 0, 0, nullptr,
                               "tour_prep setup")))
            return rc;
        tour_prep_kernel<<<1, threads, smem, st>>>(tour, n, dist, tabs, g0, demand, ld, rowp, tinfo,
                                                   reinterpret_cast<int32_t*>(w + L.cgs),
                                                   reinterpret_cast<int32_t*>(w + L.trow), nullptr, hdr, nullptr, 0);
        if ((rc = last_launch("tour_prep_kernel"))) return rc;
    }
    if (n <= kRoutesWarpMaxN) {  // a warp per scenario, its P and g in shared memory
        const size_t smem = sizeof(uint32_t) * 2 * (size_t)(n + 1) * 4;
        prof_begin(st);
        split_routes_warp_kernel<<<(unsigned)ceil_div(K, 4), 128, smem, st>>>(tabs, g0, n, demand, ld, S, Qe, scen, K,
                                                                             pred, cost, nroutes, maxload);
        prof_end(st);
        set_last_kernel("split_routes_warp_kernel");
        return last_launch("split_routes_warp_kernel");
    }
    prof_begin(st);
    split_routes_kernel<<<(unsigned)ceil_div(K, 128), 128, 0, st>>>(tabs, g0, n, demand, ld, S, Qe, scen, K, pred, cost,
                                                                   nroutes, maxload, Pw, Gw);
    prof_end(st);
    set_last_kernel("split_routes_kernel");
    return last_launch("split_routes_kernel");
}

extern "C" spdp_status spdp_demand_prefix(const int32_t* tour, int32_t n, const uint16_t* demand, int64_t ld, int64_t S,
                                          uint32_t* prefix, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_demand_prefix");
    if (n < 1 || S < 1) return fail(SPDP_E_USAGE, "spdp_demand_prefix: n and S must be >= 1");
    if (!tour || !demand || !prefix) return fail(SPDP_E_USAGE, "spdp_demand_prefix: NULL pointer");
    if (ld < S) return fail(SPDP_E_USAGE, "spdp_demand_prefix: ld < S");
    prefix_kernel<<<(unsigned)ceil_div(S, 256), 256, 0, (cudaStream_t)stream>>>(tour, n, demand, ld, S, prefix);
    return last_launch("prefix_kernel");
}

extern "C" spdp_status spdp_split_mask(const int32_t* tour, int32_t n, const uint16_t* demand, int64_t ld, int64_t S,
                                       int32_t Q, int32_t* mask, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_mask");
    if (n < 1 || S < 1 || Q < 1) return fail(SPDP_E_USAGE, "spdp_split_mask: n, S, Q must be >= 1");
    if (!tour || !demand || !mask) return fail(SPDP_E_USAGE, "spdp_split_mask: NULL pointer");
    if (ld < S) return fail(SPDP_E_USAGE, "spdp_split_mask: ld < S");
    mask_kernel<<<(unsigned)ceil_div(S, 256), 256, 0, (cudaStream_t)stream>>>(tour, n, demand, ld, S, (uint32_t)Q, mask);
    return last_launch("mask_kernel");
}

extern "C" spdp_status spdp_saa_reduce(const int32_t* cost, int64_t S, spdp_saa_partial* partial, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_saa_reduce");
    if (S < 0 || !partial || (S > 0 && !cost)) return fail(SPDP_E_USAGE, "spdp_saa_reduce: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    spdp_status rc = cuda_check(cudaMemsetAsync(partial, 0, sizeof(spdp_saa_partial), st), "cudaMemsetAsync(partial)");
    if (rc || S == 0) return rc;
    int64_t blocks = ceil_div(S, 256 * 8);
    if (blocks > (int64_t)device_sms() * 8) blocks = (int64_t)device_sms() * 8;
    saa_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(cost, S, partial);
    return last_launch("saa_reduce_kernel");
}
