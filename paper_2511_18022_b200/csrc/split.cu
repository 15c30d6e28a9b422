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

namespace spdp {

// ---------------------------------------------------------------- workspace
struct WsLayout {
    size_t hdr, tickets, g0, tabs, tabsf, tinfo, bpart, ovf, total;
    int64_t nblocks;
};

// Per-tour info for the fp32 sweep: g0f = (g(0) + OFF) / 2^24 (float bits),
// off = OFF = D[n] (makes every g(p) + OFF >= 0), ok = every value the fp32
// sweep forms is an integer (times 2^-24) below 2^24, hence exact.
struct TourInfo {
    int32_t g0f_bits, off, ok, pad;
};

constexpr int kSweepThreads = 256;
constexpr int kTabPad = 64;  // padding rows so the prefetch never reads past the table

inline WsLayout ws_layout(int32_t n, int64_t S, int32_t T) {
    WsLayout L;
    size_t off = 0;
    L.nblocks = ceil_div(S, kSweepThreads);
    L.hdr = off; off += 256;
    L.tickets = off; off = align_up(off + sizeof(unsigned) * (size_t)T, 256);
    L.g0 = off; off = align_up(off + sizeof(int32_t) * (size_t)T, 256);
    L.tabs = off; off = align_up(off + sizeof(int2) * (size_t)T * (size_t)(n + kTabPad), 256);
    L.tabsf = off; off = align_up(off + sizeof(int2) * (size_t)T * (size_t)(n + kTabPad), 256);
    L.tinfo = off; off = align_up(off + sizeof(TourInfo) * (size_t)T, 256);
    L.bpart = off; off = align_up(off + sizeof(spdp_saa_partial) * (size_t)T * (size_t)L.nblocks, 256);
    L.ovf = off; off = align_up(off + sizeof(unsigned long long) * (size_t)T * (size_t)S, 256);
    L.total = off;
    return L;
}

// header words
enum { HDR_OVF_COUNT = 0, HDR_STATUS = 1, HDR_SAMPLE_W = 2 };
enum { ST_NOT_PERM = 1, ST_NEG_DIST = 2, ST_RANGE = 4 };

// ---------------------------------------------------------------- a2: tour prep
// One CTA per tour.  tab[i] = {row of customer s_{i+1}, Cg[i]} (0-based layer i
// computes f(i+1)); tab[n-1].y = B[n].  g0[t] = c_{0,s_1}.  D is a block scan.
__global__ void __launch_bounds__(1024) tour_prep_kernel(const int32_t* __restrict__ tours, int n,
                                                         const int32_t* __restrict__ dist,
                                                         int2* __restrict__ tabs, int32_t* __restrict__ g0,
                                                         int2* __restrict__ tabsf, TourInfo* __restrict__ tinfo,
                                                         unsigned* __restrict__ hdr, unsigned* __restrict__ tickets,
                                                         int validate) {
    extern __shared__ unsigned char smem_raw[];
    long long* wsum = reinterpret_cast<long long*>(smem_raw);              // 32 warp sums
    long long* dn = wsum + 32;                                             // D[n]
    int* cmx = reinterpret_cast<int*>(dn + 1);                             // block max of the used costs
    unsigned* seen = reinterpret_cast<unsigned*>(smem_raw + 34 * sizeof(long long));  // bitmap
    const int t = blockIdx.x;
    const int32_t* tour = tours + (int64_t)t * n;
    int2* tab = tabs + (int64_t)t * (n + kTabPad);
    const int64_t N1 = n + 1;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5;

    if (t == 0 && tid == 0) hdr[HDR_OVF_COUNT] = 0u;
    if (tid == 0) {
        tickets[t] = 0u;
        *cmx = 0;
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
    }
    for (int i = n + tid; i < n + kTabPad; i += nt) tab[i] = make_int2(0, 0);
    if (tid == 0) g0[t] = dist[node(0)];
    __syncthreads();
    // fp32 tables: cg / 2^24 (exact: |cg| <= 2 cmax), g0f = (g0 + OFF) / 2^24
    {
        const long long OFF = *dn, cm = *cmx;
        int2* tabf = tabsf + (int64_t)t * (n + kTabPad);
        for (int i = tid; i < n + kTabPad; i += nt) {
            const int2 e = tab[i];
            tabf[i] = make_int2(e.x, __float_as_int((float)e.y * 0x1p-24f));
        }
        if (tid == 0) {
            TourInfo ti;
            ti.g0f_bits = __float_as_int((float)(dist[node(0)] + OFF) * 0x1p-24f);
            ti.off = (int)(OFF < INT_MAX ? OFF : INT_MAX);
            // g + OFF <= (2n + 1) cmax + OFF and f(n) + OFF <= 2 n cmax + OFF: all below 2^24
            ti.ok = ((2LL * n + 2) * cm + OFF < (1LL << 24)) ? 1 : 0;
            ti.pad = 0;
            tinfo[t] = ti;
        }
    }
    // range: |g|, |f| <= 3 n cmax (SURVEY §7 hard part 10)
    if ((long long)cmax * (3LL * n + 1) >= (long long)INT_MAX) bad |= ST_RANGE;
    if (bad) atomicOr(&hdr[HDR_STATUS], bad);
}

// ---------------------------------------------------------------- a5: the sweep
// One scenario per thread, 256 scenarios per CTA.  The candidate ring holds, for
// the last W split points p (slot p mod W): G = g(p) and Y = P'(p) + Q, where
// P'(p) = 1 + sum of the first p tour-order demands.  p is in the Eq. (3)
// window of layer i iff P'(i) - P'(p) <= Q  <=>  Y >= P'(i).
// Because q >= 0 the window is a contiguous suffix (DESIGN R5), so the
// candidate loop walks from the newest slot backwards and leaves as soon as no
// lane of the warp has a feasible candidate left.  The layer loop is unrolled
// by W so every ring index is a compile-time register name.  A scenario whose
// window would exceed the ring (the slot being evicted is still feasible) is
// appended to the overflow list and finished by split_general_kernel.
//
// Demand stream: the CTA's tile [n rows (tour order) x 256 scenarios] is staged
// through shared memory in chunks of W rows by bulk-async copies (the TMA
// engine, one 512-byte copy per row, gathered by the tour) into an NS-deep ring
// of stages guarded by mbarriers, so NS-1 chunks are always in flight while
// the CTA computes on the current one.
template <int W>
struct SweepCfg {
    static constexpr int NS = (W <= 8) ? 6 : (W <= 16 ? 4 : (W <= 32 ? 3 : 2));  // stages
    static constexpr int kStageElems = W * kSweepThreads;                        // u16 per stage
    static constexpr size_t kStageBytes = sizeof(uint16_t) * kStageElems;
    static constexpr int kHdr = 128;  // NS mbarriers (8 B) + NS stage-consumption counters (4 B)
    static size_t smem_bytes(int n) {
        return kHdr + NS * kStageBytes + sizeof(int2) * (size_t)(n + kTabPad);
    }
};

// Value / load types of the two sweep variants.  int: exact int32 with a
// predicated min per candidate (ISETP + VIMNMX on the ALU pipe).  fp32:
// integer-valued floats scaled by 2^-24 (exact, TourInfo::ok), each candidate
// masked branch-free on the FMA pipe -- s = sat(P'(i) - Y), c = sat(G + s) is G
// when feasible and 1.0 (above every G < 1) when not -- and folded with a
// 3-input min (FMNMX3), so the ALU pipe carries half an op per candidate.
template <bool F32>
struct SweepT {
    using V = int;
    using L = uint32_t;
};
template <>
struct SweepT<true> {
    using V = float;
    using L = float;
};

template <int W, int VE, bool F32>
__global__ void __launch_bounds__(kSweepThreads, (W <= 16 ? 4 : 1))
    split_sweep_kernel(const int2* __restrict__ tabs, const int32_t* __restrict__ g0s,
                       const TourInfo* __restrict__ tinfo, int n, const uint16_t* __restrict__ demand,
                       int64_t ld, int64_t S, uint32_t Q, int32_t* __restrict__ cost,
                       spdp_saa_partial* __restrict__ bpart, spdp_saa_partial* __restrict__ partial,
                       unsigned* __restrict__ tickets, unsigned long long* __restrict__ ovf_list,
                       unsigned* __restrict__ ovf_count) {
    using Cfg = SweepCfg<W>;
    using V = typename SweepT<F32>::V;
    using LT = typename SweepT<F32>::L;
    constexpr int NS = Cfg::NS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);                             // NS mbarriers
    unsigned* done = reinterpret_cast<unsigned*>(smem_raw + 64);                       // NS counters
    uint16_t* dbuf = reinterpret_cast<uint16_t*>(smem_raw + Cfg::kHdr);                // NS x W x 256
    int2* stab = reinterpret_cast<int2*>(smem_raw + Cfg::kHdr + NS * Cfg::kStageBytes);  // n + kTabPad
    __shared__ Part red[kSweepThreads / 32];
    __shared__ bool am_last;

    const int t = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t s0 = (int64_t)blockIdx.x * kSweepThreads;
    const int cols = (int)((S - s0) < kSweepThreads ? (S - s0) : kSweepThreads);
    const uint32_t row_bytes = (uint32_t)(((cols + 7) & ~7) * sizeof(uint16_t));
    const int nchunks = (n + W - 1) / W;
    {
        const int2* tab = tabs + (int64_t)t * (n + kTabPad);
        for (int i = tid; i < n + kTabPad; i += kSweepThreads) stab[i] = tab[i];
    }
    if (tid == 0) {
        for (int k = 0; k < NS; ++k) {
            mbar_init(&bar[k], 1);
            done[k] = 0u;
        }
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    // producer: one warp refills stage (c % NS) with chunk c (rows c*W .. c*W+W-1)
    auto issue = [&](int c) {
        const int stage = c % NS;
        const int r0 = c * W;
        const int rows = (n - r0) < W ? (n - r0) : W;
        if (lane == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[stage], row_bytes * (uint32_t)rows);
        }
        __syncwarp();
        for (int r = lane; r < rows; r += 32)
            bulk_g2s(dbuf + (size_t)stage * Cfg::kStageElems + r * kSweepThreads,
                     demand + (int64_t)stab[r0 + r].x * ld + s0, row_bytes, &bar[stage], pol);
    };
    if (wid == 0)
        for (int c = 0; c < NS && c < nchunks; ++c) issue(c);

    const bool live = tid < cols;
    const int col = live ? tid : cols - 1;  // tail lanes replay a real scenario
    const int64_t s = s0 + col;

    V G[W];
    LT Y[W];
    V gprev;
    LT P, Qv;
    bool f32_ok = true;
    if constexpr (F32) {
        const TourInfo ti = tinfo[t];
        f32_ok = ti.ok != 0;
        gprev = __int_as_float(ti.g0f_bits);
        P = 0.0f;
        Qv = (float)Q;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            G[k] = 0.0f;
            Y[k] = -1.0f;  // never feasible: P' >= 0
        }
    } else {
        gprev = g0s[t];
        P = 1u;
        Qv = Q;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            G[k] = INT_MAX;
            Y[k] = 0u;  // never feasible: P' >= 1
        }
    }
    uint32_t qmax = 0u;   // bad  <=> some q > Q  (Eq. (2) set empty, DESIGN R4)
    V ovfacc = (V)-1;     // ovf  <=> some evicted slot still feasible: max(Y - P'(i)) >= 0

    // One layer (computes f(L+1)); j = L mod W is a compile-time constant.
    auto layer = [&](const uint16_t* buf, const int j, const int L) {
        const uint32_t qi = buf[j * kSweepThreads];
        qmax = max(qmax, qi);
        LT Pn;
        if constexpr (F32) {
            Pn = P + __uint2float_rn(qi);
            ovfacc = fmaxf(ovfacc, Y[j] - Pn);
        } else {
            Pn = P + qi;
            ovfacc = max(ovfacc, (int)(Y[j] - Pn));
        }
        G[j] = gprev;
        Y[j] = P + Qv;
        V best = gprev;  // p = L
        if constexpr (F32) {
#pragma unroll
            for (int k0 = 1; k0 < W; k0 += VE) {
                if (!__any_sync(kFull, Y[(j - k0 + W) % W] >= Pn)) break;
                float c[VE];
#pragma unroll
                for (int u = 0; u < VE; ++u) {
                    const int k = k0 + u;
                    const int sl = (j - k + W) % W;
                    c[u] = (k < W) ? __saturatef(G[sl] + __saturatef(Pn - Y[sl])) : 1.0f;
                }
#pragma unroll
                for (int u = 0; u + 1 < VE; u += 2) best = fminf(best, fminf(c[u], c[u + 1]));
                if (VE & 1) best = fminf(best, c[VE - 1]);
            }
            gprev = best + __int_as_float(stab[L].y);
        } else {
            V best1 = best;  // second accumulator: two independent min chains
#pragma unroll
            for (int k = 1; k < W; ++k) {
                const int sl = (j - k + W) % W;
                const bool f = Y[sl] >= Pn;
                if ((k % VE) == 1 % VE && !__any_sync(kFull, f)) break;
                if (f) {
                    if (k & 1) best1 = min(best1, G[sl]);
                    else best = min(best, G[sl]);
                }
            }
            gprev = min(best, best1) + stab[L].y;
        }
        P = Pn;
    };

    // The final chunk is padded to W layers with demand q_pad = min(Q, 65535) and cg = 0:
    // a demand of Q collapses every window to the newest slot, so the padded layers
    // never flag an overflow and never disturb the ring slot that holds f(n).
    const int rem = n % W;
    const uint32_t qpad = Q < 65535u ? Q : 65535u;
    constexpr int NW = kSweepThreads / 32;
    for (int c = 0; c < nchunks; ++c) {
        const int stage = c % NS;
        mbar_wait(&bar[stage], (uint32_t)((c / NS) & 1));
        uint16_t* bufw = dbuf + (size_t)stage * Cfg::kStageElems + col;
        if (rem != 0 && c == nchunks - 1)
            for (int j = rem; j < W; ++j) bufw[j * kSweepThreads] = (uint16_t)qpad;
        const uint16_t* buf = bufw;
        const int i0 = c * W;
#pragma unroll
        for (int j = 0; j < W; ++j) layer(buf, j, i0 + j);
        // release the stage: the last warp to finish it refills it (no CTA-wide barrier,
        // so warps with narrow windows run ahead of warps with wide ones)
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) {
            __threadfence_block();
            last = (atomicAdd(&done[stage], 1u) == NW - 1);
            if (last) done[stage] = 0u;
        }
        last = __shfl_sync(kFull, last, 0);
        if (last && c + NS < nchunks) issue(c + NS);
    }
    // f(n): the slot of position n holds it (pushed by the first padded layer), or gprev if n % W == 0
    if (rem != 0) {
#pragma unroll
        for (int k = 0; k < W; ++k)
            if (k == rem) gprev = G[k];
    }
    const bool bad = qmax > Q;
    const bool ovf = (ovfacc >= (V)0) || !f32_ok;
    int fval;
    if constexpr (F32) {
        fval = (int)(gprev * 0x1p24f) - tinfo[t].off;
    } else {
        fval = gprev;
    }

    const bool deferred = live && ovf && !bad;
    if (deferred) {
        const unsigned long long key = ((unsigned long long)t << 40) | (unsigned long long)s;
        ovf_list[atomicAdd(ovf_count, 1u)] = key;
    }
    if (cost && live && !deferred) cost[(int64_t)t * S + s] = bad ? SPDP_INFEASIBLE : fval;
    if (partial == nullptr) return;

    Part p{0, 0, 0, 0, 0};
    if (live && !deferred) part_add_cost(p, fval, !bad);
    Part r = block_sum(p, red);
    if (tid == 0) {
        part_store(&bpart[(int64_t)t * gridDim.x + blockIdx.x], r);
        __threadfence();
        am_last = (atomicAdd(&tickets[t], 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    Part acc{0, 0, 0, 0, 0};
    const spdp_saa_partial* bp = bpart + (int64_t)t * gridDim.x;
    for (int b = tid; b < (int)gridDim.x; b += kSweepThreads) {
        acc.n_feas += __ldcg(&bp[b].n_feas);
        acc.n_infeas += __ldcg(&bp[b].n_infeas);
        acc.sum += __ldcg(&bp[b].sum);
        acc.sq_lo += __ldcg(&bp[b].sumsq_lo);
        acc.sq_hi += __ldcg(&bp[b].sumsq_hi);
    }
    __syncthreads();
    Part tot = block_sum(acc, red);
    if (tid == 0) {
        part_store(&partial[t], tot);
        tickets[t] = 0u;
    }
}

// ---------------------------------------------------------------- general kernel
// Transition-level parallelism: one warp per scenario, the
// lanes split the candidates p in [mask(i), i-1] and combine them with a
// shuffle min; mask(i) advances monotonically (two-pointer on the prefix).
// Handles any window width; used for the overflow list of the sweep.
__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

__global__ void __launch_bounds__(256) split_general_kernel(
    const int2* __restrict__ tabs, const int32_t* __restrict__ g0s, int n, const uint16_t* __restrict__ demand,
    int64_t ld, int64_t S, uint32_t Q, int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ partial,
    const unsigned long long* __restrict__ ovf_list, const unsigned* __restrict__ ovf_count) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int* g = reinterpret_cast<int*>(smem_raw) + (size_t)wid * 2 * (n + 1);
    uint32_t* pre = reinterpret_cast<uint32_t*>(g + (n + 1));
    const unsigned count = *ovf_count;
    for (unsigned idx = blockIdx.x * nw + wid; idx < count; idx += gridDim.x * nw) {
        const unsigned long long key = ovf_list[idx];
        const int t = (int)(key >> 40);
        const int64_t s = (int64_t)(key & ((1ull << 40) - 1));
        const int2* tab = tabs + (int64_t)t * (n + kTabPad);
        // tour-order prefix P'(i) = 1 + sum_{k<=i} q, i = 0..n
        uint32_t carry = 1u;
        if (lane == 0) pre[0] = 1u;
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            uint32_t v = (i < n) ? (uint32_t)demand[(int64_t)tab[i].x * ld + s] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t u = __shfl_up_sync(kFull, v, o);
                if (lane >= o) v += u;
            }
            if (i < n) pre[i + 1] = carry + v;
            carry += __shfl_sync(kFull, v, 31);
        }
        if (lane == 0) g[0] = g0s[t];
        __syncwarp();
        int m = 0;
        for (int L = 0; L < n; ++L) {
            const uint32_t Pn = pre[L + 1];
            while (Pn - pre[m] > Q) ++m;  // uniform across the warp (smem broadcast)
            int best = INT_MAX;
            for (int p = m + lane; p <= L; p += 32) best = min(best, g[p]);
            best = warp_min(best);
            if (lane == 0) g[L + 1] = best + tab[L].y;
            __syncwarp();
        }
        const int f = g[n];
        if (lane == 0) {
            if (cost) cost[(int64_t)t * S + s] = f;
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

// ---------------------------------------------------------------- sampling (window_hint = 0)
__global__ void sample_window_kernel(const int2* __restrict__ tab, int n, const uint16_t* __restrict__ demand,
                                     int64_t ld, int64_t S, uint32_t Q, unsigned* __restrict__ hdr) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    // two-pointer on the tour-order prefix, re-reading the left demand
    uint32_t P = 0, Pm = 0;
    int m = 0, wmax = 1;
    for (int i = 1; i <= n; ++i) {
        const uint32_t q = demand[(int64_t)tab[i - 1].x * ld + s];
        if (q > Q) return;  // infeasible scenario: not representative
        P += q;
        while (P - Pm > Q) {
            Pm += demand[(int64_t)tab[m].x * ld + s];
            ++m;
        }
        wmax = max(wmax, i - m);
    }
    atomicMax(&hdr[HDR_SAMPLE_W], (unsigned)wmax);
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
struct SweepArgs {
    const int2* tabs;
    const int2* tabsf;
    const int32_t* g0;
    const TourInfo* tinfo;
    int n;
    const uint16_t* demand;
    int64_t ld, S;
    uint32_t Q;
    int32_t* cost;
    spdp_saa_partial* bpart;
    spdp_saa_partial* partial;
    unsigned* tickets;
    unsigned long long* ovf;
    unsigned* ovf_count;
};

template <int W, int VE, bool F32>
static spdp_status launch_sweep_t(dim3 grid, cudaStream_t st, const SweepArgs& a) {
    auto kern = split_sweep_kernel<W, VE, F32>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e == cudaSuccess)  // all of the unified L1/smem as shared memory: occupancy is smem-bound
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(split_sweep)");
        attr_set = true;
    }
    prof_begin(st);
    kern<<<grid, kSweepThreads, SweepCfg<W>::smem_bytes(a.n), st>>>(F32 ? a.tabsf : a.tabs, a.g0, a.tinfo, a.n, a.demand,
                                                                    a.ld, a.S, a.Q, a.cost, a.bpart, a.partial,
                                                                    a.tickets, a.ovf, a.ovf_count);
    spdp_status rc = last_launch("split_sweep_kernel");
    prof_end(st);
    return rc;
}

// Tuning knobs (environment, read once): SPDP_SWEEP=auto|int|f32 selects the
// candidate arithmetic; SPDP_VOTE_EVERY selects the warp-vote stride.
static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

static int sweep_mode() {  // 0 auto, 1 int, 2 f32
    static int m = [] {
        const char* e = getenv("SPDP_SWEEP");
        if (!e) return 0;
        if (!strcmp(e, "int")) return 1;
        if (!strcmp(e, "f32")) return 2;
        return 0;
    }();
    return m;
}

static spdp_status launch_sweep(int W, bool f32, dim3 grid, cudaStream_t st, const SweepArgs& a) {
    static const int ve = env_int("SPDP_VOTE_EVERY", 4);
    if (f32) {
        switch (W) {
            case 8: return ve == 2 ? launch_sweep_t<8, 2, true>(grid, st, a) : launch_sweep_t<8, 4, true>(grid, st, a);
            case 16:
                return ve == 2 ? launch_sweep_t<16, 2, true>(grid, st, a)
                               : (ve == 8 ? launch_sweep_t<16, 8, true>(grid, st, a) : launch_sweep_t<16, 4, true>(grid, st, a));
            default:
                return ve == 8 ? launch_sweep_t<32, 8, true>(grid, st, a) : launch_sweep_t<32, 4, true>(grid, st, a);
        }
    }
    switch (W) {
        case 8: return ve == 2 ? launch_sweep_t<8, 2, false>(grid, st, a) : launch_sweep_t<8, 4, false>(grid, st, a);
        case 16: return ve == 2 ? launch_sweep_t<16, 2, false>(grid, st, a) : launch_sweep_t<16, 4, false>(grid, st, a);
        case 32: return ve == 2 ? launch_sweep_t<32, 2, false>(grid, st, a) : launch_sweep_t<32, 4, false>(grid, st, a);
        default: return launch_sweep_t<64, 4, false>(grid, st, a);
    }
}

static int pick_w(int hint) {
    if (hint <= 8) return 8;
    if (hint <= 16) return 16;
    if (hint <= 32) return 32;
    return 64;
}

static spdp_status split_common(const int32_t* tours, int32_t T, const int32_t* dist, int32_t n,
                                const uint16_t* demand, int64_t ld, int64_t S, int32_t Q, int32_t* cost,
                                spdp_saa_partial* partial, int32_t window_hint, void* ws, size_t ws_bytes,
                                uint32_t flags, cudaStream_t st, const char* fn) {
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
    if (L.nblocks > 0x7fffffffLL) return fail(SPDP_E_RESOURCE, "%s: grid too large", fn);
    char* w = static_cast<char*>(ws);
    unsigned* hdr = reinterpret_cast<unsigned*>(w + L.hdr);
    unsigned* tickets = reinterpret_cast<unsigned*>(w + L.tickets);
    int32_t* g0 = reinterpret_cast<int32_t*>(w + L.g0);
    int2* tabs = reinterpret_cast<int2*>(w + L.tabs);
    int2* tabsf = reinterpret_cast<int2*>(w + L.tabsf);
    TourInfo* tinfo = reinterpret_cast<TourInfo*>(w + L.tinfo);
    spdp_saa_partial* bpart = reinterpret_cast<spdp_saa_partial*>(w + L.bpart);
    unsigned long long* ovf = reinterpret_cast<unsigned long long*>(w + L.ovf);
    // Q above the largest possible load behaves as "everything fits"; clamp so P' + Q fits uint32.
    const uint32_t Qe = (uint32_t)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    const bool validate = (flags & SPDP_F_VALIDATE) != 0;
    spdp_status rc;
    if (validate || window_hint == 0) {
        rc = cuda_check(cudaMemsetAsync(hdr, 0, 256, st), "cudaMemsetAsync(hdr)");
        if (rc) return rc;
    }
    {
        const int threads = 1024;
        const size_t smem = 34 * sizeof(long long) + sizeof(unsigned) * (size_t)((n + 32) / 32 + 1);
        tour_prep_kernel<<<T, threads, smem, st>>>(tours, n, dist, tabs, g0, tabsf, tinfo, hdr, tickets, validate ? 1 : 0);
        if ((rc = last_launch("tour_prep_kernel"))) return rc;
    }
    int W = pick_w(window_hint);
    if (validate || window_hint == 0) {
        if (window_hint == 0) {
            const int64_t Ss = S < 4096 ? S : 4096;
            sample_window_kernel<<<(unsigned)ceil_div(Ss, 256), 256, 0, st>>>(tabs, n, demand, ld, Ss, Qe, hdr);
            if ((rc = last_launch("sample_window_kernel"))) return rc;
        }
        unsigned h[4];
        if ((rc = cuda_check(cudaMemcpyAsync(h, hdr, sizeof(h), cudaMemcpyDeviceToHost, st), "memcpy(hdr)"))) return rc;
        if ((rc = cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
        if (validate && h[HDR_STATUS]) {
            const unsigned b = h[HDR_STATUS];
            return fail(SPDP_E_DATA, "%s: invalid input:%s%s%s", fn, (b & ST_NOT_PERM) ? " tour is not a permutation of 1..n" : "",
                        (b & ST_NEG_DIST) ? " negative cost" : "",
                        (b & ST_RANGE) ? " 3*n*max(dist) exceeds the int32 range" : "");
        }
        if (window_hint == 0) W = pick_w((int)(h[HDR_SAMPLE_W] + h[HDR_SAMPLE_W] / 4 + 1));
    }
    const dim3 grid((unsigned)L.nblocks, (unsigned)T);
    unsigned* ovf_count = hdr + HDR_OVF_COUNT;
    const SweepArgs args{tabs, tabsf, g0, tinfo, n, demand, ld, S, Qe, cost, bpart, partial, tickets, ovf, ovf_count};
    // fp32 sweep when every load value it forms (P' <= n min(Q, 65535) for feasible scenarios,
    // Y = P' + Q) is an exact float; the per-tour cost range is checked on the device (TourInfo::ok)
    const int64_t qeff = Qe < 65535u ? (int64_t)Qe : 65535;
    const bool f32_loads_exact = ((int64_t)n + 64) * qeff + (int64_t)Qe + 1 < (1LL << 24);  // + padded layers
    const int mode = sweep_mode();
    const bool use_f32 = W <= 32 && (mode == 2 || (mode == 0 && f32_loads_exact)) && (mode != 2 || f32_loads_exact);
    rc = launch_sweep(W, use_f32, grid, st, args);
    if (rc) return rc;
    {
        // overflow list: warps per CTA limited by the per-warp smem (g and prefix: 8 (n+1) bytes)
        const size_t per_warp = 2 * sizeof(int) * (size_t)(n + 1);
        int warps = (int)((160 * 1024) / per_warp);
        warps = warps < 1 ? 1 : (warps > 8 ? 8 : warps);
        static bool attr_set = false;
        if (!attr_set) {
            cudaError_t e = cudaFuncSetAttribute(split_general_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(split_general)");
            attr_set = true;
        }
        split_general_kernel<<<296, warps * 32, per_warp * warps, st>>>(tabs, g0, n, demand, ld, S, Qe, cost, partial,
                                                                         ovf, ovf_count);
        if ((rc = last_launch("split_general_kernel"))) return rc;
    }
    return SPDP_OK;
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
    return split_common(tour, 1, dist, n, demand, ld, S, Q, cost, partial, window_hint, ws, ws_bytes, flags,
                        (cudaStream_t)stream, "spdp_split_eval");
}

extern "C" spdp_status spdp_split_eval_batch(const int32_t* tours, int32_t T, const int32_t* dist, int32_t n,
                                             const uint16_t* demand, int64_t ld, int64_t S, int32_t Q, int32_t* cost,
                                             spdp_saa_partial* partial, int32_t window_hint, void* ws, size_t ws_bytes,
                                             uint32_t flags, spdp_stream_t stream) {
    return split_common(tours, T, dist, n, demand, ld, S, Q, cost, partial, window_hint, ws, ws_bytes, flags,
                        (cudaStream_t)stream, "spdp_split_eval_batch");
}

extern "C" spdp_status spdp_demand_prefix(const int32_t* tour, int32_t n, const uint16_t* demand, int64_t ld, int64_t S,
                                          uint32_t* prefix, spdp_stream_t stream) {
    if (n < 1 || S < 1) return fail(SPDP_E_USAGE, "spdp_demand_prefix: n and S must be >= 1");
    if (!tour || !demand || !prefix) return fail(SPDP_E_USAGE, "spdp_demand_prefix: NULL pointer");
    if (ld < S) return fail(SPDP_E_USAGE, "spdp_demand_prefix: ld < S");
    prefix_kernel<<<(unsigned)ceil_div(S, 256), 256, 0, (cudaStream_t)stream>>>(tour, n, demand, ld, S, prefix);
    return last_launch("prefix_kernel");
}

extern "C" spdp_status spdp_split_mask(const int32_t* tour, int32_t n, const uint16_t* demand, int64_t ld, int64_t S,
                                       int32_t Q, int32_t* mask, spdp_stream_t stream) {
    if (n < 1 || S < 1 || Q < 1) return fail(SPDP_E_USAGE, "spdp_split_mask: n, S, Q must be >= 1");
    if (!tour || !demand || !mask) return fail(SPDP_E_USAGE, "spdp_split_mask: NULL pointer");
    if (ld < S) return fail(SPDP_E_USAGE, "spdp_split_mask: ld < S");
    mask_kernel<<<(unsigned)ceil_div(S, 256), 256, 0, (cudaStream_t)stream>>>(tour, n, demand, ld, S, (uint32_t)Q, mask);
    return last_launch("mask_kernel");
}

extern "C" spdp_status spdp_saa_reduce(const int32_t* cost, int64_t S, spdp_saa_partial* partial, spdp_stream_t stream) {
    if (S < 0 || !partial || (S > 0 && !cost)) return fail(SPDP_E_USAGE, "spdp_saa_reduce: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    spdp_status rc = cuda_check(cudaMemsetAsync(partial, 0, sizeof(spdp_saa_partial), st), "cudaMemsetAsync(partial)");
    if (rc || S == 0) return rc;
    int64_t blocks = ceil_div(S, 256 * 8);
    if (blocks > 148 * 8) blocks = 148 * 8;
    saa_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(cost, S, partial);
    return last_launch("saa_reduce_kernel");
}
