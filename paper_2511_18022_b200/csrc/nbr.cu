// nbr.cu -- f3: prefix / suffix split values of a parent tour and
// the evaluation of candidate tours that share a prefix and a suffix with it
// (the neighbourhood evaluation behind the paper's "explore many more candidate
// first-stage tours"; DESIGN R23).
//
// Values of one tour sigma (the definitions: Split of every prefix / suffix):
//   f(i) = Split(sigma_1..sigma_i),  b(i) = Split(sigma_{i+1}..sigma_n).
// With the separable route cost t(p, i) = A[p] + B[i] (split.cu):
//   f(i) = B[i] + min_{p in [mask(i), i-1]} f(p) + A[p]            (Eq. (3))
//   b(i) = A[i] + min_{j in [i+1, maxj(i)]} b(j) + B[j]            (the mirror)
// with maxj(i) = max{j : sum_{k=i+1}^{j} q <= Q}.
//
// A candidate tour that agrees with the parent on positions 1..a and s0+1..n
// (a < s0, 1-based) has f(p) = f_parent(p) for p <= a and b(i) = b_parent(i) for
// i >= s0, and every split of it has a route boundary in [s0, E] where E is the
// last layer a route starting before s0 can reach (the load of positions
// s0..E+1 exceeds Q, or E = n).  So
//   cost = min_{i in [s0, E]} f(i) + b_parent(i),
// where f(i) for i = a+1..E comes from the Eq. (3) sweep restarted at layer a+1
// on a ring seeded with f_parent(a-W+1..a) -- O(s0 - a + window) layers instead of n.
#include <climits>
#include <vector>

#include "common.cuh"
#include "split_ws.cuh"

namespace spdp {

constexpr int kNbrPf = 8;            // demand / b prefetch distance (layers)
constexpr double kNbrAutoSpan = 0.40;  // SPDP_F_NBR_AUTO: mean changed span / n above which the batch is faster
constexpr int kNbrSmemMaxN = 4095;  // position table in shared memory up to (n + 1) 16 B = 64 KB

// Per-tour position table e[i], i = 0..n:  {float bits of Cg[i] 2^-24 with Cg = A + B (the fp32
// phase of the neighbour sweep), A[i] (i < n), B[i] (i >= 1), row * ld of customer sigma_i as a
// uint32 element offset (callers check n ld < 2^32)}, A[p] = c_{0,s_{p+1}} - D[p+1], B[i] = D[i] + c_{s_i,0},
// D[1] = 0, D[i] = D[i-1] + c_{s_{i-1},s_i}.
// info[t] = {a, s0, parent index, 0}: a = common prefix length with the tour's parent
// (parents[parent_of[t]], or parents[0]), s0 = n - common suffix length (a = s0 = n: the tour
// equals its parent).  One warp per tour.
__global__ void __launch_bounds__(32) nbr_prep_kernel(const int32_t* __restrict__ tours, const int32_t* __restrict__ parents,
                                                      int n, const int32_t* __restrict__ dist, int64_t ld,
                                                      int4* __restrict__ etabs, int4* __restrict__ info,
                                                      const int32_t* __restrict__ parent_of, int P) {
    const int t = blockIdx.x, lane = threadIdx.x;
    const int32_t* tour = tours + (int64_t)t * n;
    int4* e = etabs + (int64_t)t * tour_tab_stride(n);
    const int64_t N1 = (int64_t)n + 1;
    auto node = [&](int i) -> int {  // customer at 0-based position i, clamped to 1..n
        const int c = tour[i];
        return c < 1 ? 1 : (c > n ? n : c);
    };
    long long carry = 0;  // D at the chunk's first position
    for (int b = 0; b < n; b += 32) {
        const int i = b + lane;  // 0-based position i = 1-based i + 1
        const int c = i < n ? node(i) : 1;
        const int arc = (i + 1 < n) ? dist[(int64_t)c * N1 + node(i + 1)] : 0;
        long long incl = arc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long u = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += u;
        }
        const long long D = carry + incl - arc;  // D[i+1]
        if (i < n) {
            int4 v;
            v.y = (i + 1 < n) ? (int)(dist[node(i + 1)] - (D + arc)) : 0;  // A[i+1] = c_{0,s_{i+2}} - D[i+2]
            v.z = (int)(D + dist[(int64_t)c * N1]);                          // B[i+1]
            v.x = __float_as_int((float)(v.y + v.z) * 0x1p-24f);             // Cg[i+1] 2^-24 (exact when |Cg| < 2^24)
            v.w = (int)(uint32_t)((uint64_t)(c - 1) * (uint64_t)ld);  // element offset of the row (n ld < 2^32)
            e[i + 1] = v;
        }
        carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) e[0] = make_int4(0, dist[node(0)], 0, 0);  // A[0] = c_{0,s_1}
    if (lane < kTourTabPad) e[n + 1 + lane] = make_int4(0, 0, 0, 0);  // padding (demand row 0)
    if (parents && info) {
        int par = parent_of ? parent_of[t] : 0;
        par = par < 0 ? 0 : (par >= P ? P - 1 : par);  // (clamped: a bad index cannot read out of bounds)
        const int32_t* parent = parents + (int64_t)par * n;
        int a = n, last = -1;
        for (int b = 0; b < n; b += 32) {
            const int i = b + lane;
            const unsigned mm = __ballot_sync(kFull, i < n && tour[i] != parent[i]);
            if (mm) {
                a = b + __ffs(mm) - 1;
                break;
            }
        }
        for (int b = n - 1; b >= 0 && a < n; b -= 32) {
            const int i = b - lane;
            const unsigned mm = __ballot_sync(kFull, i >= 0 && tour[i] != parent[i]);
            if (mm) {
                last = b - (__ffs(mm) - 1);
                break;
            }
        }
        if (lane == 0) info[t] = make_int4(a, a < n ? last + 1 : n, par, 0);
    }
}

// f and b of one tour, one scenario per thread: two-pointer masks (PAPER:120-127 and
// its mirror), window minima read back from the thread's own rows of fwd / bwd
// ([n+1][S], coalesced across the warp).  Any window width.  INF = SPDP_INFEASIBLE
// where the prefix / suffix holds a demand above Q (DESIGN R4).
__global__ void __launch_bounds__(256) split_values_kernel(const int4* __restrict__ e, int n,
                                                           const uint16_t* __restrict__ demand, int64_t ld, int64_t S,
                                                           int Q, int32_t* fwd, int32_t* bwd,
                                                           const int64_t* __restrict__ list,
                                                           const unsigned* __restrict__ count) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= (list ? (int64_t)*count : S)) return;
    const int64_t s = list ? list[w] : w;
    const uint16_t* dcol = demand + s;
    int32_t* fc = fwd + s;
    int32_t* bc = bwd + s;
    auto q_at = [&](int i) -> int { return dcol[(uint32_t)__ldg(&e[i].w)]; };  // q of position i >= 1
    // forward: f(i) = B[i] + min_{p in [m, i-1]} f(p) + A[p], m = mask(i)
    fc[0] = 0;
    {
        int P = 0, Pm = 0, m = 0;
        bool bad = false;
        for (int i = 1; i <= n; ++i) {
            const int4 ei = __ldg(&e[i]);
            const int q = dcol[(uint32_t)ei.w];
            bad |= q > Q;
            if (bad) {
                fc[(int64_t)i * S] = SPDP_INFEASIBLE;
                continue;
            }
            P += q;
            while (P - Pm > Q) Pm += q_at(++m);  // P(m) = sum_{k<=m} q; stops at m <= i-1 (q <= Q)
            int best = INT_MAX;
            for (int p = m; p < i; ++p) best = min(best, fc[(int64_t)p * S] + __ldg(&e[p].y));
            fc[(int64_t)i * S] = best + ei.z;
        }
    }
    // backward: b(i) = A[i] + min_{j in [i+1, M]} b(j) + B[j], M = maxj(i); R(i) = sum_{k>i} q
    bc[(int64_t)n * S] = 0;
    {
        int R = 0, RM = 0, M = n;
        bool bad = false;
        for (int i = n - 1; i >= 0; --i) {
            const int q = q_at(i + 1);
            bad |= q > Q;
            if (bad) {
                bc[(int64_t)i * S] = SPDP_INFEASIBLE;
                continue;
            }
            R += q;
            while (R - RM > Q) RM += q_at(M--);  // R(M-1) = R(M) + q(M); stops at M >= i+1
            int best = INT_MAX;
            for (int j = i + 1; j <= M; ++j) best = min(best, bc[(int64_t)j * S] + __ldg(&e[j].z));
            bc[(int64_t)i * S] = best + __ldg(&e[i].y);
        }
    }
}

// The register-ring version of the same two passes (the common case): one scenario per
// thread, a W-entry ring {value, load + Q} per direction, layers unrolled by W, demands
// prefetched kNbrPf layers ahead.  Forward: G = f(p) + A[p], Y = P(p) + Q, window of
// layer i = ring entries with Y >= P(i).  Backward (the mirror): H = b(j) + B[j], Y =
// R(j) + Q with R(j) = sum_{k>j} q, window of position i = entries with Y >= R(i).  A
// scenario whose window outgrows the ring (or that holds a demand above Q) is listed
// for split_values_kernel.
template <int W>
__device__ __forceinline__ bool values_pass(const int4* __restrict__ e, int n, const uint16_t* __restrict__ dcol,
                                            int Q, int32_t* __restrict__ outc, int64_t S, bool backward) {
    int G[W], Y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        G[k] = INT_MAX;
        Y[k] = INT_MIN;
    }
    // position of step L: forward i = L + 1 (its g-entry at i-1 = L), backward i = n - 1 - L
    auto qpos = [&](int L) -> int { return backward ? n - L : L + 1; };  // the demand entering step L
    int qb[kNbrPf];
#pragma unroll
    for (int k = 0; k < kNbrPf; ++k) qb[k] = (k < n) ? (int)dcol[(uint32_t)e[qpos(k)].w] : 0;
    // entry for the start point: forward p = 0 (f = 0, G = A[0]), backward j = n (b = 0, H = B[n])
    int cur = backward ? e[n].z : e[0].y;
    int P = 0;
    bool ok = true;
    for (int L0 = 0; L0 < n; L0 += W) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int L = L0 + j;
            if (L < n) {
                const int q = qb[j % kNbrPf];
                if (L + kNbrPf < n) qb[j % kNbrPf] = dcol[(uint32_t)e[qpos(L + kNbrPf)].w];
                const int Pn = P + q;
                ok &= q <= Q;
                ok &= !(Y[j] >= Pn);  // the slot being overwritten (age W + 1) still in the window
                G[j] = cur;
                Y[j] = P + Q;
                int best = cur;
#pragma unroll
                for (int k = 1; k < W; ++k) {
                    const int sl = (j - k + W) % W;
                    if (Y[sl] < Pn) break;  // the window is a contiguous run of the newest entries (R5)
                    best = min(best, G[sl]);
                }
                const int i = backward ? n - 1 - L : L + 1;
                const int4 ei = e[i];
                // forward: f(i) = best + B[i], next entry g(i) = f(i) + A[i]
                // backward: b(i) = best + A[i], next entry h(i) = b(i) + B[i]
                const int val = backward ? best + ei.y : best + ei.z;
                outc[(int64_t)i * S] = val;
                cur = val + (backward ? ei.z : ei.y);
                P = Pn;
            }
        }
    }
    return ok;
}

template <int W>
__global__ void __launch_bounds__(128) split_values_ring_kernel(const int4* __restrict__ etab, int n,
                                                                const uint16_t* __restrict__ demand, int64_t S, int Q,
                                                                int32_t* __restrict__ fwd, int32_t* __restrict__ bwd,
                                                                int64_t* __restrict__ list, unsigned* __restrict__ count,
                                                                int table_in_smem) {
    extern __shared__ int4 sm4[];
    const int4* e = etab;
    if (table_in_smem) {
        for (int i = threadIdx.x; i <= n; i += blockDim.x) sm4[i] = etab[i];
        __syncthreads();
        e = sm4;
    }
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const uint16_t* dcol = demand + s;
    // blockIdx.y: the forward (0) or the backward (1) pass -- two independent threads per scenario
    const bool backward = blockIdx.y != 0;
    int32_t* out = backward ? bwd : fwd;
    out[(backward ? (int64_t)n * S : 0) + s] = 0;
    // (a scenario deferred by both passes is listed twice: the general kernel writes the same values)
    if (!values_pass<W>(e, n, dcol, Q, out + s, S, backward)) list[atomicAdd(count, 1u)] = s;
}

// The restarted sweep: one scenario per thread, one candidate tour per blockIdx.x.
// Ring of the last W split points p (slot (p - a - 1) mod W): {G = f(p) + A[p],
// Y = P(p) + Q} with P relative to P(a) = 0; p is in the window of layer i iff
// Y >= P(i).  Seeded from the parent's f(a-W+1..a).  The candidate's position
// table sits in shared memory (SM) or is read through L1 (padded past n, so the
// demand prefetch kNbrPf layers ahead needs no bounds check; addresses are one
// 32-bit multiply-add from the row offset).  Phase A (layers a+1..s0-1, whole
// W-layer chunks) is the plain Eq. (3) sweep; phase B (from the chunk holding s0)
// adds the suffix combination min f(i) + b_parent(i), the per-lane stop once no
// route starting before s0 reaches the layer, and the b_parent prefetch.  Ages
// 2..kNbrU0+1 are scanned unconditionally, then groups of 4 behind a warp vote.
// A lane whose window reaches the oldest ring age is appended to the overflow list
// (finished from scratch by split_finish_kernel on the candidate's own tables).
constexpr int kNbrThreads = 128;
constexpr int kNbrU0 = 8;  // (measured at C3: 4 / 8 / 12 -> population 9.3 / 9.0 / 8.7 ms, granular 3.11 / 3.14 / 3.19 ms)

__device__ __forceinline__ const void* mad_wide(uint32_t a, uint32_t b, const void* base) {
    uint64_t r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(base));
    return reinterpret_cast<const void*>(r);
}

template <int W, bool SM>
__global__ void __launch_bounds__(kNbrThreads, (W <= 16 ? 6 : 1)) split_nbr_kernel(
    const int4* __restrict__ etabs, const int4* __restrict__ info, int n, const uint16_t* __restrict__ demand,
    int64_t S, int Q, const int32_t* __restrict__ fwd, const int32_t* __restrict__ bwd,
    int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ slots, unsigned long long* __restrict__ ovf_list,
    unsigned* __restrict__ ovf_count, const TourInfo* __restrict__ tinfo, int f32_loads, int64_t s_off) {
    static_assert(W % kNbrPf == 0, "the prefetch distance must divide the ring");
    static_assert(kNbrU0 % 4 == 0 && kNbrU0 < W, "unconditional ages");
    __shared__ Part red[kNbrThreads / 32];
    extern __shared__ int4 stab[];
    const int t = blockIdx.x;  // tours fastest: the CTAs resident together share scenario tiles (L2 reuse)
    const int4 in = info[t];
    const int a = in.x, s0 = in.y;
    const int stride = tour_tab_stride(n);
    const int4* e = etabs + (int64_t)t * stride;
    if constexpr (SM) {
        for (int i = threadIdx.x; i < stride; i += kNbrThreads) stab[i] = e[i];
        __syncthreads();
    }
    auto tab = [&](int i) -> int4 {
        if constexpr (SM) return stab[i];
        else return __ldg(&e[i]);
    };
    auto rowoff = [&](int i) -> uint32_t {
        if constexpr (SM) return (uint32_t)stab[i].w;
        else return (uint32_t)__ldg(&e[i].w);
    };
    const int64_t s = s_off + (int64_t)blockIdx.y * kNbrThreads + threadIdx.x;  // (launches of <= 65535 tiles)
    const bool live = s < S;
    const int64_t col = live ? s : S - 1;
    const int64_t pbase = (int64_t)in.z * (int64_t)(n + 1) * S;  // the tour's parent's value rows
    const int32_t* fcol = fwd + pbase + col;
    const int32_t* bcol = bwd + pbase + col;
    const uint16_t* dcol = demand + col;
    const uint32_t Su = (uint32_t)S, S4 = 4u * (uint32_t)S;  // (n + 1) S < 2^32, 4 S < 2^32
    auto dem = [&](uint32_t off) -> int { return *static_cast<const uint16_t*>(mad_wide(off, 2u, dcol)); };
    auto bwd_at = [&](int i) -> int { return *static_cast<const int32_t*>(mad_wide((uint32_t)i, S4, bcol)); };
    const int pc = fcol[(uint32_t)n * Su];  // the parent's cost: same customers, same feasibility (R4)
    int result = pc;
    bool ovf = false;
    if (a < n) {  // (a, s0 are uniform per CTA; every lane enters: the loops vote over the full warp)
        int G[W], Y[W];
        {
            int P = 0;  // P(p) - P(a), walking p down from a
#pragma unroll
            for (int k = 1; k <= W; ++k) {
                const int p = a + 1 - k;
                if (p >= 0) {
                    const int4 ep = tab(p);
                    G[W - k] = fcol[(uint32_t)p * Su] + ep.y;
                    Y[W - k] = P + Q;
                    if (p >= 1) P -= dem((uint32_t)ep.w);
                } else {
                    G[W - k] = INT_MAX;
                    Y[W - k] = INT_MIN;  // never in a window
                }
            }
        }
        int qb[kNbrPf];
#pragma unroll
        for (int k = 0; k < kNbrPf; ++k) qb[k] = dem(rowoff(a + 1 + k));  // (padded past n)
        int P = 0;
        // candidate scan of layer (slot j, load Pn): age 1 (slot j-1) is always in the window (q <= Q)
        auto scan = [&](const int j, const int Pn, const bool active) -> int {
            int best = G[(j - 1 + W) % W], best1 = INT_MAX;
#pragma unroll
            for (int k = 2; k < 2 + kNbrU0; ++k) {
                const int sl = (j - k + W) % W;
                if (Y[sl] >= Pn) {
                    if (k & 1) best1 = min(best1, G[sl]);
                    else best = min(best, G[sl]);
                }
            }
#pragma unroll
            for (int k0 = 2 + kNbrU0; k0 <= W; k0 += 4) {
                if (!__any_sync(kFull, active && Y[(j - k0 + W) % W] >= Pn)) break;
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int k = k0 + v;
                    if (k <= W) {
                        const int sl = (j - k + W) % W;
                        if (Y[sl] >= Pn) {
                            if (k & 1) best1 = min(best1, G[sl]);
                            else best = min(best, G[sl]);
                        }
                    }
                }
            }
            // age W (slot j) still in the window: the window may reach past the ring (conservative
            // when that point is position 0; the finish kernel then recomputes the lane exactly)
            if (active && Y[j] >= Pn) ovf = true;
            return min(best, best1);
        };
        const bool feas = pc != SPDP_INFEASIBLE;  // an infeasible scenario only follows the warp
        int base = a + 1;
        const TourInfo ti = tinfo[t];
        if (f32_loads && ti.ok && base + W <= s0) {
            // phase A in exact fp32, the candidate masking on the FMA pipe (as split_sweep_f2_kernel):
            // G = (g + OFF) 2^-24 in [0, 1); loads as the bits of 2^23 + BIAS + P (+ Q), so P += q is an
            // integer add on the bits; s = sat(P(i) - Y) is 0 inside the window and 1 outside, and
            // G + s >= 1 > every in-window G.  (Host: (n + W) Qe + Q + 1 < 2^23; tour: TourInfo::ok.)
            constexpr uint32_t kMagic = 0x4B000000u;
            const uint32_t bias = (uint32_t)W * (uint32_t)Q + 1u;  // every seed load >= -W Q: bias + P >= 1
            const float offf = (float)ti.off;
            float Gf[W];
            uint32_t Yb[W];
#pragma unroll
            for (int k = 0; k < W; ++k) {
                Gf[k] = (Y[k] == INT_MIN) ? 0.0f : ((float)(G[k] + ti.off)) * 0x1p-24f;
                Yb[k] = (Y[k] == INT_MIN) ? 0u : kMagic + bias + (uint32_t)Y[k];  // (float 0: never in a window)
            }
            uint32_t Pb = kMagic + bias + (uint32_t)P;
            while (base + W <= s0) {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    const int i = base + j;
                    const uint32_t q = (uint32_t)qb[j % kNbrPf];
                    qb[j % kNbrPf] = dem(rowoff(i + kNbrPf));
                    const uint32_t Pnb = Pb + q;
                    const float Pn = __uint_as_float(Pnb);
                    auto cand = [&](const int k) -> float {
                        const int sl = (j - k + W) % W;
                        return Gf[sl] + __saturatef(Pn - __uint_as_float(Yb[sl]));
                    };
                    float best = Gf[(j - 1 + W) % W];  // age 1
#pragma unroll
                    for (int k = 2; k < 2 + kNbrU0; k += 2) best = fminf(best, fminf(cand(k), cand(k + 1)));
#pragma unroll
                    for (int k0 = 2 + kNbrU0; k0 <= W; k0 += 4) {
                        if (!__any_sync(kFull, feas && Yb[(j - k0 + W) % W] >= Pnb)) break;
#pragma unroll
                        for (int v = 0; v < 4; v += 2)
                            if (k0 + v + 1 <= W) best = fminf(best, fminf(cand(k0 + v), cand(k0 + v + 1)));
                            else if (k0 + v <= W) best = fminf(best, cand(k0 + v));
                    }
                    if (feas && Yb[j] >= Pnb) ovf = true;  // age W still in the window
                    Gf[j] = best + __int_as_float(tab(i).x);  // + Cg[i] 2^-24
                    Yb[j] = Pnb + (uint32_t)Q;
                    Pb = Pnb;
                }
                base += W;
            }
            // back to the int32 ring for phase B
#pragma unroll
            for (int k = 0; k < W; ++k) {
                G[k] = (int)(Gf[k] * 0x1p24f) - ti.off;
                Y[k] = (Yb[k] < kMagic) ? INT_MIN : (int)(Yb[k] - kMagic - bias);
            }
            P = (int)(Pb - kMagic - bias);
            (void)offf;
        }
        // (without the fp32 phase, phase B runs every layer: one int32 body keeps the code small)
        // phase B: from the chunk holding s0 to the stop
        int bb[kNbrPf];
#pragma unroll
        for (int k = 0; k < kNbrPf; ++k) {
            const int i = base + k;
            bb[k] = (i >= s0 && i <= n) ? bwd_at(i) : 0;
        }
        int Ps = P;  // P(s0 - 1) when base == s0; else set at layer s0 - 1 below
        int total = INT_MAX;
        bool active = feas;
        for (;; base += W) {
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const int i = base + j;
                if (i > n) break;  // warp-uniform
                const int q = qb[j % kNbrPf];
                const int bv = bb[j % kNbrPf];
                const int ia = i + kNbrPf;
                qb[j % kNbrPf] = dem(rowoff(ia));
                if (ia >= s0 && ia <= n) bb[j % kNbrPf] = bwd_at(ia);
                const int Pn = P + q;
                // no route starting before s0 reaches layer i: the boundary set [s0, i-1] is complete
                if (i > s0 && Pn - Ps > Q) active = false;
                const int best = scan(j, Pn, active);
                const int4 ei = tab(i);
                if (active && i >= s0) total = min(total, best + ei.z + bv);
                G[j] = best + ei.y + ei.z;
                Y[j] = Pn + Q;
                if (i == s0 - 1) Ps = Pn;
                P = Pn;
            }
            if (base + W > n || !__any_sync(kFull, active && !ovf)) break;
        }
        result = feas ? total : pc;
    }
    const bool deferred = live && ovf;
    if (deferred) ovf_list[atomicAdd(ovf_count, 1u)] = ((unsigned long long)t << 40) | (unsigned long long)s;
    if (cost && live && !deferred) cost[(int64_t)t * S + s] = result;
    if (slots) {
        Part p{0, 0, 0, 0, 0};
        if (live && !deferred) part_add_cost(p, result, result != SPDP_INFEASIBLE);
        const Part r = block_sum(p, red);
        if (threadIdx.x == 0) {
            spdp_saa_partial* d = &slots[(int64_t)t * kSlots + (blockIdx.y % kSlots)];
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_feas), (unsigned long long)r.n_feas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_infeas), (unsigned long long)r.n_infeas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sum), (unsigned long long)r.sum);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sumsq_lo), (unsigned long long)r.sq_lo);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sumsq_hi), (unsigned long long)r.sq_hi);
        }
    }
}

spdp_status launch_tour_table(const int32_t* tours, int32_t T, const int32_t* parent, int32_t n, const int32_t* dist,
                              int64_t ld, int4* etabs, int4* info, cudaStream_t st) {
    nbr_prep_kernel<<<T, 32, 0, st>>>(tours, parent, n, dist, ld, etabs, info, nullptr, 1);
    return last_launch("nbr_prep_kernel");
}

// The same restarted sweep with the ring in shared memory ([W][NT] {G, Y} per CTA,
// slot p mod W, conflict-free 8-byte rows): the layer loop is unrolled only by the
// prefetch distance and the candidate scan is a loop of 4-candidate groups behind a
// warp vote, so the code stays small (the register ring's unrolled W-layer body
// overflows the instruction cache: ncu no_instruction stalls) and registers few.
// Any power-of-two W (64 covers the C4 windows).
template <int W, int NT>
__global__ void __launch_bounds__(NT) split_nbr_smem_kernel(
    const int4* __restrict__ etabs, const int4* __restrict__ info, int n, const uint16_t* __restrict__ demand,
    int64_t S, int Q, const int32_t* __restrict__ fwd, const int32_t* __restrict__ bwd,
    int32_t* __restrict__ cost, spdp_saa_partial* __restrict__ slots, unsigned long long* __restrict__ ovf_list,
    unsigned* __restrict__ ovf_count, int table_in_smem, int64_t s_off) {
    static_assert((W & (W - 1)) == 0 && W >= 8, "W: a power of two");
    __shared__ Part red[NT / 32];
    extern __shared__ int4 sm4[];
    int2* ring = reinterpret_cast<int2*>(sm4);  // [W][NT]
    const int t = blockIdx.x;
    const int4 in = info[t];
    const int a = in.x, s0 = in.y;
    const int4* tb = etabs + (int64_t)t * tour_tab_stride(n);
    if (table_in_smem) {
        int4* st = sm4 + (W * NT) / 2;
        for (int i = threadIdx.x; i <= n; i += NT) st[i] = tb[i];
        __syncthreads();
        tb = st;
    }
    const int tid = threadIdx.x;
    auto R = [&](int p) -> int2& { return ring[(p & (W - 1)) * NT + tid]; };
    const int64_t s = s_off + (int64_t)blockIdx.y * NT + tid;
    const bool live = s < S;
    const int64_t col = live ? s : S - 1;
    const int64_t pbase = (int64_t)in.z * (int64_t)(n + 1) * S;  // the tour's parent's value rows
    const int32_t* fcol = fwd + pbase + col;
    const int32_t* bcol = bwd + pbase + col;
    const uint16_t* dcol = demand + col;
    const uint32_t Su = (uint32_t)S;
    const int pc = fcol[(uint32_t)n * Su];
    int result = pc;
    bool ovf = false;
    if (a < n) {
        {
            int P = 0;
            for (int k = 1; k <= W; ++k) {
                const int p = a + 1 - k;
                if (p >= 0) {
                    const int4 ep = tb[p];
                    R(p) = make_int2(fcol[(uint32_t)p * Su] + ep.y, P + Q);
                    if (p >= 1) P -= dcol[(uint32_t)ep.w];
                } else {
                    R(p) = make_int2(INT_MAX, INT_MIN);
                }
            }
        }
        int qb[kNbrPf], bb[kNbrPf];
#pragma unroll
        for (int k = 0; k < kNbrPf; ++k) {
            const int i = a + 1 + k;
            qb[k] = 0;
            bb[k] = 0;
            if (i <= n) {
                qb[k] = dcol[(uint32_t)tb[i].w];
                if (i >= s0) bb[k] = bcol[(uint32_t)i * Su];
            }
        }
        int P = 0, Ps = 0;
        int gprev = R(a).x;  // g(a), age 1 of layer a + 1
        int total = INT_MAX;
        bool active = pc != SPDP_INFEASIBLE;
        for (int base = a + 1;; base += kNbrPf) {
#pragma unroll
            for (int j = 0; j < kNbrPf; ++j) {
                const int i = base + j;
                if (i > n) break;  // warp-uniform
                const int4 ei = tb[i];
                const int q = qb[j];
                const int bv = bb[j];
                const int ia = i + kNbrPf;
                if (ia <= n) {
                    qb[j] = dcol[(uint32_t)tb[ia].w];
                    if (ia >= s0) bb[j] = bcol[(uint32_t)ia * Su];
                }
                const int Pn = P + q;
                if (i > s0 && Pn - Ps > Q) active = false;
                int best = gprev, best1 = INT_MAX;  // age 1 is always in the window (q <= Q)
                bool deep = true;
                for (int k0 = 2; k0 <= W; k0 += 4) {
                    if (!__any_sync(kFull, active && R(i - k0).y >= Pn)) {
                        deep = false;
                        break;
                    }
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int k = k0 + v;
                        if (k <= W) {
                            const int2 c = R(i - k);
                            if (c.y >= Pn) {
                                if (v & 1) best1 = min(best1, c.x);
                                else best = min(best, c.x);
                            }
                        }
                    }
                }
                best = min(best, best1);
                // the scan reached age W still inside the window and an older point exists
                if (deep && active && R(i - W).y >= Pn && i - W >= 1) ovf = true;
                if (active && i >= s0) total = min(total, best + ei.z + bv);
                gprev = best + ei.y + ei.z;  // g(i) = f(i) + A[i]
                R(i) = make_int2(gprev, Pn + Q);  // (slot of position i - W, no longer needed)
                if (i == s0 - 1) Ps = Pn;
                P = Pn;
            }
            if (base + kNbrPf > n || !__any_sync(kFull, active && !ovf)) break;
        }
        result = pc == SPDP_INFEASIBLE ? pc : total;
    }
    const bool deferred = live && ovf;
    if (deferred) ovf_list[atomicAdd(ovf_count, 1u)] = ((unsigned long long)t << 40) | (unsigned long long)s;
    if (cost && live && !deferred) cost[(int64_t)t * S + s] = result;
    if (slots) {
        Part p{0, 0, 0, 0, 0};
        if (live && !deferred) part_add_cost(p, result, result != SPDP_INFEASIBLE);
        const Part r = block_sum(p, red);
        if (threadIdx.x == 0) {
            spdp_saa_partial* d = &slots[(int64_t)t * kSlots + (blockIdx.y % kSlots)];
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_feas), (unsigned long long)r.n_feas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_infeas), (unsigned long long)r.n_infeas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sum), (unsigned long long)r.sum);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sumsq_lo), (unsigned long long)r.sq_lo);
            atomicAdd(reinterpret_cast<unsigned long long*>(&d->sumsq_hi), (unsigned long long)r.sq_hi);
        }
    }
}

static size_t etab_bytes(int32_t n, int32_t T) { return align_up(sizeof(int4) * (size_t)T * (size_t)tour_tab_stride(n), 256); }

static spdp_status check_common(const char* fn, int32_t n, int64_t S, int32_t Q, int64_t ld, const void* demand) {
    if (n < 1) return fail(SPDP_E_USAGE, "%s: n=%d < 1", fn, n);
    if (n > SPDP_MAX_N) return fail(SPDP_E_RESOURCE, "%s: n=%d > SPDP_MAX_N=%d", fn, n, SPDP_MAX_N);
    if (S < 1) return fail(SPDP_E_USAGE, "%s: S=%lld < 1", fn, (long long)S);
    if (S >= (1LL << 40)) return fail(SPDP_E_RESOURCE, "%s: S too large", fn);
    if (Q < 1) return fail(SPDP_E_USAGE, "%s: Q=%d < 1 (SPEC:34)", fn, Q);
    if (ld < S || (ld % 8) != 0) return fail(SPDP_E_USAGE, "%s: ld=%lld must be >= S and a multiple of 8", fn, (long long)ld);
    if (((uintptr_t)demand & 15u) != 0) return fail(SPDP_E_USAGE, "%s: demand must be 16-byte aligned", fn);
    return SPDP_OK;
}

}  // namespace spdp

using namespace spdp;

extern "C" size_t spdp_values_workspace_bytes(int32_t n, int64_t S) {
    if (n < 1 || S < 1) return 0;
    return etab_bytes(n, 1) + align_up(sizeof(int64_t) * 2 * (size_t)S, 256) + 256;
}

extern "C" spdp_status spdp_split_values(const int32_t* tour, const int32_t* dist, int32_t n, const uint16_t* demand,
                                         int64_t ld, int64_t S, int32_t Q, int32_t* fwd, int32_t* bwd, void* ws,
                                         size_t ws_bytes, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_values");
    const char* fn = "spdp_split_values";
    spdp_status rc = check_common(fn, n, S, Q, ld, demand);
    if (rc) return rc;
    if (!tour || !dist || !demand || !fwd || !bwd || !ws) return fail(SPDP_E_USAGE, "%s: NULL required pointer", fn);
    if (ws_bytes < spdp_values_workspace_bytes(n, S)) return fail(SPDP_E_USAGE, "%s: workspace too small", fn);
    if ((uint64_t)n * (uint64_t)ld >= (1ull << 32)) return fail(SPDP_E_RESOURCE, "%s: n ld must stay below 2^32", fn);
    cudaStream_t st = (cudaStream_t)stream;
    char* w = static_cast<char*>(ws);
    int4* e = reinterpret_cast<int4*>(w);
    int64_t* list = reinterpret_cast<int64_t*>(w + etab_bytes(n, 1));
    unsigned* count = reinterpret_cast<unsigned*>(w + etab_bytes(n, 1) + align_up(sizeof(int64_t) * 2 * (size_t)S, 256));
    nbr_prep_kernel<<<1, 32, 0, st>>>(tour, nullptr, n, dist, ld, e, nullptr, nullptr, 1);
    if ((rc = last_launch("nbr_prep_kernel"))) return rc;
    if ((rc = cuda_check(cudaMemsetAsync(count, 0, sizeof(unsigned), st), "cudaMemsetAsync(count)"))) return rc;
    // Q above the largest possible load behaves as "everything fits"; clamp so sums stay in int32
    const int Qe = (int)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    const bool tsm = n <= kNbrSmemMaxN;
    if ((rc = kernel_setup((const void*)split_values_ring_kernel<32>, (int)(sizeof(int4) * (kNbrSmemMaxN + 1)), -1, 0, 0,
                           nullptr, "split_values_ring_kernel setup")))
        return rc;
    prof_begin(st);
    split_values_ring_kernel<32><<<dim3((unsigned)ceil_div(S, 128), 2), 128, tsm ? sizeof(int4) * (size_t)(n + 1) : 0, st>>>(
        e, n, demand, S, Qe, fwd, bwd, list, count, tsm ? 1 : 0);
    if ((rc = last_launch("split_values_ring_kernel"))) return rc;
    // the scenarios whose window outgrew the ring (or with a demand above Q): the general kernel
    split_values_kernel<<<(unsigned)ceil_div(2 * S, 256), 256, 0, st>>>(e, n, demand, ld, S, Qe, fwd, bwd, list, count);
    prof_end(st);
    set_last_kernel("split_values_ring_kernel<32>");
    return last_launch("split_values_kernel");
}

extern "C" size_t spdp_neighbour_workspace_bytes(int32_t n, int64_t S, int32_t T) {
    if (n < 1 || S < 1 || T < 1) return 0;
    return ws_layout(n, S, T).total + etab_bytes(n, T) + align_up(sizeof(int4) * (size_t)T, 256);
}


template <int W>
static spdp_status launch_nbr_t(cudaStream_t st, const int4* e, const int4* info, int n, const uint16_t* demand,
                                int64_t S, int T, int Q, const int32_t* fwd, const int32_t* bwd,
                                int32_t* cost, spdp_saa_partial* slots, unsigned long long* ovf, unsigned* ovf_count,
                                const TourInfo* tinfo, int f32_loads) {
    const int64_t ntile = ceil_div(S, kNbrThreads);
    prof_begin(st);
    for (int64_t y0 = 0; y0 < ntile; y0 += 65535) {  // (grid.y <= 65535 tiles per launch)
    const dim3 grid((unsigned)T, (unsigned)(ntile - y0 < 65535 ? ntile - y0 : 65535));
    const int64_t s_off = y0 * kNbrThreads;
    if (n <= kNbrSmemMaxN) {
        const size_t smem = sizeof(int4) * (size_t)tour_tab_stride(n);
        if (spdp_status e = kernel_setup((const void*)split_nbr_kernel<W, true>, (int)(sizeof(int4) * tour_tab_stride(kNbrSmemMaxN)),
                                         -1, 0, 0, nullptr, "split_nbr_kernel setup"))
            return e;
        split_nbr_kernel<W, true><<<grid, kNbrThreads, smem, st>>>(e, info, n, demand, S, Q, fwd, bwd, cost, slots, ovf,
                                                                   ovf_count, tinfo, f32_loads, s_off);
    } else {
        split_nbr_kernel<W, false><<<grid, kNbrThreads, 0, st>>>(e, info, n, demand, S, Q, fwd, bwd, cost, slots, ovf,
                                                                 ovf_count, tinfo, f32_loads, s_off);
    }
    }
    prof_end(st);
    set_last_kernel("split_nbr_kernel<%d,%d>", W, n <= kNbrSmemMaxN ? 1 : 0);
    return last_launch("split_nbr_kernel");
}

constexpr int kNbrSmemThreads = 128;

template <int W>
static spdp_status launch_nbr_smem_t(cudaStream_t st, const int4* e, const int4* info, int n, const uint16_t* demand,
                                     int64_t S, int T, int Q, const int32_t* fwd, const int32_t* bwd, int32_t* cost,
                                     spdp_saa_partial* slots, unsigned long long* ovf, unsigned* ovf_count) {
    constexpr int NT = kNbrSmemThreads;
    const bool tsm = n <= kNbrSmemMaxN;
    const size_t ring = sizeof(int2) * (size_t)W * NT;
    const size_t smem = ring + (tsm ? sizeof(int4) * (size_t)(n + 1) : 0);
    if (spdp_status e = kernel_setup((const void*)split_nbr_smem_kernel<W, NT>, (int)(ring + sizeof(int4) * (kNbrSmemMaxN + 1)),
                                     -1, 0, 0, nullptr, "split_nbr_smem_kernel setup"))
        return e;
    const int64_t ntile = ceil_div(S, NT);
    prof_begin(st);
    for (int64_t y0 = 0; y0 < ntile; y0 += 65535) {  // (grid.y <= 65535 tiles per launch)
        const dim3 grid((unsigned)T, (unsigned)(ntile - y0 < 65535 ? ntile - y0 : 65535));
        split_nbr_smem_kernel<W, NT><<<grid, NT, smem, st>>>(e, info, n, demand, S, Q, fwd, bwd, cost, slots, ovf,
                                                             ovf_count, tsm ? 1 : 0, y0 * NT);
    }
    prof_end(st);
    set_last_kernel("split_nbr_smem_kernel<%d>", W);
    return last_launch("split_nbr_smem_kernel");
}

extern "C" spdp_status spdp_split_eval_neighbours_multi(const int32_t* parents, int32_t P, const int32_t* parent_of,
                                                        const int32_t* fwd, const int32_t* bwd, const int32_t* tours,
                                                        int32_t T, const int32_t* dist, int32_t n, const uint16_t* demand,
                                                        int64_t ld, int64_t S, int32_t Q, int32_t* cost,
                                                        spdp_saa_partial* partial, int32_t window_hint, void* ws,
                                                        size_t ws_bytes, uint32_t flags, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval_neighbours_multi");
    const char* fn = "spdp_split_eval_neighbours";
    const int32_t* parent = parents;
    if (P < 1) return fail(SPDP_E_USAGE, "%s: P=%d < 1", fn, P);
    if (P > 1 && !parent_of) return fail(SPDP_E_USAGE, "%s: parent_of is NULL with P=%d parents", fn, P);
    spdp_status rc = check_common(fn, n, S, Q, ld, demand);
    if (rc) return rc;
    if (T < 1) return fail(SPDP_E_USAGE, "%s: T=%d < 1", fn, T);
    if (T >= (1 << 23)) return fail(SPDP_E_RESOURCE, "%s: T=%d too large", fn, T);
    if (window_hint < 0) return fail(SPDP_E_USAGE, "%s: window_hint < 0", fn);
    if (!parent || !fwd || !bwd || !tours || !dist || !demand || !ws)
        return fail(SPDP_E_USAGE, "%s: NULL required pointer", fn);
    if (ws_bytes < spdp_neighbour_workspace_bytes(n, S, T)) return fail(SPDP_E_USAGE, "%s: workspace too small", fn);
    if ((uint64_t)n * (uint64_t)ld >= (1ull << 32) || (uint64_t)(n + 1) * (uint64_t)S >= (1ull << 32) || S >= (1LL << 30))
        return fail(SPDP_E_RESOURCE, "%s: n ld and (n + 1) S must stay below 2^32, S below 2^30", fn);
    cudaStream_t st = (cudaStream_t)stream;
    const WsLayout L = ws_layout(n, S, T);
    char* w = static_cast<char*>(ws);
    int4* e = reinterpret_cast<int4*>(w + L.total);
    int4* info = reinterpret_cast<int4*>(w + L.total + etab_bytes(n, T));
    const bool validate = (flags & SPDP_F_VALIDATE) != 0;
    unsigned* hdr = reinterpret_cast<unsigned*>(w + L.hdr);
    if (validate && (rc = cuda_check(cudaMemsetAsync(hdr, 0, 256, st), "cudaMemsetAsync(hdr)"))) return rc;
    // the candidates' own tables (for the overflow path) + zeroed SAA slots / partials
    if ((rc = launch_tour_prep(tours, T, n, dist, demand, ld, w, L, partial, partial != nullptr, validate, st))) return rc;
    if (validate) {
        unsigned h[2];
        if ((rc = cuda_check(cudaMemcpyAsync(h, hdr, sizeof(h), cudaMemcpyDeviceToHost, st), "memcpy(hdr)"))) return rc;
        if ((rc = cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
        if (h[HDR_STATUS]) return fail(SPDP_E_DATA, "%s: invalid candidate tour or costs (status %u)", fn, h[HDR_STATUS]);
    }
    nbr_prep_kernel<<<T, 32, 0, st>>>(tours, parents, n, dist, ld, e, info, parent_of, P);
    if ((rc = last_launch("nbr_prep_kernel"))) return rc;
    if (flags & SPDP_F_NBR_AUTO) {
        // whole-call choice: when the candidates' changed spans average more than kNbrAutoSpan of the
        // tour, the batched sweep is faster (measured crossover at C3): read the spans back
        std::vector<int4> h((size_t)T);
        if ((rc = cuda_check(cudaMemcpyAsync(h.data(), info, sizeof(int4) * (size_t)T, cudaMemcpyDeviceToHost, st),
                             "memcpy(info)")))
            return rc;
        if ((rc = cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
        double span = 0.0;
        for (int32_t t = 0; t < T; ++t) span += (double)(h[(size_t)t].y - h[(size_t)t].x);
        if (span > kNbrAutoSpan * (double)T * (double)n)
            return spdp_split_eval_batch(tours, T, dist, n, demand, ld, S, Q, cost, partial, window_hint, ws, ws_bytes,
                                         flags & ~(SPDP_F_NBR_AUTO | SPDP_F_NBR_SMEM | SPDP_F_VALIDATE), stream);
    }
    const int Qe = (int)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    spdp_saa_partial* slots = partial ? reinterpret_cast<spdp_saa_partial*>(w + L.slots) : nullptr;
    unsigned long long* ovf = reinterpret_cast<unsigned long long*>(w + L.ovf);
    unsigned* ovf_count = hdr + HDR_OVF_COUNT;
    if (flags & SPDP_F_NBR_SMEM) {  // the shared-memory ring (W = 32, or 64 for hinted windows above 32)
        rc = (window_hint > 32) ? launch_nbr_smem_t<64>(st, e, info, n, demand, S, T, Qe, fwd, bwd, cost, slots, ovf, ovf_count)
                                : launch_nbr_smem_t<32>(st, e, info, n, demand, S, T, Qe, fwd, bwd, cost, slots, ovf, ovf_count);
    } else {  // the register ring: 16 entries up to a hinted window of 24 (measured faster than 24 or 32
              // entries at C3 even with the overflow lanes it sends to the finish kernel), else 32
        const TourInfo* tinfo = reinterpret_cast<const TourInfo*>(w + L.tinfo);
        // the fp32 phase: every load value it forms, (n + W) Qe + Q + 1, below 2^23 (exact floats)
        const int f32 = ((flags & SPDP_F_SWEEP_INT) == 0 &&
                         ((int64_t)n + 32) * (int64_t)Qe + (int64_t)Qe + 1 < (1LL << 23)) ? 1 : 0;
        if (window_hint != 0 && window_hint <= 24)
            rc = launch_nbr_t<16>(st, e, info, n, demand, S, T, Qe, fwd, bwd, cost, slots, ovf, ovf_count, tinfo, f32);
        else
            rc = launch_nbr_t<32>(st, e, info, n, demand, S, T, Qe, fwd, bwd, cost, slots, ovf, ovf_count, tinfo, f32);
    }
    if (rc) return rc;
    return launch_finish(w, L, T, n, demand, ld, S, (uint32_t)Qe, cost, partial, false, st);
}

extern "C" spdp_status spdp_split_eval_neighbours(const int32_t* parent, const int32_t* fwd, const int32_t* bwd,
                                                  const int32_t* tours, int32_t T, const int32_t* dist, int32_t n,
                                                  const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                                  int32_t* cost, spdp_saa_partial* partial, int32_t window_hint,
                                                  void* ws, size_t ws_bytes, uint32_t flags, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval_neighbours");
    return spdp_split_eval_neighbours_multi(parent, 1, nullptr, fwd, bwd, tours, T, dist, n, demand, ld, S, Q, cost,
                                            partial, window_hint, ws, ws_bytes, flags, stream);
}
