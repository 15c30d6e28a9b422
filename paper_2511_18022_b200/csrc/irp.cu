// irp.cu -- a9/a10: inventory-routing recourse DP (PAPER:7 names the
// application and its "three-dimensional GPU parallelism"; the model is
// SURVEY §8(c6), DESIGN R21).
//
// Per scenario s and customer m, forward over periods t = 0..H-1 with state I
// (inventory) in [0, U]:
//   step A (delivery, masked min-plus over the band I in [y - z X, y]):
//       W[y] = min_I V[I] + c (y - I) = c y + min_I (V[I] - c I)
//   step B (demand d, lost sales):
//       V'[J] = W[J + d] + h J            (1 <= J, J + d <= U)
//       V'[0] = b d + min_{y <= min(d,U)} (W[y] - b y)
// cost_s = sum_m min_J V_H[J].
//
// Parallel layout (the "3-D" of PAPER:7): (scenario x customer) -> warps,
// inventory state y -> lanes (K consecutive states per lane, in registers),
// the band of step A -> a warp prefix-min scan when X >= U (the band is
// [0, y]) or an explicit band loop otherwise; periods are the sequential
// layers.  A warp takes a tile of 32 scenarios of one customer: the tile's
// demands [H][32] are staged in shared memory with coalesced loads.
#include <climits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace spdp {

constexpr int32_t kIrpInf = 1 << 30;  // "unreachable"; all real values are < 2^29 (host check)

struct IrpCust {
    int32_t U, X, I0, h, b, c;
};

template <int K>
__global__ void __launch_bounds__(128) irp_kernel(const uint8_t* __restrict__ visit, const IrpCust* __restrict__ cust,
                                                  int H, int M, const uint16_t* __restrict__ demand, int64_t ld,
                                                  int64_t S, long long* __restrict__ cost) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // per warp: demand tile [H][32] u16, then W buffer [32*K] int32
    uint16_t* dtile = reinterpret_cast<uint16_t*>(smem_raw) + (size_t)wid * (H * 32 + 2 * 32 * K);
    int32_t* wbuf = reinterpret_cast<int32_t*>(dtile + H * 32);
    const int64_t ntile = (S + 31) / 32;
    const int64_t ntask = ntile * M;
    for (int64_t task = (int64_t)blockIdx.x * nw + wid; task < ntask; task += (int64_t)gridDim.x * nw) {
        const int m = (int)(task % M);
        const int64_t s0 = (task / M) * 32;
        const IrpCust p = cust[m];
        for (int t = 0; t < H; ++t) {
            const int64_t s = s0 + lane;
            dtile[t * 32 + lane] = (s < S) ? demand[((int64_t)t * M + m) * ld + s] : (uint16_t)0;
        }
        __syncwarp();
        const int jmax = (int)((S - s0) < 32 ? (S - s0) : 32);
        for (int j = 0; j < jmax; ++j) {
            int32_t v[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int y = lane * K + k;
                v[k] = (y == p.I0) ? 0 : kIrpInf;
            }
            for (int t = 0; t < H; ++t) {
                const int d = dtile[t * 32 + j];
                const bool vis = visit[(int64_t)m * H + t] != 0;
                // ---- step A
                if (vis && p.X > 0) {
                    if (p.X >= p.U) {
                        // band [0, y]: prefix-min of V[I] - c I, then + c y
                        int32_t run = kIrpInf;
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const int y = lane * K + k;
                            const int32_t a = (v[k] >= kIrpInf) ? kIrpInf : v[k] - p.c * y;
                            run = min(run, a);
                            v[k] = run;  // lane-local inclusive prefix-min
                        }
                        int32_t carry = run;  // inclusive scan of lane totals
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int32_t u = __shfl_up_sync(kFull, carry, o);
                            if (lane >= o) carry = min(carry, u);
                        }
                        int32_t excl = __shfl_up_sync(kFull, carry, 1);
                        if (lane == 0) excl = kIrpInf;
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const int y = lane * K + k;
                            const int32_t mn = min(v[k], excl);
                            v[k] = (mn >= kIrpInf / 2) ? kIrpInf : mn + p.c * y;
                        }
                    } else {
                        // explicit band [max(0, y - X), y] (DESIGN: general X < U path)
#pragma unroll
                        for (int k = 0; k < K; ++k) wbuf[lane * K + k] = v[k];
                        __syncwarp();
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const int y = lane * K + k;
                            int32_t best = kIrpInf;
                            if (y <= p.U) {
                                for (int I = max(0, y - p.X); I <= y; ++I) {
                                    const int32_t a = wbuf[I];
                                    if (a < kIrpInf) best = min(best, a + p.c * (y - I));
                                }
                            }
                            v[k] = best;
                        }
                        __syncwarp();
                    }
                }
                // states above U are never reachable
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (lane * K + k > p.U) v[k] = kIrpInf;
                // ---- step B
                int32_t m0 = kIrpInf;  // min_{y <= min(d,U)} W[y] - b y
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int y = lane * K + k;
                    wbuf[y] = v[k];
                    if (y <= d && v[k] < kIrpInf) m0 = min(m0, v[k] - p.b * y);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) m0 = min(m0, __shfl_xor_sync(kFull, m0, o));
                __syncwarp();
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int J = lane * K + k;
                    int32_t nv;
                    if (J == 0) {
                        nv = (m0 >= kIrpInf) ? kIrpInf : m0 + p.b * d;
                    } else if (J + d <= p.U) {
                        const int32_t wv = wbuf[J + d];
                        nv = (wv >= kIrpInf) ? kIrpInf : wv + p.h * J;
                    } else {
                        nv = kIrpInf;
                    }
                    v[k] = nv;
                }
                __syncwarp();
            }
            int32_t best = kIrpInf;
#pragma unroll
            for (int k = 0; k < K; ++k) best = min(best, v[k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
            if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&cost[s0 + j]), (unsigned long long)best);
        }
        __syncwarp();
    }
}

// Lane-per-scenario variant (used when every customer has X == 0 or X >= U, so the
// delivery band of step A is the prefix [0, y]).  A warp owns 32 scenarios (one per
// lane) and loops over customers and periods; the inventory states of each lane live
// in shared memory ([U+1][32], lane-contiguous, conflict-free).  Step A and step B
// are fused into ONE in-place pass over y = 0..U:
//     run  = min(run, V[y] - c y)                 prefix-min of the band (X >= U)
//     W    = run + c y                             (= V[y] when the period is not visited)
//     m0   = min(m0, W - b y)        if y <= d     V'[0] = m0 + b d
//     V[y - d] = W + h (y - d)       if y - d >= 1 (index y - d was already read)
// States above `top` are unreachable (+inf) and are never read.  Values stay below
// 2^29 (host check) and the sentinel is 2^30, so sums never overflow and no special
// casing of +inf is needed: every result is clamped with one min at the end.
__global__ void __launch_bounds__(256) irp_lane_kernel(const uint8_t* __restrict__ visit,
                                                       const IrpCust* __restrict__ cust, int H, int M, int Umax,
                                                       const uint16_t* __restrict__ demand, int64_t ld, int64_t S,
                                                       long long* __restrict__ cost) {
    extern __shared__ int32_t vsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int32_t* V = vsm + (size_t)wid * (Umax + 1) * 32 + lane;  // V[y] at V[y * 32]
    const int64_t ntile = (S + 31) / 32;
    for (int64_t tile = (int64_t)blockIdx.x * nw + wid; tile < ntile; tile += (int64_t)gridDim.x * nw) {
        const int64_t s0 = tile * 32;
        const bool live = s0 + lane < S;
        const int64_t s = live ? s0 + lane : S - 1;
        long long total = 0;
        for (int m = 0; m < M; ++m) {
            const IrpCust p = cust[m];
            const int U = p.U;
            for (int y = 0; y <= U; ++y) V[y * 32] = kIrpInf;
            V[p.I0 * 32] = 0;
            int top = U;  // states above top are +inf
            int d = demand[(int64_t)m * ld + s];
            for (int t = 0; t < H; ++t) {
                const int dn = (t + 1 < H) ? demand[((int64_t)(t + 1) * M + m) * ld + s] : 0;  // prefetch
                const bool deliver = visit[(int64_t)m * H + t] != 0 && p.X > 0;
                const int ylim = deliver ? U : top;
                int run = kIrpInf, m0 = kIrpInf;
                for (int y = 0; y <= ylim; ++y) {
                    const int v = (y <= top) ? V[y * 32] : kIrpInf;
                    int w;
                    if (deliver) {
                        run = min(run, v - p.c * y);
                        w = run + p.c * y;
                    } else {
                        w = v;
                    }
                    if (y <= d) m0 = min(m0, w - p.b * y);
                    const int J = y - d;
                    if (J >= 1) V[J * 32] = min(w + p.h * J, kIrpInf);
                }
                V[0] = min(m0 + p.b * d, kIrpInf);
                top = max(0, ylim - d);
                d = dn;
            }
            int best = kIrpInf;
            for (int y = 0; y <= top; ++y) best = min(best, V[y * 32]);
            total += best;
        }
        if (live) cost[s] = total;
    }
}

// Lane-per-scenario variant with a LAZY demand shift and an AFFINE TAIL (same results as
// irp_lane_kernel; DESIGN §6 "IRP").  Per (scenario, customer) the value function is kept as
//     V[J] = A[(J + off) mod B] + alpha J + K     J in [0, E]   (explicit, B = U + 1, per lane)
//     V[J] = Ta + Ts J                             J in (E, F]   (affine tail)
//     V[J] = +inf                                  J in (F, U]
// Step B (demand d) is exact on this form in O(min(d, E)):
//     V'[J] = V[J + d] + h J  ==>  off += d, K += alpha d, alpha += h; Ta += Ts d, Ts += h;
//                                  E -= d (>= 0), F -= d (>= E)
//     V'[0] = b d + min_{y <= min(d, U)} (V[y] - b y): explicit y by a scan, the tail y in
//             (E, min(d, F)] at its two ends (affine)             written at A[off'] - K'.
// Step A (delivery, band [0, y]: X >= U) is W[y] = min(W[y - 1] + c, V[y]) (W[-1] = +inf).  The
// tail always satisfies V[E + 1] >= V[E] + c and has slope Ts >= c (*) (and +inf above F needs no
// condition), so for y > E the
// recursion takes W[y - 1] + c every time: W[y] = W[E] + c (y - E) up to U.  A delivery therefore
// rewrites only the explicit entries (O(E)), then sets Ta = W[E] - c E, Ts = c, F = U,
// alpha = K = 0.  (*) holds after a delivery with equality and is kept by step B: a shift adds
// h >= 0 to every difference, and a new V'[0] (the minimum above includes y = min(d, E) or the
// tail's first point) never exceeds the value it sits next to.  E never grows: it starts at I0
// (V_0 = [I0]: nothing above is reachable yet) and loses every period's demand, so once a
// customer's cumulative demand passes I0 its DP is O(1) per period.  Sentinels: values >= 2^29 are unreachable (host check: every real value is
// below); explicit unreachable entries are stored as 2^30 and reads add alpha J + K < 2^29.
//
// Layout: the ring needs only B = I0 + 1 slots (the explicit region never leaves [0, I0]), per warp
// [Bmax][32] int32 lane-interleaved (conflict-free), then the task's demands [H][32] u16 staged in
// one burst of coalesced loads (the per-period reads are then shared-memory hits), and the
// customer's visit pattern as a bit mask built by two ballots (H <= 64; else read per period).
__global__ void __launch_bounds__(128) irp_lazy_kernel(const uint8_t* __restrict__ visit,
                                                       const IrpCust* __restrict__ cust, int H, int M, int Bmax,
                                                       const uint16_t* __restrict__ demand, int64_t ld, int64_t S,
                                                       long long* __restrict__ cost) {
    extern __shared__ int32_t vsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const size_t dt_words = (size_t)(H + 1) / 2 * 32;  // the demand tile [H][32] u16 (rounded to 2 rows)
    const size_t warp_words = (size_t)Bmax * 32 + dt_words;
    int32_t* A = vsm + (size_t)wid * warp_words + lane;  // A[x] at A[x * 32]
    uint32_t* dtw = reinterpret_cast<uint32_t*>(vsm + (size_t)wid * warp_words + (size_t)Bmax * 32);
    constexpr int32_t kReal = 1 << 29;                        // values >= kReal are unreachable
    const int64_t ntile = (S + 31) / 32;
    const int64_t ntask = ntile * M;
    // the demand tile of a task, [H][32] u16, by cp.async (4 B = 2 scenarios per copy; lanes 0-15 row
    // t, lanes 16-31 row t + 1; columns at or past ld read as zeros): all H / 2 copies of a lane in
    // flight at once.  (Staging the next task's tile during this one, in a second buffer with a
    // persistent grid, measured slower: 0.19-0.20 vs 0.18 ms at C5 -- the extra shared memory costs
    // more resident warps than the hidden latency gains.)
    auto stage = [&](int64_t task, uint32_t* buf) {
        const int64_t tl = task / M;
        const int mm = (int)(task - tl * M);
        const int64_t col = tl * 32 + 2 * (lane & 15);
        for (int t = lane >> 4; t < H; t += 2) {
            const bool in = col < ld;
            const uint16_t* src = demand + ((int64_t)t * M + mm) * ld + (in ? col : 0);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(buf + t * 16 + (lane & 15))),
                         "l"(src), "r"(in ? 4 : 0) : "memory");
        }
    };
    // one warp task = (32-scenario tile, customer): M times more independent warps than tiles, so
    // the launch fills every SM several times over; the customer costs are summed with atomics
    // into cost[] (zeroed by the host code)
    for (int64_t task = (int64_t)blockIdx.x * nw + wid; task < ntask; task += (int64_t)gridDim.x * nw) {
        const int64_t tile = task / M;
        const int m = (int)(task - tile * M);
        const int64_t s0 = tile * 32;
        const bool live = s0 + lane < S;
        const int64_t s = live ? s0 + lane : S - 1;
        const IrpCust p = cust[m];
        const int U = p.U, B = p.I0 + 1;
        const int32_t* const aend = A + B * 32;  // (one past the last ring slot of this lane)
        __syncwarp();  // (the previous task's reads of the tile are done)
        stage(task, dtw);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        const uint16_t* dt = reinterpret_cast<const uint16_t*>(dtw) + lane;  // dt[t * 32]
        const bool vis_lo = lane < H && visit[(int64_t)m * H + lane] != 0;
        const bool vis_hi = lane + 32 < H && visit[(int64_t)m * H + lane + 32] != 0;
        const unsigned long long vmask =
            p.X > 0 ? ((unsigned long long)__ballot_sync(kFull, vis_hi) << 32) | __ballot_sync(kFull, vis_lo) : 0ull;
        // V_0 = [I0]: explicit [0, I0] (+inf below I0), +inf above (no tail: F = E)
        for (int y = 0; y <= p.I0; ++y) A[y * 32] = (y == p.I0) ? 0 : kIrpInf;
        int off = 0, E = p.I0, F = p.I0;  // explicit [0, E], affine tail (E, F]
        int32_t alpha = 0, K = 0, Ta = 0, Ts = 0;
        int t = 0;
        for (; t < H; ++t) {
            if (__all_sync(kFull, E == 0)) break;  // every lane's explicit region is {0}: register loop below
            const int d = dt[t * 32];
            const bool deliver = t < 64 ? ((vmask >> t) & 1ull) != 0ull : (p.X > 0 && visit[(int64_t)m * H + t] != 0);
            if (deliver) {  // (warp-uniform)
                int32_t R = kIrpInf, u = K;  // u = alpha y + K
                int32_t* ap = A + off * 32;  // slot (y + off) mod B, a pointer stepping with wrap
#pragma unroll 1
                for (int y = 0; y <= E; ++y) {
                    R = min(R + p.c, *ap + u);
                    *ap = R >= kReal ? kIrpInf : R;
                    u += alpha;
                    ap += 32;
                    if (ap == aend) ap = A;
                }
                if (E < U && R < kReal) {  // W[y] = W[E] + c (y - E) for y in (E, U]
                    Ta = R - p.c * E;
                    Ts = p.c;
                    F = U;
                } else {
                    F = E;  // (no tail: E == U, or nothing reachable)
                }
                alpha = 0;
                K = 0;
            }
            // demand d: V'[0] = b d + min_{y <= min(d, U)} (V[y] - b y); V'[J] = V[J + d] + h J
            int32_t m0 = kIrpInf;
            {
                const int ylim = d < E ? d : E;
                const int32_t du = alpha - p.b;
                int32_t u = K;  // (alpha - b) y + K
                const int32_t* ap = A + off * 32;
                int y = 0;
#pragma unroll 1
                for (; y + 1 <= ylim; y += 2) {  // two states per trip (the loop is per lane: its length is)
                    const int32_t* ap1 = ap + 32 == aend ? A : ap + 32;
                    m0 = min(m0, min(*ap + u, *ap1 + u + du));
                    u += 2 * du;
                    ap = ap1 + 32 == aend ? A : ap1 + 32;
                }
                if (y <= ylim) m0 = min(m0, *ap + u);
            }
            if (d > E && F > E) {  // the tail's part of the minimum: an affine function, at its ends
                const int y2 = d < F ? d : F;
                m0 = min(m0, Ta + (Ts - p.b) * (E + 1));
                m0 = min(m0, Ta + (Ts - p.b) * y2);
            }
            const int dd = d < B ? d : B;  // (a shift by >= B leaves only J = 0; K is then relative)
            K += alpha * dd;
            alpha += p.h;
            off += dd;
            if (off >= B) off -= B;
            const int En = d <= E ? E - d : 0;
            const int Fn = F - d > En ? F - d : En;
            if (Fn > En) {  // the tail survives the shift (then d < F <= U: no overflow)
                Ta += Ts * d;
                Ts += p.h;
            }
            E = En;
            F = Fn;
            const int32_t v0 = (m0 >= kReal) ? kIrpInf : m0 + p.b * d;
            A[off * 32] = (v0 >= kReal) ? kIrpInf : v0 - K;
        }
        int32_t best = F > E ? Ta + Ts * (E + 1) : kIrpInf;  // (the tail's minimum: slope Ts >= 0)
        if (t < H) {
            // collapsed: E == 0 in every lane, so the explicit part is the one value V0 = V[0] (in a
            // register) and a period is O(1): the same steps as above with E = 0
            int32_t V0 = A[off * 32] + K;
            for (; t < H; ++t) {
                const int d = dt[t * 32];
                const bool deliver = t < 64 ? ((vmask >> t) & 1ull) != 0ull : (p.X > 0 && visit[(int64_t)m * H + t] != 0);
                if (deliver) {
                    if (U > 0 && V0 < kReal) {  // W[y] = V0 + c y
                        Ta = V0;
                        Ts = p.c;
                        F = U;
                    } else {
                        F = 0;
                    }
                }
                int32_t m0 = V0;
                if (d > 0 && F > 0) {
                    const int y2 = d < F ? d : F;
                    m0 = min(m0, min(Ta + (Ts - p.b), Ta + (Ts - p.b) * y2));
                }
                const int Fn = F - d > 0 ? F - d : 0;
                if (Fn > 0) {
                    Ta += Ts * d;
                    Ts += p.h;
                }
                F = Fn;
                const int32_t v0 = (m0 >= kReal) ? kIrpInf : m0 + p.b * d;
                V0 = (v0 >= kReal) ? kIrpInf : v0;
            }
            best = min(F > 0 ? Ta + Ts : kIrpInf, V0);
        } else {
            int x = off;
            for (int y = 0; y <= E; ++y) {
                best = min(best, A[x * 32] + alpha * y + K);
                x = (x + 1 == B) ? 0 : x + 1;
            }
        }
        if (live) atomicAdd(reinterpret_cast<unsigned long long*>(&cost[s]), (unsigned long long)(long long)best);
    }
}

__global__ void __launch_bounds__(256) irp_reduce_kernel(const long long* __restrict__ cost, int64_t S,
                                                         spdp_saa_partial* __restrict__ partial) {
    __shared__ Part red[8];
    Part p{0, 0, 0, 0, 0};
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x)
        part_add_cost(p, cost[s], true);
    Part r = block_sum(p, red);
    if (threadIdx.x == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_feas), (unsigned long long)r.n_feas);
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sum), (unsigned long long)r.sum);
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_lo), (unsigned long long)r.sq_lo);
        atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_hi), (unsigned long long)r.sq_hi);
    }
}

template <int K>
static spdp_status launch_irp(const uint8_t* visit, const IrpCust* cust, int H, int M, const uint16_t* demand,
                              int64_t ld, int64_t S, long long* cost, cudaStream_t st) {
    const int warps = 4;
    const size_t smem = (size_t)warps * (sizeof(uint16_t) * H * 32 + sizeof(int32_t) * 32 * K);
    if (spdp_status e = kernel_setup((const void*)irp_kernel<K>, 200 * 1024, -1, 0, 0, nullptr, "irp_kernel setup")) return e;
    const int64_t ntask = ((S + 31) / 32) * M;
    int64_t blocks = ceil_div(ntask, warps);
    if (blocks > (int64_t)device_sms() * 16) blocks = (int64_t)device_sms() * 16;
    prof_begin(st);
    irp_kernel<K><<<(unsigned)blocks, warps * 32, smem, st>>>(visit, cust, H, M, demand, ld, S, cost);
    spdp_status rc = last_launch("irp_kernel");
    set_last_kernel("irp_kernel<%d>", K);
    prof_end(st);
    return rc;
}

}  // namespace spdp

using namespace spdp;

extern "C" size_t spdp_irp_workspace_bytes(int32_t H, int32_t M, int64_t S) {
    (void)S;
    if (H < 1 || M < 1) return 0;
    return align_up(sizeof(IrpCust) * (size_t)M, 256) + align_up((size_t)M * (size_t)H, 256);
}

extern "C" spdp_status spdp_irp_dp(const uint8_t* visit_h, const spdp_irp_customer* cust_h, int32_t H, int32_t M,
                                   const uint16_t* demand, int64_t ld, int64_t S, int64_t* cost,
                                   spdp_saa_partial* partial, void* ws, size_t ws_bytes, uint32_t flags,
                                   spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_irp_dp");
    if (H < 1 || M < 1 || S < 1) return fail(SPDP_E_USAGE, "spdp_irp_dp: H, M, S must be >= 1");
    if (!visit_h || !cust_h || !demand || !cost || !ws) return fail(SPDP_E_USAGE, "spdp_irp_dp: NULL pointer");
    if (ld < S) return fail(SPDP_E_USAGE, "spdp_irp_dp: ld < S");
    if (ws_bytes < spdp_irp_workspace_bytes(H, M, S)) return fail(SPDP_E_USAGE, "spdp_irp_dp: workspace too small");
    int Umax = 0;
    long long total_bound = 0;  // bound on a scenario's cost (the sum over customers)
    for (int m = 0; m < M; ++m) {
        const spdp_irp_customer& c = cust_h[m];
        if (c.U < 0 || c.X < 0 || c.I0 < 0 || c.I0 > c.U || c.h < 0 || c.b < 0 || c.c < 0)
            return fail(SPDP_E_DATA, "spdp_irp_dp: customer %d has invalid parameters", m);
        // every reachable value <= H (c X + h U + b 65535) must stay below 2^29
        const long long bound = (long long)H * ((long long)c.c * c.X + (long long)c.h * c.U + (long long)c.b * 65535LL);
        if (bound >= (1LL << 29)) return fail(SPDP_E_RESOURCE, "spdp_irp_dp: cost bound %lld exceeds int32 kernel range", bound);
        total_bound += bound;
        Umax = c.U > Umax ? c.U : Umax;
    }
    // the SAA partial squares each cost into the summable {sumsq_lo, sumsq_hi} halves, which stay
    // exact while cost^2 < 2^62 (spdp_saa_partial): reject larger totals rather than wrap
    if (partial && total_bound >= (1LL << 31))
        return fail(SPDP_E_RESOURCE, "spdp_irp_dp: cost bound %lld (sum over customers) >= 2^31: the SAA partial "
                    "would overflow (pass partial = NULL and reduce the int64 costs elsewhere)", total_bound);
    if (Umax + 1 > 32 * 32) return fail(SPDP_E_RESOURCE, "spdp_irp_dp: U=%d > 1023", Umax);
    cudaStream_t st = (cudaStream_t)stream;
    char* w = static_cast<char*>(ws);
    IrpCust* dcust = reinterpret_cast<IrpCust*>(w);
    uint8_t* dvisit = reinterpret_cast<uint8_t*>(w + align_up(sizeof(IrpCust) * (size_t)M, 256));
    spdp_status rc;
    if ((rc = cuda_check(cudaMemcpyAsync(dcust, cust_h, sizeof(IrpCust) * M, cudaMemcpyHostToDevice, st), "H2D cust"))) return rc;
    if ((rc = cuda_check(cudaMemcpyAsync(dvisit, visit_h, (size_t)M * H, cudaMemcpyHostToDevice, st), "H2D visit"))) return rc;
    long long* c = reinterpret_cast<long long*>(cost);
    bool prefix_band = true;  // every customer's delivery band is [0, y] (or empty)
    for (int m = 0; m < M; ++m) prefix_band &= (cust_h[m].X == 0 || cust_h[m].X >= cust_h[m].U);
    const size_t lane_smem_warp = sizeof(int32_t) * 32 * (size_t)(Umax + 1);
    int I0max = 0;
    for (int m = 0; m < M; ++m) I0max = cust_h[m].I0 > I0max ? cust_h[m].I0 : I0max;
    const size_t lazy_smem_warp = sizeof(int32_t) * 32 * ((size_t)(I0max + 1) + (size_t)(H + 1) / 2);
    const int irp_mode = (flags & SPDP_F_IRP_EAGER) ? 1 : 0;  // the eager-shift lane kernel instead of the lazy one
    const bool states = (flags & SPDP_F_IRP_STATES) != 0;  // force the state-parallel kernel
    if (prefix_band && lazy_smem_warp <= 48 * 1024 && irp_mode == 0 && !states) {
        // lazy-shift lane kernel: 4 warps per CTA, several CTAs per SM
        // one task per warp (the hardware fills SMs as tasks finish; tasks are short and uneven)
        const int warps = 4;
        if ((rc = kernel_setup((const void*)irp_lazy_kernel, 200 * 1024, 100, 0, 0, nullptr, "irp_lazy setup"))) return rc;
        const int64_t ntask = ((S + 31) / 32) * M;
        const int64_t blocks = (ntask + warps - 1) / warps;
        if ((rc = cuda_check(cudaMemsetAsync(c, 0, sizeof(long long) * (size_t)S, st), "cudaMemsetAsync(cost)"))) return rc;
        prof_begin(st);
        irp_lazy_kernel<<<(unsigned)blocks, warps * 32, lazy_smem_warp * warps, st>>>(dvisit, dcust, H, M, I0max + 1, demand,
                                                                                     ld, S, c);
        rc = last_launch("irp_lazy_kernel");
        set_last_kernel("irp_lazy_kernel");
        prof_end(st);
    } else if (prefix_band && lane_smem_warp <= 96 * 1024 && !states) {
        int warps = (int)((192 * 1024) / lane_smem_warp);
        warps = warps < 1 ? 1 : (warps > 8 ? 8 : warps);
        if ((rc = kernel_setup((const void*)irp_lane_kernel, 200 * 1024, 100, 0, 0, nullptr, "irp_lane setup"))) return rc;
        const int64_t ntile = (S + 31) / 32;
        int64_t blocks = (ntile + warps - 1) / warps;
        prof_begin(st);
        irp_lane_kernel<<<(unsigned)blocks, warps * 32, lane_smem_warp * warps, st>>>(dvisit, dcust, H, M, Umax, demand,
                                                                                     ld, S, c);
        rc = last_launch("irp_lane_kernel");
        set_last_kernel("irp_lane_kernel");
        prof_end(st);
    } else {
    if ((rc = cuda_check(cudaMemsetAsync(cost, 0, sizeof(int64_t) * (size_t)S, st), "memset cost"))) return rc;
    const int need = Umax + 1;
    if (need <= 32) rc = launch_irp<1>(dvisit, dcust, H, M, demand, ld, S, c, st);
    else if (need <= 64) rc = launch_irp<2>(dvisit, dcust, H, M, demand, ld, S, c, st);
    else if (need <= 128) rc = launch_irp<4>(dvisit, dcust, H, M, demand, ld, S, c, st);
    else if (need <= 256) rc = launch_irp<8>(dvisit, dcust, H, M, demand, ld, S, c, st);
    else if (need <= 512) rc = launch_irp<16>(dvisit, dcust, H, M, demand, ld, S, c, st);
    else rc = launch_irp<32>(dvisit, dcust, H, M, demand, ld, S, c, st);
    }
    if (rc) return rc;
    if (partial) {
        if ((rc = cuda_check(cudaMemsetAsync(partial, 0, sizeof(spdp_saa_partial), st), "memset partial"))) return rc;
        int64_t blocks = ceil_div(S, 256 * 8);
        if (blocks > (int64_t)device_sms() * 8) blocks = (int64_t)device_sms() * 8;
        irp_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(c, S, partial);  // (|cost| < 2^31: checked above)
        if ((rc = last_launch("irp_reduce_kernel"))) return rc;
    }
    return SPDP_OK;
}
