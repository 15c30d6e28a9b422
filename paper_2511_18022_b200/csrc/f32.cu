// f32.cu -- the fp32 mode of the split (SURVEY §8(a) a2 / a5 "fp32 (one add + exact min)",
// §8(c3) "fp32 mode (secondary)"; DESIGN R25): real-valued route costs.
//
//   Dd[1] = 0, Dd[i] = Dd[i-1] + c[s_{i-1}][s_i]               (fp64, sequential: one thread)
//   T32(p, i) = fl32((c[0][s_{p+1}] + (Dd[i] - Dd[p+1])) + c[s_i][0])   (Eq. (1)'s route cost,
//               rounded once from fp64)
//   f(0) = 0,  f(i) = min_{mask(i) <= p <= i-1} fl32(f(p) + T32(p, i))
//
// Unlike the integer mode the rounded route cost is not separable into A[p] + B[i], so each
// candidate forms T32 from the tour's fp64 prefix table (two fp64 adds and one rounding, in
// the oracle's order) and adds it to f(p) with one IEEE single add; the min is exact.  The
// result is therefore bit-identical to oracle_split_f32 for any launch configuration.
#include <climits>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "split_ws.cuh"
#include "tma.cuh"

namespace spdp {

struct F32Pos {
    double Dd, c0, ci0;  // Dd[i], c[0][s_i], c[s_i][0]
    uint32_t rowoff;     // (s_i - 1) * ld (n ld < 2^32)
    uint32_t pad;
};

constexpr int kF32SmemMaxN = 4095;  // position table in shared memory up to 128 KB

// (also: the TMA sweep's gather rows trow[i] = demand row of tour position i + 1 (i < n), n past the
// end, for i < len; and the zeroed list counters count[0..1])
__global__ void __launch_bounds__(256) f32_prep_kernel(const int32_t* __restrict__ tour, int n,
                                                       const double* __restrict__ dist, int64_t ld,
                                                       F32Pos* __restrict__ tab, int32_t* __restrict__ trow, int len,
                                                       unsigned* __restrict__ count) {
    if (blockIdx.x != 0) return;
    const int64_t N1 = (int64_t)n + 1;
    auto node = [&](int i) -> int {  // customer at 0-based position i, clamped to 1..n
        const int c = tour[i];
        return c < 1 ? 1 : (c > n ? n : c);
    };
    if (threadIdx.x < 2) count[threadIdx.x] = 0u;
    if (trow)
        for (int i = threadIdx.x; i < len; i += blockDim.x) trow[i] = i < n ? node(i) - 1 : n;
    // every position's costs in parallel (Dd temporarily holds the arc into position i)
    for (int i = threadIdx.x; i <= n; i += blockDim.x) {
        if (i == 0) {
            tab[0] = F32Pos{0.0, 0.0, 0.0, 0u, 0u};
            continue;
        }
        const int c = node(i - 1);
        const double arc = i >= 2 ? dist[(int64_t)node(i - 2) * N1 + c] : 0.0;
        tab[i] = F32Pos{arc, dist[c], dist[(int64_t)c * N1], (uint32_t)((uint64_t)(c - 1) * (uint64_t)ld), 0u};
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    // Dd[1] = 0, Dd[i] = Dd[i-1] + c[s_{i-1}][s_i]: the fp64 sum in the oracle's (sequential) order
    double D = 0.0;
    for (int i = 1; i <= n; ++i) {
        if (i >= 2) D = __dadd_rn(D, tab[i].Dd);
        tab[i].Dd = D;
    }
}

// The general kernel (any window; the scenarios the ring kernel deferred, or all of them): one
// scenario per thread, two-pointer mask, f in the thread's own rows of the
// workspace ([n+1][S] fp32, coalesced across the warp), T32 formed per candidate.
__global__ void __launch_bounds__(256) split_f32_kernel(const F32Pos* __restrict__ tab_g, int n,
                                                        const uint16_t* __restrict__ demand, int64_t S, int Q,
                                                        float* fsc, float* __restrict__ cost, int table_in_smem,
                                                        const int64_t* __restrict__ list,
                                                        const unsigned* __restrict__ count) {
    extern __shared__ F32Pos ftab[];
    const F32Pos* tab = tab_g;
    const int64_t nw = list ? (int64_t)*count : S;
    if ((int64_t)blockIdx.x * blockDim.x >= nw) return;  // (block-uniform: before the table copy)
    if (table_in_smem) {
        for (int i = threadIdx.x; i <= n; i += blockDim.x) ftab[i] = tab_g[i];
        __syncthreads();
        tab = ftab;
    }
    // (list mode: a grid of a few CTAs per SM strides over the listed scenarios)
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = list ? list[w] : w;
        const uint16_t* dcol = demand + s;
        float* fc = fsc + s;
        fc[0] = 0.0f;
        int P = 0, Pm = 0, m = 0;
        bool bad = false;
        for (int i = 1; i <= n && !bad; ++i) {
            const int q = dcol[tab[i].rowoff];
            if (q > Q) {  // Eq. (2)'s set is empty from here on (DESIGN R4)
                bad = true;
                break;
            }
            P += q;
            while (P - Pm > Q) Pm += dcol[tab[++m].rowoff];  // P(m) = sum_{k<=m} q; stops at m <= i-1
            const double Di = tab[i].Dd, ci0 = tab[i].ci0;
            float best = INFINITY;
            for (int p = i - 1; p >= m; --p) {
                const double t64 = __dadd_rn(__dadd_rn(tab[p + 1].c0, __dsub_rn(Di, tab[p + 1].Dd)), ci0);
                best = fminf(best, __fadd_rn(fc[(int64_t)p * S], __double2float_rn(t64)));
            }
            fc[(int64_t)i * S] = best;
        }
        cost[s] = bad ? INFINITY : fc[(int64_t)n * S];
    }
}

// ---------------------------------------------------------------- the TMA-fed fp32 ring sweep
// The common case (every scenario whose loads stay below 2^30; the rest, and the scenarios this
// kernel lists, go through split_f32_kernel): the packed-u16 sweep's work decomposition (split_u16.cu: persistent CTAs of 4 consumer
// warps + 1 producer warp, the producer gathering 4 tour-ordered demand rows x 128 scenarios per
// TMA instruction into an NS-stage shared-memory ring) with one scenario per lane and fp32 values.
// Per lane a W-entry register ring of {f(p), Y(p) = P(p) + Q} (split point p in slot p mod W).
// Candidate p of layer i (age k = i - p): val = fl32(f(p) + T32(p, i)) (one IEEE add of the
// band-table entry, staged per chunk next to the demand rows); d = Y(p) - P(i) >= 0 iff p is in
// the window, so d's sign bit is set exactly outside it, and
//   key = bits(val) | (d & 0x80000000)      (one LOP3)
// orders like val inside the window (val >= 0: IEEE order of non-negative floats is the order of
// their bit patterns) and above every in-window key outside it: the masked min of Eq. (3) is an
// unsigned 3-input integer min (VIMNMX3) of keys, exact.  Four layers per step (as in the u16
// sweep: the candidates made before the step first, one warp vote per deeper group of ages for all
// four layers), ages 1..A0 unconditionally; a window that reaches age W lists the scenario for
// split_f32_kernel.  Measured (C2, 10^6 scenarios): 0.61 ms (the previous one-thread-per-scenario
// ring with LDG demand loads) -> 0.153 ms; on a set ordered by total demand with longest-first tile
// claims (lpt_block) and A0 = 6: 0.130 ms (A0 = 5 / 7 / 8: 0.132 / 0.144 / 0.145 ms).
constexpr int kF32Cons = 4;                      // consumer warps per CTA
constexpr int kF32Threads = 32 * (kF32Cons + 1);
constexpr int kF32Tile = 32 * kF32Cons;          // scenarios per tile = TMA box columns
constexpr int kF32TW = 20;                       // ring width of the TMA sweep
constexpr int kF32TA0 = 6;                       // unconditional ages

template <int W, int NST>
struct F32TCfg {
    static constexpr int NS = NST;
    static constexpr int kRowBytes = kF32Tile * 2;                // 256 B
    static constexpr int kRowsBytes = W * kRowBytes;
    static constexpr int kBandOff = kRowsBytes;                   // W layers x W ages fp32
    static constexpr int kBandBytes = W * W * 4;
    static constexpr int kHdrOff = kBandOff + kBandBytes;         // {tile, chunk}
    static constexpr int kStageBytes = (kHdrOff + 16 + 127) / 128 * 128;
    static constexpr size_t kSmem = (size_t)NS * kStageBytes + 2 * NS * sizeof(uint64_t);
    static_assert(W % 4 == 0, "W must be a multiple of 4");
};

// band rows of the TMA sweep: tbw[i][k - 1] = T32(i - k, i), k = 1..W, rows i = 0 .. n + W (zero
// past n and for k > i), so a chunk's W rows are one contiguous bulk copy
__global__ void f32_bandw_kernel(const F32Pos* __restrict__ tab, int n, int W, float* __restrict__ tb) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)(n + 1 + W) * W) return;
    const int i = (int)(idx / W), k = (int)(idx % W) + 1;
    float v = 0.0f;
    if (i <= n && k <= i) {
        const int p = i - k;
        v = __double2float_rn(__dadd_rn(__dadd_rn(tab[p + 1].c0, __dsub_rn(tab[i].Dd, tab[p + 1].Dd)), tab[i].ci0));
    }
    tb[idx] = v;
}


__device__ __forceinline__ uint32_t f32_key(float val, uint32_t d) {
    uint32_t k;
    asm("lop3.b32 %0, %1, %2, %3, 0xF8;" : "=r"(k) : "r"(__float_as_uint(val)), "r"(d), "r"(0x80000000u));
    return k;  // val | (d & 0x80000000)
}

template <int N>
__device__ __forceinline__ uint32_t umin_tree32(const uint32_t* v);
// minimum of v[lo .. N - 1] (lo a compile-time constant after unrolling)
template <int N>
__device__ __forceinline__ uint32_t umin_tree32_from(const uint32_t* v, const int lo) {
    if (lo == 0) return umin_tree32<N>(v);
    if constexpr (N > 1) return umin_tree32_from<N - 1>(v + 1, lo - 1);
    return v[0];
}
template <int N>
__device__ __forceinline__ uint32_t umin_tree32(const uint32_t* v) {
    if constexpr (N == 1) return v[0];
    else if constexpr (N == 2) return min(v[0], v[1]);
    else if constexpr (N == 3) return __vimin3_u32(v[0], v[1], v[2]);
    else return __vimin3_u32(umin_tree32<N - 2>(v), v[N - 2], v[N - 1]);
}

template <int W, int A0, int UG, int NST, int LS>
__global__ void __launch_bounds__(kF32Threads) split_f32_tma_kernel(
    const __grid_constant__ CUtensorMap dmap, const int32_t* __restrict__ trow, const float* __restrict__ tbw, int n,
    int64_t S, int Q, float* __restrict__ cost, int64_t* __restrict__ list, unsigned* __restrict__ count) {
    using Cfg = F32TCfg<W, NST>;
    constexpr int NS = Cfg::NS;
    static_assert(A0 >= 2 && A0 <= W && UG >= 1 && W % LS == 0 && A0 >= LS + 1 && (LS == 2 || LS == 4), "bad fp32 sweep config");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + NS * Cfg::kStageBytes);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t ntiles = (uint32_t)((S + kF32Tile - 1) / kF32Tile);
    const int nchunks = (n + W - 1) / W;
    if (tid == 0) {
        for (int k = 0; k < NS; ++k) {
            mbar_init(&full[k], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (__any_sync(kFull, wid == kF32Cons)) {
        // ---- producer (see split_sweep_u16_kernel): tile blockIdx.x first, then the counter count[1]
        int c = nchunks, st = 0, tile = -1;
        unsigned r = 0u, id = blockIdx.x;
        for (;;) {
            if (r > 0) stage_acquire(st, 32 * (kF32Cons + 1));  // the consumers released the previous use (round r - 1)
            if (c == nchunks) {
                if (tile >= 0) {
                    if (lane == 0) id = atomicAdd(count + 1, 1u) + gridDim.x;
                    id = __shfl_sync(kFull, id, 0);
                }
                tile = id < ntiles ? (int)lpt_block(id, ntiles, kF32Tile) : -1;  // (longest first on an ordered set)
                c = 0;
            }
            unsigned char* sb = smem_raw + (size_t)st * Cfg::kStageBytes;
            uint64_t* fb = &full[st];
            if (lane == 0) *reinterpret_cast<int4*>(sb + Cfg::kHdrOff) = make_int4(tile, c, 0, 0);
            if (__any_sync(kFull, tile < 0)) {
                if (lane == 0) mbar_arrive(fb);
                break;
            }
            if (lane == 0) {
                const int r0 = c * W;  // layers r0 + 1 .. r0 + W: tour positions r0 .. r0 + W - 1
                int4 rq[W / 4];
#pragma unroll
                for (int g = 0; g < W / 4; ++g) rq[g] = __ldg(reinterpret_cast<const int4*>(trow + r0) + g);
                mbar_arrive_expect_tx(fb, (uint32_t)(Cfg::kRowsBytes + Cfg::kBandBytes));
#pragma unroll
                for (int g = 0; g < W / 4; ++g)
                    tma_gather4(sb + g * 4 * Cfg::kRowBytes, &dmap, tile * kF32Tile, rq[g].x, rq[g].y, rq[g].z, rq[g].w,
                                fb);
                bulk_g2s_plain(sb + Cfg::kBandOff, tbw + (int64_t)(r0 + 1) * W, Cfg::kBandBytes, fb);
            }
            __syncwarp();
            ++c;
            if (++st == NS) {
                st = 0;
                ++r;
            }
        }
    } else {
        __syncwarp();
        const int rem = n % W;
        float F[W];
        int32_t Y[W];
        int cs = 0;
        unsigned cr = 0u;
        for (;;) {
            unsigned char* sb = smem_raw + (size_t)cs * Cfg::kStageBytes;
            mbar_wait_warp(&full[cs], cr & 1u);
            const int4 th = *reinterpret_cast<const int4*>(sb + Cfg::kHdrOff);
            if (__all_sync(kFull, th.x < 0)) break;
            const int64_t s = (int64_t)th.x * kF32Tile + wid * 32 + lane;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                F[k] = 0.0f;
                Y[k] = -(1 << 30) - 1;  // no split point: never in a window (d < 0)
            }
            Y[0] = Q;  // split point 0: f = 0, P = 0
            int32_t P = 0;
            uint32_t qmax = 0u, ovf = 0u;
            for (int c = 0;;) {
                const uint16_t* rows = reinterpret_cast<const uint16_t*>(sb) + wid * 32 + lane;
                const float* band = reinterpret_cast<const float*>(sb + Cfg::kBandOff);
                const bool last = c == nchunks - 1;
                const int ilast = n - c * W;  // local index (1-based) of layer n in the last chunk
                // layer jj (local, 0-based; global i = c W + jj + 1) uses slot (1 + jj - k) mod W for age k
                auto cand = [&](const int jj, const int32_t Pn, const int k, uint32_t& d) -> uint32_t {
                    const int sl = (1 + jj - k + 2 * W) % W;
                    d = (uint32_t)(Y[sl] - Pn);
                    return f32_key(__fadd_rn(F[sl], band[jj * W + k - 1]), d);
                };
                // age W inside the window of a real layer i > W (i <= n): an older split point may be too
                auto overflow = [&](const int jj, const uint32_t d) {
                    if (c >= 1 && (!last || jj + 1 <= ilast)) ovf |= ~d;
                };
                // steps of LS layers (split_u16.cu): layer j + l's candidates of age >= max(2, l + 1) are
                // split points made before the step; they and the voted deeper groups of all LS layers run
                // first, the split points made inside the step are folded in last
                uint32_t qn = rows[0];
#pragma unroll
                for (int j = 0; j < W; j += LS) {
                    uint32_t qv[LS];
                    qv[0] = qn;
#pragma unroll
                    for (int l = 1; l < LS; ++l) qv[l] = rows[(j + l) * kF32Tile];
                    if (j + LS < W) qn = rows[(j + LS) * kF32Tile];
                    int32_t Pn[LS];
                    Pn[0] = P + (int32_t)qv[0];
#pragma unroll
                    for (int l = 1; l < LS; ++l) Pn[l] = Pn[l - 1] + (int32_t)qv[l];
#pragma unroll
                    for (int l = 0; l < LS; l += 2) qmax = max(qmax, max(qv[l], qv[l + 1]));
                    uint32_t a[LS];
#pragma unroll
                    for (int l = 0; l < LS; ++l) {
                        const int lo = l + 1 > 2 ? l + 1 : 2;
                        uint32_t kk[A0 - 1];
#pragma unroll
                        for (int k = 2; k <= A0; ++k) {
                            uint32_t d;
                            kk[k - 2] = k < lo ? 0xffffffffu : cand(j + l, Pn[l], k, d);
                        }
                        a[l] = umin_tree32_from<A0 - 1>(kk, lo - 2);
                    }
#pragma unroll
                    for (int gi = 0; gi < W; ++gi) {
                        const int ag = A0 + 1 + gi * UG;
                        if (ag > W) break;
                        uint32_t dg[LS], dall = 0xffffffffu;
#pragma unroll
                        for (int l = 0; l < LS; ++l) {
                            dg[l] = (uint32_t)(Y[(1 + j + l - ag + 2 * W) % W] - Pn[l]);
                            dall &= dg[l];
                        }
                        if (!__any_sync(kFull, (dall >> 31) == 0u)) break;  // some lane has age ag inside
#pragma unroll
                        for (int l = 0; l < LS; ++l) {
                            uint32_t e[UG + 1];
                            e[0] = a[l];
                            e[1] = f32_key(__fadd_rn(F[(1 + j + l - ag + 2 * W) % W], band[(j + l) * W + ag - 1]), dg[l]);
                            if (ag == W) overflow(j + l, dg[l]);
#pragma unroll
                            for (int u = 1; u < UG; ++u) {
                                if (ag + u <= W) {
                                    uint32_t dd;
                                    e[u + 1] = cand(j + l, Pn[l], ag + u, dd);
                                    if (ag + u == W) overflow(j + l, dd);
                                } else {
                                    e[u + 1] = 0xffffffffu;
                                }
                            }
                            a[l] = umin_tree32<UG + 1>(e);
                        }
                    }
                    // the split points of the step: fn[m] = f(i_j + m), i_j = c W + j + 1 (layer j's)
                    float fn[LS];
                    const float fprev = F[(j + 2 * W) % W];  // f(i_j - 1): age 1 of layer j
#pragma unroll
                    for (int l = 0; l < LS; ++l) {
                        uint32_t m = a[l];
                        // in-step ages 2 .. l: split point i_j + l - k = fn[l - k], Y = Pn[l - k] + Q
                        if (l == 2) {
                            m = min(m, f32_key(__fadd_rn(fn[0], band[(j + l) * W + 1]), (uint32_t)(Pn[0] + Q - Pn[l])));
                        } else if (l == 3) {
                            m = __vimin3_u32(m, f32_key(__fadd_rn(fn[1], band[(j + l) * W + 1]), (uint32_t)(Pn[1] + Q - Pn[l])),
                                             f32_key(__fadd_rn(fn[0], band[(j + l) * W + 2]), (uint32_t)(Pn[0] + Q - Pn[l])));
                        }
                        // age 1 (split point i_j + l - 1): always inside when q <= Q (q > Q: qmax)
                        const float f1 = l == 0 ? fprev : fn[l - 1];
                        fn[l] = __uint_as_float(min(m, __float_as_uint(__fadd_rn(f1, band[(j + l) * W]))));
                    }
#pragma unroll
                    for (int l = 0; l < LS; ++l) {  // (after every read of these slots' previous contents)
                        F[(1 + j + l) % W] = fn[l];
                        Y[(1 + j + l) % W] = Pn[l] + Q;
                    }
                    P = Pn[LS - 1];
                }
                stage_release(cs, 32 * (kF32Cons + 1));
                if (++cs == NS) {
                    cs = 0;
                    ++cr;
                }
                if (++c >= nchunks) break;
                sb = smem_raw + (size_t)cs * Cfg::kStageBytes;
                mbar_wait_warp(&full[cs], cr & 1u);
            }
            // f(n) sits in slot n mod W (the padded layers after it wrote fewer than W slots)
            uint32_t fin = 0u;  // (a select chain, not an indexed read: F stays in registers)
#pragma unroll
            for (int k = 0; k < W; ++k) fin = k == rem ? __float_as_uint(F[k]) : fin;
            if (s < S) {
                // the window of some real layer reached age W: an older split point may be inside
                if (qmax > (uint32_t)Q) cost[s] = INFINITY;  // Eq. (2)'s set is empty at some layer (R4)
                else if (ovf & 0x80000000u) list[atomicAdd(count, 1u)] = s;
                else cost[s] = __uint_as_float(fin);
            }
        }
    }
}

// SAA moments of fp32 costs in fp64: acc = {m, sum c, sum (c - center)^2, infeasible} over the
// finite costs (block tree sums, one fp64 atomic per block and field).
__global__ void __launch_bounds__(256) saa_f32_moments_kernel(const float* __restrict__ cost, int64_t S, double center,
                                                              double* __restrict__ acc) {
    __shared__ double sh[4][8];
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
        const float c = cost[s];
        if (isinf(c)) {
            v[3] += 1.0;
            continue;
        }
        const double d = (double)c - center;
        v[0] += 1.0;
        v[1] += (double)c;
        v[2] += d * d;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[f] += __shfl_xor_sync(kFull, v[f], o);
        if (lane == 0) sh[f][wid] = v[f];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[threadIdx.x][w];
        atomicAdd(&acc[threadIdx.x], t);
    }
}

static size_t f32_table_bytes(int32_t n) { return align_up(sizeof(F32Pos) * (size_t)(n + 1 + 8), 256); }
static size_t f32_list_bytes(int64_t S) { return align_up(sizeof(int64_t) * (size_t)S, 256) + 256; }
static int f32_tw_chunks(int32_t n) { return (n + kF32TW - 1) / kF32TW; }
static size_t f32_trow_bytes(int32_t n) { return align_up(sizeof(int32_t) * (size_t)(f32_tw_chunks(n) * kF32TW + 4), 256); }
static size_t f32_bandw_bytes(int32_t n) { return align_up(sizeof(float) * (size_t)(n + 1 + kF32TW) * kF32TW, 256); }

}  // namespace spdp

using namespace spdp;

extern "C" size_t spdp_f32_workspace_bytes(int32_t n, int64_t S) {
    if (n < 1 || S < 1) return 0;
    return f32_table_bytes(n) + f32_list_bytes(S) +
           align_up(sizeof(float) * (size_t)(n + 1) * (size_t)S, 256) + f32_trow_bytes(n) + f32_bandw_bytes(n);
}

extern "C" spdp_status spdp_split_eval_f32(const int32_t* tour, const double* dist, int32_t n, const uint16_t* demand,
                                           int64_t ld, int64_t S, int32_t Q, float* cost, void* ws, size_t ws_bytes,
                                           spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval_f32");
    const char* fn = "spdp_split_eval_f32";
    if (n < 1) return fail(SPDP_E_USAGE, "%s: n=%d < 1", fn, n);
    if (n > SPDP_MAX_N) return fail(SPDP_E_RESOURCE, "%s: n=%d > SPDP_MAX_N=%d", fn, n, SPDP_MAX_N);
    if (S < 1) return fail(SPDP_E_USAGE, "%s: S=%lld < 1", fn, (long long)S);
    if (Q < 1) return fail(SPDP_E_USAGE, "%s: Q=%d < 1 (SPEC:34)", fn, Q);
    if (ld < S || (ld % 8) != 0) return fail(SPDP_E_USAGE, "%s: ld=%lld must be >= S and a multiple of 8", fn, (long long)ld);
    if (!tour || !dist || !demand || !cost || !ws) return fail(SPDP_E_USAGE, "%s: NULL required pointer", fn);
    if (ws_bytes < spdp_f32_workspace_bytes(n, S)) return fail(SPDP_E_USAGE, "%s: workspace too small", fn);
    if ((uint64_t)n * (uint64_t)ld >= (1ull << 32)) return fail(SPDP_E_RESOURCE, "%s: n ld must stay below 2^32", fn);
    cudaStream_t st = (cudaStream_t)stream;
    char* w = static_cast<char*>(ws);
    F32Pos* tab = reinterpret_cast<F32Pos*>(w);
    int64_t* list = reinterpret_cast<int64_t*>(w + f32_table_bytes(n));
    unsigned* count = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(list) + align_up(sizeof(int64_t) * (size_t)S, 256));
    float* fsc = reinterpret_cast<float*>(w + f32_table_bytes(n) + f32_list_bytes(S));
    const int Qe = (int)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    // the TMA sweep keeps Y = P + Q and P(i) - Y in int32: every load it forms (including the padded
    // layers' zero demands) is at most (n + W) min(Q, 65535) (larger demands make the scenario
    // infeasible, and its value is not used), so Y < 2^30 + Q suffices
    const int64_t qcap = Qe < 65535 ? Qe : 65535;
    const bool tma = ((int64_t)n + kF32TW) * qcap + Qe < (1LL << 30);
    int32_t* trow = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(fsc) + align_up(sizeof(float) * (size_t)(n + 1) * (size_t)S, 256));
    float* tbw = reinterpret_cast<float*>(reinterpret_cast<char*>(trow) + f32_trow_bytes(n));
    f32_prep_kernel<<<1, 256, 0, st>>>(tour, n, dist, ld, tab, tma ? trow : nullptr, f32_tw_chunks(n) * kF32TW + 4,
                                       count);
    spdp_status rc = last_launch("f32_prep_kernel");
    if (rc) return rc;
    if (tma) {
        const int64_t nbw = (int64_t)(n + 1 + kF32TW) * kF32TW;
        f32_bandw_kernel<<<(unsigned)ceil_div(nbw, 256), 256, 0, st>>>(tab, n, kF32TW, tbw);
        if ((rc = last_launch("f32_bandw_kernel"))) return rc;
        auto go = [&](auto kern, size_t smem) -> spdp_status {
            int bps = 1;
            spdp_status r2;
            if ((r2 = kernel_setup((const void*)kern, (int)smem, 100, kF32Threads, smem, &bps, "split_f32_tma setup")))
                return r2;
            CUtensorMap map;
            if ((r2 = make_demand_map(&map, demand, ld, S, n, kF32Tile))) return r2;
            const int64_t ntiles = ceil_div(S, kF32Tile);
            int64_t grid = (int64_t)bps * device_sms();
            if (grid > ntiles) grid = ntiles;
            prof_begin(st);
            kern<<<(unsigned)grid, kF32Threads, smem, st>>>(map, trow, tbw, n, S, Qe, cost, list, count);
            return last_launch("split_f32_tma_kernel");
        };
        rc = go(split_f32_tma_kernel<kF32TW, kF32TA0, 2, 3, 4>, F32TCfg<kF32TW, 3>::kSmem);
        if (rc) return rc;
        set_last_kernel("split_f32_tma_kernel<%d,%d,%d,4>", kF32TW, kF32TA0, 2);
    } else {  // (loads near 2^30: every scenario through the general kernel)
        prof_begin(st);
        list = nullptr;
        set_last_kernel("split_f32_kernel");
    }
    const bool tsm = n <= kF32SmemMaxN;
    if ((rc = kernel_setup((const void*)split_f32_kernel, (int)(sizeof(F32Pos) * (kF32SmemMaxN + 1)), -1, 0, 0, nullptr,
                           "split_f32_kernel setup")))
        return rc;
    int64_t fgrid = ceil_div(S, 256);
    if (list && fgrid > 2 * (int64_t)device_sms()) fgrid = 2 * (int64_t)device_sms();  // (strides over the list)
    split_f32_kernel<<<(unsigned)fgrid, 256, tsm ? sizeof(F32Pos) * (size_t)(n + 1) : 0, st>>>(
        tab, n, demand, S, Qe, fsc, cost, tsm ? 1 : 0, list, count);
    prof_end(st);
    return last_launch("split_f32_kernel");
}

extern "C" spdp_status spdp_split_eval_batch_f32(const int32_t* tours, int32_t T, const double* dist, int32_t n,
                                                 const uint16_t* demand, int64_t ld, int64_t S, int32_t Q, float* cost,
                                                 void* ws, size_t ws_bytes, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval_batch_f32");
    if (T < 1) return fail(SPDP_E_USAGE, "spdp_split_eval_batch_f32: T=%d < 1", T);
    if (!tours || !cost) return fail(SPDP_E_USAGE, "spdp_split_eval_batch_f32: NULL required pointer");
    // the tours one after the other on the stream (the workspace of one tour is reused)
    for (int32_t t = 0; t < T; ++t) {
        spdp_status rc = spdp_split_eval_f32(tours + (int64_t)t * n, dist, n, demand, ld, S, Q, cost + (int64_t)t * S, ws,
                                             ws_bytes, stream);
        if (rc) return rc;
    }
    return SPDP_OK;
}

extern "C" spdp_status spdp_saa_f32_moments(const float* cost, int64_t S, double center, double* moments,
                                             spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_saa_f32_moments");
    if (!cost || !moments || S < 1) return fail(SPDP_E_USAGE, "spdp_saa_f32_moments: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    spdp_status rc = cuda_check(cudaMemsetAsync(moments, 0, 4 * sizeof(double), st), "cudaMemsetAsync(moments)");
    if (rc) return rc;
    int64_t blocks = ceil_div(S, 256 * 8);
    if (blocks > (int64_t)device_sms() * 8) blocks = (int64_t)device_sms() * 8;
    saa_f32_moments_kernel<<<(unsigned)blocks, 256, 0, st>>>(cost, S, center, moments);
    return last_launch("saa_f32_moments_kernel");
}

// fp32-mode SAA finalize (host): from the summed pass-1 moments {m, sum c, -, infeasible} the
// count and mean; with the pass-2 moments (centred on that mean) also the unbiased variance,
// standard error and 95 % interval (the sample average of the second-stage costs).
extern "C" spdp_status spdp_saa_finalize_f32(const double* m1, const double* m2, spdp_saa_estimate* out) {
    NvtxScope nvtx_("spdp_saa_finalize_f32");
    const char* fn = "spdp_saa_finalize_f32";
    if (!m1 || !out) return fail(SPDP_E_USAGE, "%s: NULL pointer", fn);
    if (!(m1[0] >= 0.0) || !(m1[3] >= 0.0)) return fail(SPDP_E_USAGE, "%s: negative counts", fn);
    const int64_t m = (int64_t)llround(m1[0]);
    out->m = m;
    out->infeasible = (int64_t)llround(m1[3]);
    out->mean = out->var = out->std_err = out->ci95_lo = out->ci95_hi = NAN;
    if (m == 0) return fail(SPDP_E_DATA, "%s: all scenarios infeasible (SPEC:287)", fn);
    out->mean = m1[1] / (double)m;
    if (!m2) return SPDP_OK;
    out->var = m >= 2 ? m2[2] / (double)(m - 1) : 0.0;
    out->std_err = sqrt(out->var / (double)m);
    out->ci95_lo = out->mean - 1.96 * out->std_err;
    out->ci95_hi = out->mean + 1.96 * out->std_err;
    return SPDP_OK;
}

extern "C" spdp_status spdp_saa_estimate_f32(const float* cost, int64_t S, spdp_saa_estimate* out, void* ws,
                                             size_t ws_bytes, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_saa_estimate_f32");
    const char* fn = "spdp_saa_estimate_f32";
    if (!cost || !out || !ws || S < 1) return fail(SPDP_E_USAGE, "%s: bad arguments", fn);
    if (ws_bytes < 64) return fail(SPDP_E_USAGE, "%s: workspace < 64 bytes", fn);
    cudaStream_t st = (cudaStream_t)stream;
    double* acc = static_cast<double*>(ws);
    double h1[4], h2[4];
    // pass 1: count and sum -> mean; pass 2: squared deviations about that mean (two-pass variance)
    spdp_status rc = spdp_saa_f32_moments(cost, S, 0.0, acc, stream);
    if (rc) return rc;
    if ((rc = cuda_check(cudaMemcpyAsync(h1, acc, sizeof(h1), cudaMemcpyDeviceToHost, st), "memcpy(moments)"))) return rc;
    if ((rc = cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
    if ((rc = spdp_saa_finalize_f32(h1, nullptr, out))) return rc;
    if ((rc = spdp_saa_f32_moments(cost, S, out->mean, acc, stream))) return rc;
    if ((rc = cuda_check(cudaMemcpyAsync(h2, acc, sizeof(h2), cudaMemcpyDeviceToHost, st), "memcpy(moments)"))) return rc;
    if ((rc = cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
    return spdp_saa_finalize_f32(h1, h2, out);
}
