// limits.cu -- f4: the split with a route-duration limit and a
// fleet limit (DESIGN R24; "route length/duration constraints, if
// applicable"; "three vehicles available"):
//   a route (p, i] is admissible iff  sum_{k=p+1}^{i} q <= Q  (Eq. (2)) and
//   t(p, i) = A[p] + B[i] <= Lmax  (duration = route cost, scenario-invariant);
//   F_0(0) = 0,  F_k(i) = min_{admissible (p, i]} F_{k-1}(p) + t(p, i),
//   cost = min_{k <= K} F_k(n)   (K <= 0: no fleet limit -> one pass of Eq. (3)).
// The fleet limit adds the vehicle-count layer dimension to the layered DAG, kept
// to the band of k that the capacity bounds allow (ring kernel below).  Fleet launches: a classify
// pass (infeasible scenarios finished; the rest listed by the band width their slack K - kT
// needs), one ring pass per band width 2 / 4 / 8 / 16 over its list, a warp-per-scenario kernel for
// slack 16..31 and windows longer than the ring, the general kernel for the rest (C2, K = 27:
// 3.9 -> 1.37 ms).  The masks
// mask(i) of Eq. (2) do not depend on k: they are computed once per scenario (two
// pointers) and reused for every k.
#include <climits>

#include "common.cuh"
#include "split_ws.cuh"

namespace spdp {

constexpr int kLimTableSmemMaxN = 2047;  // position table staged in shared memory up to 32 KB
constexpr int kLimBig = 1 << 30;  // no admissible split (above every finite value, R17 range bound)
constexpr int kLimThreads = 64;
// persistent grid of the general kernel (its per-scenario arrays in the workspace): enough warps
// to hide the latency of its serial loops, within a bounded workspace
__host__ __device__ inline int lim_blocks_per_sm(int n) { return n <= 256 ? 16 : (n <= 2048 ? 8 : 2); }

// The general kernel (any window, any number of routes): one scenario per thread,
// grid-stride over the scenarios (or over the `list` of scenarios the ring kernel
// deferred, `count` of them).  Per-thread arrays of n+1 ints (mask | kP << 16, F_a,
// F_b; element p of thread r at base[p * stride + r], coalesced) live in the
// workspace (shared memory would leave 1-2 CTAs per SM).  The tour's position table
// {row, A, B, row offset} is staged in shared memory.
__global__ void __launch_bounds__(kLimThreads) split_limits_kernel(const int4* __restrict__ e, int n,
                                                                  const uint16_t* __restrict__ demand, int64_t S, int Q,
                                                                  int Lmax, int K, int32_t* __restrict__ cost,
                                                                  spdp_saa_partial* __restrict__ partial, int* gscratch,
                                                                  const int64_t* __restrict__ list,
                                                                  const unsigned* __restrict__ count) {
    extern __shared__ int4 sm4[];
    __shared__ Part red[kLimThreads / 32];
    const int4* tb = e;  // staged in shared memory up to kLimTableSmemMaxN positions, else read through L1
    if (n <= kLimTableSmemMaxN) {
        for (int i = threadIdx.x; i <= n; i += blockDim.x) sm4[i] = e[i];
        __syncthreads();
        tb = sm4;
    }
    int* arr = gscratch;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int* Mk = arr + r;
    int* Fa = arr + (int64_t)(n + 1) * stride + r;
    int* Fb = arr + 2 * (int64_t)(n + 1) * stride + r;
    const bool fleet = K > 0 && K < n;
    Part acc{0, 0, 0, 0, 0};
    const int64_t nwork = list ? (int64_t)*count : S;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwork; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = list ? list[w] : w;
        const uint16_t* dcol = demand + s;
        // tour-order prefix loads (in Fb) and the Eq. (2) masks
        int P = 0;
        bool bad = false;
        Fb[0] = 0;
        for (int i = 1; i <= n; ++i) {
            const int q = dcol[(uint32_t)tb[i].w];
            bad |= q > Q;
            P += q;
            Fb[(int64_t)i * stride] = P;
        }
        int result = SPDP_INFEASIBLE;
        if (!bad) {
            // masks (low 16 bits) and kP(i), the greedy route count of the prefix (high 16 bits)
            int m = 0, Pm = 0, kp = 0, load = Q + 1;
            for (int i = 1; i <= n; ++i) {
                const int Pi = Fb[(int64_t)i * stride];
                const int q = Pi - Fb[(int64_t)(i - 1) * stride];
                load += q;
                if (load > Q) {
                    ++kp;
                    load = q;
                }
                while (Pi - Pm > Q) Pm = Fb[(int64_t)(++m) * stride];
                Mk[(int64_t)i * stride] = m | (kp << 16);
            }
            const int kT = kp;
            // one pass of the layered sweep: cur[i] = min_{admissible p} prev[p] + A[p] + B[i]
            auto pass = [&](const int* prev, int* cur) -> bool {
                bool any = false;
                for (int i = 1; i <= n; ++i) {
                    const int Bi = tb[i].z;
                    const int thr = Lmax - Bi;  // duration: A[p] <= Lmax - B[i]
                    const int lo = Mk[(int64_t)i * stride] & 0xffff;
                    int best = kLimBig;
                    for (int p = i - 1; p >= lo; --p) {
                        const int Ap = tb[p].y;
                        const int fp = prev[(int64_t)p * stride];
                        if (Ap <= thr && fp < kLimBig) best = min(best, fp + Ap);
                    }
                    const int v = best >= kLimBig ? kLimBig : best + Bi;
                    cur[(int64_t)i * stride] = v;
                    any |= v < kLimBig;
                }
                return any;
            };
            int res;
            if (!fleet) {  // Eq. (3) in place: F(i) reads F(p < i) of the same pass
                Fa[0] = 0;
                pass(Fa, Fa);
                res = Fa[(int64_t)n * stride];
            } else if (K < kT) {  // more routes needed than available (capacity bound)
                res = kLimBig;
            } else {
                // pass k only visits the band of layers i with kP(i) <= k <= kP(i) + K - kT (the
                // ring kernel's bound, see below); kP is nondecreasing, so the band is a range
                // [lo_k, hi_k] moving right with k, and cells left behind are reset to infinity
                const int slack = K - kT;
                for (int i = 0; i <= n; ++i) {
                    Fa[(int64_t)i * stride] = i == 0 ? 0 : kLimBig;  // F_0
                    Fb[(int64_t)i * stride] = kLimBig;
                }
                int* prev = Fa;
                int* cur = Fb;
                res = kLimBig;
                int lo = 1, hi = 0, lo2 = 1, lo1 = 1;  // lo2 / lo1: the bands' starts two / one passes ago
                auto kp_at = [&](int i) -> int { return Mk[(int64_t)i * stride] >> 16; };
                for (int k = 1; k <= K; ++k) {
                    while (lo <= n && kp_at(lo) < k - slack) ++lo;
                    while (hi + 1 <= n && kp_at(hi + 1) <= k) ++hi;
                    cur[0] = kLimBig;  // F_k(0), k >= 1
                    for (int i = lo2; i < lo && i <= n; ++i) cur[(int64_t)i * stride] = kLimBig;
                    for (int i = lo; i <= hi; ++i) {
                        const int Bi = tb[i].z;
                        const int thr = Lmax - Bi;
                        const int mlo = Mk[(int64_t)i * stride] & 0xffff;
                        int best = kLimBig;
                        for (int p = i - 1; p >= mlo; --p) {
                            const int Ap = tb[p].y;
                            const int fp = prev[(int64_t)p * stride];
                            if (Ap <= thr && fp < kLimBig) best = min(best, fp + Ap);
                        }
                        cur[(int64_t)i * stride] = best >= kLimBig ? kLimBig : best + Bi;
                    }
                    if (hi == n) res = min(res, cur[(int64_t)n * stride]);
                    int* tmp = prev;
                    prev = cur;
                    cur = tmp;
                    lo2 = lo1;
                    lo1 = lo;
                }
            }
            result = res >= kLimBig ? SPDP_INFEASIBLE : res;
        }
        if (cost) cost[s] = result;
        part_add_cost(acc, result, result != SPDP_INFEASIBLE);
    }
    if (partial) {
        const Part t = block_sum(acc, red);
        if (threadIdx.x == 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_feas), (unsigned long long)t.n_feas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_infeas), (unsigned long long)t.n_infeas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sum), (unsigned long long)t.sum);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_lo), (unsigned long long)t.sq_lo);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_hi), (unsigned long long)t.sq_hi);
        }
    }
}

// The ring kernel (the common case): one scenario per thread; the last kRing positions
// of the DP live in a per-thread shared-memory ring (slot p mod kRing, [slot][tid]
// layout: conflict-free).  Eq. (2) mask by two pointers over the ring's prefix loads.
// Fleet limit (BW > 1): the vehicle-count dimension is kept to a band.  With kP(i) the
// greedy (minimum, R5) number of capacity-feasible routes for the prefix 1..i and
// kT = kP(n), F_k(i) is infinite for k < kP(i), and a state with k > kP(i) + K - kT
// cannot complete within K routes (the suffix needs at least kT - kP(i)), so layer i
// keeps k in [kP(i), kP(i) + K - kT] only: K - kT + 1 <= BW values per position (the
// duration limit only removes routes, so these capacity bounds stay valid).  A
// scenario whose window outgrows the ring or whose band exceeds BW is deferred to the
// general kernel (list).  (Without a fleet limit the launcher uses the register-ring kernel
// below instead of BW = 1 here: measured 0.59 vs 1.03 ms at C2.)  F of a (slot, thread) is BW
// contiguous ints, so a BW % 4 == 0 band loads with 16-byte accesses.
template <int BW, int NT, int kRing>
__global__ void __launch_bounds__(NT) split_limits_ring_kernel(const int4* __restrict__ e, int n,
                                                               const uint16_t* __restrict__ demand, int64_t S, int Q,
                                                               int Lmax, int K, int32_t* __restrict__ cost,
                                                               spdp_saa_partial* __restrict__ partial,
                                                               int2* __restrict__ list, unsigned* __restrict__ count,
                                                               int table_in_smem, const int2* __restrict__ in_list,
                                                               const unsigned* __restrict__ in_count) {
    constexpr bool FLEET = BW > 1;
    extern __shared__ int4 sm4[];
    __shared__ Part red[NT / 32];
    const int tid = threadIdx.x;
    int* ringP = reinterpret_cast<int*>(sm4);                  // [kRing][NT]
    int* ringK = ringP + kRing * NT;                           // [kRing][NT]: kP(p) (fleet)
    int* ringF = ringK + (FLEET ? kRing * NT : 0);             // [kRing][BW][NT]
    const int4* tb = e;
    if (table_in_smem) {
        int4* st = reinterpret_cast<int4*>(ringF + kRing * BW * NT);
        for (int i = tid; i <= n; i += NT) st[i] = e[i];
        __syncthreads();
        tb = st;
    }
    auto P_at = [&](int p) -> int& { return ringP[(p & (kRing - 1)) * NT + tid]; };
    auto K_at = [&](int p) -> int& { return ringK[(p & (kRing - 1)) * NT + tid]; };
    // F of one (slot, thread): BW contiguous ints ([kRing][NT][BW]: one 16-byte load when BW = 4)
    auto F_at = [&](int p, int b) -> int& { return ringF[((p & (kRing - 1)) * NT + tid) * BW + b]; };
    Part acc{0, 0, 0, 0, 0};
    // the scenario: the thread's own (natural order) or the w-th entry of the classify pass's list for
    // this band width (its slack already known and in [0, BW): no pre-pass)
    const int64_t w = (int64_t)blockIdx.x * NT + tid;
    const bool listed = in_list != nullptr;
    const int64_t s = listed ? (w < (int64_t)*in_count ? (int64_t)in_list[w].x : S) : w;
    if (s < S) {
        const uint16_t* dcol = demand + s;
        int result = SPDP_INFEASIBLE;
        bool defer = false;
        // capacity pre-pass: any demand above Q (R4) and kT = greedy route count of the whole tour
        bool bad = false;
        int kT = listed ? K - in_list[w].y : 0;
        if (!listed) {
            int load = Q + 1;
            for (int i = 1; i <= n; ++i) {
                const int q = dcol[(uint32_t)tb[i].w];
                bad |= q > Q;
                load += q;
                if (load > Q) {
                    ++kT;
                    load = q;
                }
            }
        }
        const int slack = FLEET ? K - kT : 0;
        if (!bad && slack >= 0) {
            if (slack >= BW) {
                defer = true;
            } else {
                P_at(0) = 0;
                if (FLEET) {
                    K_at(0) = 0;
#pragma unroll
                    for (int b = 0; b < BW; ++b) F_at(0, b) = b == 0 ? 0 : kLimBig;  // F_0(0) = 0
                } else {
                    F_at(0, 0) = 0;
                }
                int P = 0, m = 0, kp = 0, load = Q + 1;
                for (int i = 1; i <= n && !defer; ++i) {
                    const int4 ei = tb[i];
                    const int q = dcol[(uint32_t)ei.w];
                    P += q;
                    load += q;
                    if (load > Q) {  // greedy prefix route count kP(i)
                        ++kp;
                        load = q;
                    }
                    if (m < i - kRing) {  // the ring holds positions i-32..i-1 only: defer (conservative)
                        defer = true;
                        break;
                    }
                    while (P - P_at(m) > Q) ++m;  // mask(i), m <= i - 1 since q <= Q
                    const int thr = Lmax - ei.z;  // duration: A[p] <= Lmax - B[i]
                    int best[BW];
#pragma unroll
                    for (int b = 0; b < BW; ++b) best[b] = kLimBig;
                    for (int p = i - 1; p >= m; --p) {
                        const int Ap = tb[p].y;
                        if (Ap > thr) continue;
                        if constexpr (BW % 4 == 0) {
                            // a feasible route (p, i] holds at most one greedy route start, so
                            // d = kP(i) - kP(p) is 0 or 1 for every in-window p: F_{k-1}(p), k = kP(i) + b,
                            // is band entry b - 1 + d -- a select between two fixed registers
                            const int d = kp - K_at(p);
                            int v[BW];
#pragma unroll
                            for (int b4 = 0; b4 < BW; b4 += 4) {
                                const int4 f4 = *reinterpret_cast<const int4*>(&F_at(p, b4));
                                v[b4] = f4.x;
                                v[b4 + 1] = f4.y;
                                v[b4 + 2] = f4.z;
                                v[b4 + 3] = f4.w;
                            }
#pragma unroll
                            for (int b = 0; b < BW; ++b) {
                                const int c = d ? v[b] : (b ? v[b - 1] : kLimBig);
                                if (c < kLimBig) best[b] = min(best[b], c + Ap);
                            }
                        } else if constexpr (BW == 2) {  // (the same select, one 8-byte load)
                            const int d = kp - K_at(p);
                            const int2 f2 = *reinterpret_cast<const int2*>(&F_at(p, 0));
                            const int v[2] = {f2.x, f2.y};
#pragma unroll
                            for (int b = 0; b < BW; ++b) {
                                const int c = d ? v[b] : (b ? v[b - 1] : kLimBig);
                                if (c < kLimBig) best[b] = min(best[b], c + Ap);
                            }
                        } else if (FLEET) {
                            const int off = kp - 1 - K_at(p);  // F_{k-1}(p), k = kp + b: band index off + b
#pragma unroll
                            for (int b = 0; b < BW; ++b) {
                                const int bb = off + b;
                                if (bb >= 0 && bb < BW) {
                                    const int fp = F_at(p, bb);
                                    if (fp < kLimBig) best[b] = min(best[b], fp + Ap);
                                }
                            }
                        } else {
                            const int fp = F_at(p, 0);
                            if (fp < kLimBig) best[0] = min(best[0], fp + Ap);
                        }
                    }
                    // layer i overwrites slot i mod 32 (position i - 32 is out of every later window)
                    P_at(i) = P;
                    if (FLEET) K_at(i) = kp;
#pragma unroll
                    for (int b = 0; b < BW; ++b) {
                        int v = best[b] >= kLimBig ? kLimBig : best[b] + ei.z;
                        if (FLEET && (b > slack || kp + b > K)) v = kLimBig;  // outside the band
                        F_at(i, b) = v;
                    }
                }
                if (!defer) {
                    int res = kLimBig;
#pragma unroll
                    for (int b = 0; b < BW; ++b) res = min(res, F_at(n, b));
                    result = res >= kLimBig ? SPDP_INFEASIBLE : res;
                }
            }
        }
        if (defer) {  // (the window outgrew the ring: the warp-per-scenario kernel, any window)
            list[atomicAdd(count, 1u)] = make_int2((int)s, FLEET ? K - kT : 0);
        } else {
            if (cost) cost[s] = result;
            part_add_cost(acc, result, result != SPDP_INFEASIBLE);
        }
    }
    if (partial) {
        const Part t = block_sum(acc, red);
        if (tid == 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_feas), (unsigned long long)t.n_feas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_infeas), (unsigned long long)t.n_infeas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sum), (unsigned long long)t.sum);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_lo), (unsigned long long)t.sq_lo);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_hi), (unsigned long long)t.sq_hi);
        }
    }
}

// Fleet limit, pass 0: one thread per scenario (coalesced column reads): any demand
// above Q (R4) and kT = the greedy (minimum) route count of the whole tour.  slack = K - kT < 0 (or
// a demand above Q): infeasible, finished here.  Otherwise the scenario goes to the list of the
// band width its slack needs (BW = 2, 4, 8, 16: slack < BW) -- or, wider, to the general kernel's
// list -- so that each ring pass runs warps whose lanes all need (about) the same band and no lane
// idles on an infeasible scenario (at C2, K = kmin + 2: 72 % infeasible, slack spread over 0..15).
constexpr int kLimBands = 4;  // band widths 2, 4, 8, 16
constexpr int kLimWarpBW = 32;  // the warp kernel's band: one lane per vehicle count
__global__ void __launch_bounds__(256) limits_classify_kernel(const int4* __restrict__ tb, int n,
                                                              const uint16_t* __restrict__ demand, int64_t S, int Q, int K,
                                                              int32_t* __restrict__ cost,
                                                              spdp_saa_partial* __restrict__ partial,
                                                              int2* __restrict__ blists, int64_t cap,
                                                              unsigned* __restrict__ bcounts,
                                                              int64_t* __restrict__ list, unsigned* __restrict__ count,
                                                              int warp_ok) {
    // blists: [kLimBands + 1][cap] {scenario, slack} (the last: the warp kernel's), bcounts likewise
    __shared__ Part red[8];
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    Part acc{0, 0, 0, 0, 0};
    int cls = -1;  // -1: none (finished or no scenario), 0..3: band list, 4: the warp kernel, 5: the general kernel
    int slack = 0;
    if (s < S) {
        const uint16_t* dcol = demand + s;
        bool bad = false;
        int kT = 0, load = Q + 1;
        for (int i = 1; i <= n; ++i) {
            const int q = dcol[(uint32_t)__ldg(&tb[i].w)];
            bad |= q > Q;
            load += q;
            if (load > Q) {
                ++kT;
                load = q;
            }
        }
        slack = K - kT;
        if (bad || slack < 0) {
            if (cost) cost[s] = SPDP_INFEASIBLE;
            part_add_cost(acc, SPDP_INFEASIBLE, false);
        } else {
            cls = slack < 2 ? 0 : slack < 4 ? 1 : slack < 8 ? 2 : slack < 16 ? 3 : (warp_ok && slack < kLimWarpBW) ? 4 : 5;
        }
    }
    // warp-aggregated appends: one atomic per (warp, list)
#pragma unroll
    for (int c = 0; c <= kLimBands + 1; ++c) {
        const unsigned m = __ballot_sync(kFull, cls == c);
        if (m == 0u) continue;
        unsigned base = 0u;
        const int leader = __ffs(m) - 1;
        if (lane == leader) base = atomicAdd(c <= kLimBands ? &bcounts[c] : count, (unsigned)__popc(m));
        base = __shfl_sync(kFull, base, leader);
        if (cls == c) {
            const unsigned idx = base + (unsigned)__popc(m & ((1u << lane) - 1u));
            if (c <= kLimBands) blists[(int64_t)c * cap + idx] = make_int2((int)s, slack);
            else list[idx] = s;
        }
    }
    if (partial) {
        const Part t = block_sum(acc, red);
        if (threadIdx.x == 0 && t.n_infeas) atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_infeas),
                                                      (unsigned long long)t.n_infeas);
    }
}


// Fleet limit, the rare cases (slack 16..31, or a window longer than the ring): ONE WARP PER
// SCENARIO, lane b = vehicle-count offset b (k = kP(i) + b), any window.  Per warp in shared memory
// the prefix loads P[0..n], kP[0..n] and the band F[0..n][32]; the layer loop and the candidate
// loop are warp-uniform (the mask two-pointer and the duration test do not depend on k), each lane
// forms F_{k-1}(p) + t(p, i) for its own k, band entry b - 1 + (kP(i) - kP(p)) (R24, ring kernel).
__global__ void __launch_bounds__(256) split_limits_warp_kernel(const int4* __restrict__ tb, int n,
                                                                const uint16_t* __restrict__ demand, int Q, int Lmax,
                                                                int K, int32_t* __restrict__ cost,
                                                                spdp_saa_partial* __restrict__ partial,
                                                                const int2* __restrict__ wlist,
                                                                const unsigned* __restrict__ wcount) {
    extern __shared__ int smw[];
    __shared__ Part red[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int* Pw = smw + (size_t)wid * (n + 1) * (kLimWarpBW + 2);
    int* Kw = Pw + (n + 1);
    int* Fw = Kw + (n + 1);
    Part acc{0, 0, 0, 0, 0};
    const unsigned total = *wcount;
    for (unsigned w = blockIdx.x * nw + wid; w < total; w += gridDim.x * nw) {
        const int2 ent = wlist[w];
        const int64_t s = ent.x;
        const uint16_t* dcol = demand + s;
        // tour-order prefix loads, 32 positions at a time (warp scan)
        int base = 0;
        bool bad = false;
        if (lane == 0) Pw[0] = 0;
        for (int i0 = 1; i0 <= n; i0 += 32) {
            const int i = i0 + lane;
            int q = i <= n ? (int)dcol[(uint32_t)__ldg(&tb[i].w)] : 0;
            bad |= q > Q;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(kFull, q, o);
                if (lane >= o) q += v;
            }
            if (i <= n) Pw[i] = base + q;
            base += __shfl_sync(kFull, q, 31);
        }
        __syncwarp();
        if (lane == 0) {  // kP(i): the greedy (minimum) route count of the prefix 1..i
            int kp = 0, load = Q + 1;
            Kw[0] = 0;
            for (int i = 1; i <= n; ++i) {
                const int q = Pw[i] - Pw[i - 1];
                load += q;
                if (load > Q) {
                    ++kp;
                    load = q;
                }
                Kw[i] = kp;
            }
        }
        __syncwarp();
        const int slack = K - Kw[n];
        int result = SPDP_INFEASIBLE;
        if (!__any_sync(kFull, bad) && slack >= 0) {
            Fw[lane] = lane == 0 ? 0 : kLimBig;  // F_0(0) = 0
            int m = 0;
            for (int i = 1; i <= n; ++i) {
                const int Pi = Pw[i];
                while (Pi - Pw[m] > Q) ++m;  // mask(i)
                const int kpi = Kw[i];
                const int Bi = __ldg(&tb[i].z);
                const int thr = Lmax - Bi;
                int best = kLimBig;
                __syncwarp();
                for (int p = i - 1; p >= m; --p) {
                    const int Ap = __ldg(&tb[p].y);
                    if (Ap > thr) continue;  // (warp-uniform) the route (p, i] exceeds the duration limit
                    const int bb = lane - 1 + (kpi - Kw[p]);
                    if (bb >= 0 && bb <= slack) {
                        const int f = Fw[p * kLimWarpBW + bb];
                        if (f < kLimBig) best = min(best, f + Ap);
                    }
                }
                int v = best >= kLimBig ? kLimBig : best + Bi;
                if (lane > slack || kpi + lane > K) v = kLimBig;
                Fw[i * kLimWarpBW + lane] = v;
            }
            __syncwarp();
            int r = lane <= slack ? Fw[n * kLimWarpBW + lane] : kLimBig;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) r = min(r, __shfl_xor_sync(kFull, r, o));
            result = r >= kLimBig ? SPDP_INFEASIBLE : r;
        }
        if (lane == 0) {
            if (cost) cost[s] = result;
            part_add_cost(acc, result, result != SPDP_INFEASIBLE);
        }
        __syncwarp();
    }
    if (partial) {
        const Part t = block_sum(acc, red);
        if (threadIdx.x == 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_feas), (unsigned long long)t.n_feas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_infeas), (unsigned long long)t.n_infeas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sum), (unsigned long long)t.sum);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_lo), (unsigned long long)t.sq_lo);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_hi), (unsigned long long)t.sq_hi);
        }
    }
}

// (n too large for the warp kernel's shared memory) the ring passes' deferrals to the general kernel
__global__ void limits_wlist_to_general_kernel(const int2* __restrict__ wl, const unsigned* __restrict__ wc,
                                               int64_t* __restrict__ list, unsigned* __restrict__ count) {
    for (unsigned w = blockIdx.x * blockDim.x + threadIdx.x; w < *wc; w += gridDim.x * blockDim.x)
        list[atomicAdd(count, 1u)] = wl[w].x;
}

// Without a fleet limit: the duration-limited Eq. (3) sweep on a 32-entry REGISTER ring (the
// integer sweep's structure).  The duration test of a candidate depends only on the layer i and
// the age k (t(i-k, i) = A[i-k] + B[i] is scenario-invariant), so it is a per-layer bitmask
// dm[i] (bit k-1: route (i-k, i] within Lmax) built once per call into the table's .x field;
// per candidate the window test and the (warp-uniform) mask bit, then a predicated min.  Values
// G = F + A with F = +inf kept at kLimBig (a layer may have no admissible split).  A scenario
// whose window outgrows the ring is deferred to the general kernel.
__global__ void limits_dmask_kernel(int4* __restrict__ tab, int n, int Lmax) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    unsigned dm = 0u;
    if (i >= 1) {
        const int Bi = tab[i].z;
        for (int k = 1; k <= 32 && k <= i; ++k)
            if (tab[i - k].y <= Lmax - Bi) dm |= 1u << (k - 1);
    }
    tab[i].x = (int)dm;
}

__global__ void __launch_bounds__(256) split_limits_reg_kernel(const int4* __restrict__ tab, int n,
                                                               const uint16_t* __restrict__ demand, int64_t S, int Q,
                                                               int32_t* __restrict__ cost,
                                                               spdp_saa_partial* __restrict__ partial,
                                                               int64_t* __restrict__ list, unsigned* __restrict__ count) {
    constexpr int W = 32;
    __shared__ Part red[8];
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = s < S;
    const uint16_t* dcol = demand + (live ? s : S - 1);
    auto q_at = [&](int i) -> int { return i <= n ? (int)dcol[(uint32_t)__ldg(&tab[i].w)] : 0; };
    int G[W], Y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        G[k] = kLimBig;
        Y[k] = INT_MIN;  // no split point yet
    }
    G[0] = __ldg(&tab[0].y);  // position 0: F = 0, G = A[0]
    Y[0] = Q;
    int qb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) qb[k] = q_at(1 + k);
    int P = 0, fin = kLimBig;
    bool bad = false, ovf = false;
    for (int b = 1; b <= n; b += W) {  // layer i = b + j sits in slot (1 + j) mod W
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int i = b + j;
            if (i > n) break;  // warp-uniform
            const int q = qb[j % 8];
            qb[j % 8] = q_at(i + 8);
            bad |= q > Q;
            const int Pn = P + q;
            const int4 ei = __ldg(&tab[i]);
            const unsigned dm = (unsigned)ei.x;
            int best = kLimBig;
#pragma unroll
            for (int k = 1; k <= 8; ++k) {
                const int sl = (1 + j - k + 2 * W) % W;
                if (((dm >> (k - 1)) & 1u) && Y[sl] >= Pn) best = min(best, G[sl]);
            }
#pragma unroll
            for (int k0 = 9; k0 <= W; k0 += 4) {
                if (!__any_sync(kFull, Y[(1 + j - k0 + 2 * W) % W] >= Pn)) break;
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int k = k0 + v;
                    const int sl = (1 + j - k + 2 * W) % W;
                    if (((dm >> (k - 1)) & 1u) && Y[sl] >= Pn) best = min(best, G[sl]);
                }
            }
            const int si = (1 + j) % W;  // = the slot of age W, overwritten now
            ovf |= Y[si] >= Pn && i - W >= 1;
            const int F = best >= kLimBig ? kLimBig : best + ei.z;  // F(i) = min G + B[i]
            G[si] = F >= kLimBig ? kLimBig : F + ei.y;              // G(i) = F(i) + A[i]
            Y[si] = Pn + Q;
            if (i == n) fin = F;
            P = Pn;
        }
    }
    Part acc{0, 0, 0, 0, 0};
    if (live) {
        if (ovf && !bad) {
            list[atomicAdd(count, 1u)] = s;
        } else {
            const int result = (bad || fin >= kLimBig) ? SPDP_INFEASIBLE : fin;
            if (cost) cost[s] = result;
            part_add_cost(acc, result, result != SPDP_INFEASIBLE);
        }
    }
    if (partial) {
        const Part t = block_sum(acc, red);
        if (threadIdx.x == 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_feas), (unsigned long long)t.n_feas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->n_infeas), (unsigned long long)t.n_infeas);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sum), (unsigned long long)t.sum);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_lo), (unsigned long long)t.sq_lo);
            atomicAdd(reinterpret_cast<unsigned long long*>(&partial->sumsq_hi), (unsigned long long)t.sq_hi);
        }
    }
}

static int lim_num_sms() { return device_sms(); }

static size_t lim_table_bytes(int32_t n) { return align_up(sizeof(int4) * (size_t)tour_tab_stride(n), 256); }
static size_t lim_scratch_bytes(int32_t n) {
    const size_t threads = (size_t)lim_num_sms() * lim_blocks_per_sm(n) * kLimThreads;
    return align_up(3 * sizeof(int) * (size_t)(n + 1) * threads, 256);
}
constexpr size_t kLimSmemCap = 200 * 1024;

template <int BW, int NT, int kRing>
static size_t ring_smem(int32_t n) {
    return sizeof(int) * (size_t)kRing * NT * (BW + (BW > 1 ? 2 : 1)) +
           (n <= kLimTableSmemMaxN ? sizeof(int4) * (size_t)(n + 1) : 0);
}

template <int BW, int NT, int kRing>
static spdp_status launch_ring(cudaStream_t st, const int4* e, int n, const uint16_t* demand, int64_t S, int Q, int Lmax,
                               int K, int32_t* cost, spdp_saa_partial* partial, int2* list, unsigned* count,
                               const int2* in_list = nullptr, const unsigned* in_count = nullptr, int64_t nwork = -1) {
    const size_t smem = ring_smem<BW, NT, kRing>(n);
    if (spdp_status e = kernel_setup((const void*)split_limits_ring_kernel<BW, NT, kRing>,
                                     (int)ring_smem<BW, NT, kRing>(kLimTableSmemMaxN), -1, 0, 0, nullptr,
                                     "split_limits_ring_kernel setup"))
        return e;
    split_limits_ring_kernel<BW, NT, kRing><<<(unsigned)ceil_div(nwork < 0 ? S : nwork, NT), NT, smem, st>>>(
        e, n, demand, S, Q, Lmax, K, cost, partial, list, count, n <= kLimTableSmemMaxN ? 1 : 0, in_list, in_count);
    set_last_kernel("split_limits_ring_kernel<%d,%d>", BW, kRing);
    return last_launch("split_limits_ring_kernel");
}

}  // namespace spdp

using namespace spdp;

extern "C" size_t spdp_limits_workspace_bytes(int32_t n, int64_t S) {
    if (n < 1 || S < 1) return 0;
    return lim_table_bytes(n) + lim_scratch_bytes(n) + align_up(sizeof(int64_t) * (size_t)S, 256) + 256 +
           align_up(sizeof(int2) * (size_t)(kLimBands + 1) * (size_t)S, 256) + 256;
}

extern "C" spdp_status spdp_split_eval_limits(const int32_t* tour, const int32_t* dist, int32_t n,
                                              const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                              int32_t max_duration, int32_t max_routes, int32_t* cost,
                                              spdp_saa_partial* partial, void* ws, size_t ws_bytes, uint32_t flags,
                                              spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval_limits");
    const char* fn = "spdp_split_eval_limits";
    if (n < 1) return fail(SPDP_E_USAGE, "%s: n=%d < 1", fn, n);
    if (n > SPDP_MAX_N) return fail(SPDP_E_RESOURCE, "%s: n=%d > SPDP_MAX_N=%d", fn, n, SPDP_MAX_N);
    if (S < 1) return fail(SPDP_E_USAGE, "%s: S=%lld < 1", fn, (long long)S);
    if (Q < 1) return fail(SPDP_E_USAGE, "%s: Q=%d < 1 (SPEC:34)", fn, Q);
    if (ld < S || (ld % 8) != 0) return fail(SPDP_E_USAGE, "%s: ld=%lld must be >= S and a multiple of 8", fn, (long long)ld);
    if (!tour || !dist || !demand || !ws) return fail(SPDP_E_USAGE, "%s: NULL required pointer", fn);
    if (((uintptr_t)demand & 15u) != 0) return fail(SPDP_E_USAGE, "%s: demand must be 16-byte aligned", fn);
    if (ws_bytes < spdp_limits_workspace_bytes(n, S)) return fail(SPDP_E_USAGE, "%s: workspace too small", fn);
    if ((uint64_t)n * (uint64_t)ld >= (1ull << 32)) return fail(SPDP_E_RESOURCE, "%s: n ld must stay below 2^32", fn);
    if (S >= (1LL << 31)) return fail(SPDP_E_RESOURCE, "%s: S >= 2^31", fn);
    cudaStream_t st = (cudaStream_t)stream;
    char* w = static_cast<char*>(ws);
    int4* e = reinterpret_cast<int4*>(w);
    int* scratch = reinterpret_cast<int*>(w + lim_table_bytes(n));
    int64_t* list = reinterpret_cast<int64_t*>(w + lim_table_bytes(n) + lim_scratch_bytes(n));
    unsigned* count = reinterpret_cast<unsigned*>(w + lim_table_bytes(n) + lim_scratch_bytes(n) +
                                                  align_up(sizeof(int64_t) * (size_t)S, 256));
    spdp_status rc = launch_tour_table(tour, 1, nullptr, n, dist, ld, e, nullptr, st);
    if (rc) return rc;
    if (partial && (rc = cuda_check(cudaMemsetAsync(partial, 0, sizeof(spdp_saa_partial), st), "cudaMemsetAsync(partial)")))
        return rc;
    // band lists of the fleet passes: [kLimBands][S] {scenario, slack} and their counts
    int2* blists = reinterpret_cast<int2*>(reinterpret_cast<char*>(count) + 256);
    unsigned* bcounts = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(blists) +
                                                    align_up(sizeof(int2) * (size_t)(kLimBands + 1) * (size_t)S, 256));
    if ((rc = cuda_check(cudaMemsetAsync(count, 0, sizeof(unsigned), st), "cudaMemsetAsync(count)"))) return rc;
    if ((rc = cuda_check(cudaMemsetAsync(bcounts, 0, (kLimBands + 1) * sizeof(unsigned), st), "cudaMemsetAsync(bcounts)")))
        return rc;
    const int Qe = (int)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    const int Lmax = max_duration < 0 ? INT_MAX / 2 : max_duration;
    const bool fleet = max_routes > 0 && max_routes < n;
    const int K = fleet ? max_routes : 0;
    prof_begin(st);
    // (1) the ring kernel for every scenario; (2) the general kernel for the ones it deferred
    const bool general_only = (flags & SPDP_F_SCRATCH_GLOBAL) != 0;
    if (!general_only) {
        // fleet: the classify pass (infeasible scenarios finished, the rest listed by the band width their
        // slack needs), then one 16-position-ring pass per band width 2 / 4 / 8 / 16 over its list
        // (measured at C2, K = 27: one natural-order pass with 8 counts per position 3.9 ms, whose warps
        // ran every lane at the widest band of the warp, infeasible lanes idle)
        if (fleet) {
            const size_t per_warp = sizeof(int) * (size_t)(n + 1) * (kLimWarpBW + 2);
            const bool warp_fits = per_warp <= kLimSmemCap;
            limits_classify_kernel<<<(unsigned)ceil_div(S, 256), 256, 0, st>>>(e, n, demand, S, Qe, K, cost, partial,
                                                                            blists, S, bcounts, list, count,
                                                                            warp_fits ? 1 : 0);
            if ((rc = last_launch("limits_classify_kernel"))) return rc;
            int2* wl = blists + (int64_t)kLimBands * S;  // the warp kernel's list (+ the ring passes' deferrals)
            unsigned* wc = bcounts + kLimBands;
            if (!rc) rc = launch_ring<2, 64, 16>(st, e, n, demand, S, Qe, Lmax, K, cost, partial, wl, wc, blists, bcounts, S);
            if (!rc) rc = launch_ring<4, 64, 16>(st, e, n, demand, S, Qe, Lmax, K, cost, partial, wl, wc, blists + S,
                                                 bcounts + 1, S);
            if (!rc) rc = launch_ring<8, 64, 16>(st, e, n, demand, S, Qe, Lmax, K, cost, partial, wl, wc, blists + 2 * S,
                                                 bcounts + 2, S);
            if (!rc) rc = launch_ring<16, 64, 16>(st, e, n, demand, S, Qe, Lmax, K, cost, partial, wl, wc, blists + 3 * S,
                                                  bcounts + 3, S);
            if (rc) return rc;
            if (warp_fits) {
                int warps = (int)(kLimSmemCap / per_warp);
                warps = warps > 8 ? 8 : warps;
                if ((rc = kernel_setup((const void*)split_limits_warp_kernel, (int)kLimSmemCap, -1, 0, 0, nullptr,
                                       "split_limits_warp_kernel setup")))
                    return rc;
                split_limits_warp_kernel<<<(unsigned)(lim_num_sms() * 2), warps * 32, per_warp * warps, st>>>(
                    e, n, demand, Qe, Lmax, K, cost, partial, wl, wc);
                if ((rc = last_launch("split_limits_warp_kernel"))) return rc;
            } else {
                limits_wlist_to_general_kernel<<<lim_num_sms(), 256, 0, st>>>(wl, wc, list, count);
                if ((rc = last_launch("limits_wlist_to_general_kernel"))) return rc;
            }
            set_last_kernel("split_limits_ring_kernel<2|4|8|16,16>");
        } else {  // duration only (or no limit): the register ring with the per-layer duration bitmask
            limits_dmask_kernel<<<(unsigned)ceil_div(n + 1, 256), 256, 0, st>>>(e, n, Lmax);
            if ((rc = last_launch("limits_dmask_kernel"))) return rc;
            split_limits_reg_kernel<<<(unsigned)ceil_div(S, 256), 256, 0, st>>>(e, n, demand, S, Qe, cost, partial,
                                                                              list, count);
            set_last_kernel("split_limits_reg_kernel<32>");
            rc = last_launch("split_limits_reg_kernel");
        }
        if (rc) return rc;
    }
    const size_t smem = n <= kLimTableSmemMaxN ? sizeof(int4) * (size_t)(n + 1) : 0;
    if ((rc = kernel_setup((const void*)split_limits_kernel, (int)kLimSmemCap, -1, 0, 0, nullptr, "split_limits_kernel setup")))
        return rc;
    const int per_sm = lim_blocks_per_sm(n);
    int64_t grid = (int64_t)lim_num_sms() * per_sm;
    const int64_t need = ceil_div(S, kLimThreads);
    if (grid > need) grid = need;
    split_limits_kernel<<<(unsigned)grid, kLimThreads, smem, st>>>(e, n, demand, S, Qe, Lmax, K, cost, partial, scratch,
                                                                  general_only ? nullptr : list,
                                                                  general_only ? nullptr : count);
    prof_end(st);
    if (general_only) set_last_kernel("split_limits_kernel<global>");
    return last_launch("split_limits_kernel");
}
