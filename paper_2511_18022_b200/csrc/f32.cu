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

namespace spdp {

struct F32Pos {
    double Dd, c0, ci0;  // Dd[i], c[0][s_i], c[s_i][0]
    uint32_t rowoff;     // (s_i - 1) * ld (n ld < 2^32)
    uint32_t pad;
};

constexpr int kF32SmemMaxN = 4095;  // position table in shared memory up to 128 KB

__global__ void f32_prep_kernel(const int32_t* __restrict__ tour, int n, const double* __restrict__ dist, int64_t ld,
                                F32Pos* __restrict__ tab) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t N1 = (int64_t)n + 1;
    auto node = [&](int i) -> int {  // customer at 0-based position i, clamped to 1..n
        const int c = tour[i];
        return c < 1 ? 1 : (c > n ? n : c);
    };
    double D = 0.0;
    tab[0] = F32Pos{0.0, 0.0, 0.0, 0u, 0u};
    for (int i = 1; i <= n; ++i) {
        const int c = node(i - 1);
        if (i >= 2) D = __dadd_rn(D, dist[(int64_t)node(i - 2) * N1 + c]);
        tab[i] = F32Pos{D, dist[c], dist[(int64_t)c * N1], (uint32_t)((uint64_t)(c - 1) * (uint64_t)ld), 0u};
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
    if (table_in_smem) {
        for (int i = threadIdx.x; i <= n; i += blockDim.x) ftab[i] = tab_g[i];
        __syncthreads();
        tab = ftab;
    }
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= (list ? (int64_t)*count : S)) return;
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

// The band table of the ring kernel: tb[i][k - 1] = T32(i - k, i), k = 1..W (the route costs of
// every candidate the ring can hold, scenario-invariant), formed in the oracle's fp64 order.
__global__ void f32_band_kernel(const F32Pos* __restrict__ tab, int n, int W, float* __restrict__ tb) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)(n + 1) * W) return;
    const int i = (int)(idx / W), k = (int)(idx % W) + 1;
    float v = 0.0f;  // (k > i: no such split point; its ring slot is never in a window)
    if (k <= i) {
        const int p = i - k;
        v = __double2float_rn(__dadd_rn(__dadd_rn(tab[p + 1].c0, __dsub_rn(tab[i].Dd, tab[p + 1].Dd)), tab[i].ci0));
    }
    tb[idx] = v;
}

// The ring kernel (the common case): one scenario per thread, a W-entry register ring of
// {f(p), P(p) + Q} (slot p mod W), layers unrolled by W, each candidate one fp32 add of the
// band-table entry and a masked min; ages 1..8 unconditionally, then groups of 4 behind a warp
// vote.  A scenario whose window outgrows the ring is listed for the general kernel.
constexpr int kF32W = 32;
constexpr int kF32Pf = 8;
constexpr int kF32BandSmemMaxN = 375;  // band table (n + 1) W 4 B staged in shared memory up to 48 KB

__global__ void __launch_bounds__(256) split_f32_ring_kernel(const F32Pos* __restrict__ tab, const float* __restrict__ tb_g,
                                                             int n, const uint16_t* __restrict__ demand, int64_t S,
                                                             int Q, float* __restrict__ cost, int64_t* __restrict__ list,
                                                             unsigned* __restrict__ count, int band_in_smem) {
    constexpr int W = kF32W;
    extern __shared__ float tbs[];
    const float* tb = tb_g;
    uint32_t* rows = reinterpret_cast<uint32_t*>(tbs + (n + 1) * W);  // row offsets, padded with 0
    if (band_in_smem) {
        for (int i = threadIdx.x; i < (n + 1) * W; i += blockDim.x) tbs[i] = tb_g[i];
        for (int i = threadIdx.x; i < n + 1 + kF32Pf; i += blockDim.x) rows[i] = i <= n ? tab[i].rowoff : 0u;
        __syncthreads();
        tb = tbs;
    }
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = s < S;
    const uint16_t* dcol = demand + (live ? s : S - 1);
    auto q_at = [&](int i) -> int {
        if (band_in_smem) return (int)dcol[rows[i]];  // (padded past n: row 0)
        return i <= n ? (int)dcol[tab[i].rowoff] : 0;
    };
    float F[W];
    int Y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        F[k] = 0.0f;
        Y[k] = INT_MIN;  // no split point yet: never in a window
    }
    Y[0] = Q;  // position 0: f = 0, P = 0
    int qb[kF32Pf];
#pragma unroll
    for (int k = 0; k < kF32Pf; ++k) qb[k] = q_at(1 + k);
    int P = 0;
    bool bad = false, ovf = false;
    float fin = 0.0f;
    for (int b = 1; b <= n; b += W) {  // layer i = b + j sits in slot (1 + j) mod W
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int i = b + j;
            if (i > n) break;  // warp-uniform
            const int q = qb[j % kF32Pf];
            qb[j % kF32Pf] = q_at(i + kF32Pf);
            bad |= q > Q;
            const int Pn = P + q;
            const float* row = tb + (int64_t)i * W;
            float best = INFINITY;
#pragma unroll
            for (int k = 1; k <= 8; ++k) {
                const int sl = (1 + j - k + 2 * W) % W;
                if (Y[sl] >= Pn) best = fminf(best, __fadd_rn(F[sl], row[k - 1]));
            }
#pragma unroll
            for (int k0 = 9; k0 <= W; k0 += 4) {
                if (!__any_sync(kFull, Y[(1 + j - k0 + 2 * W) % W] >= Pn)) break;
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int k = k0 + v;
                    if (k <= W) {
                        const int sl = (1 + j - k + 2 * W) % W;
                        if (Y[sl] >= Pn) best = fminf(best, __fadd_rn(F[sl], row[k - 1]));
                    }
                }
            }
            const int si = (1 + j) % W;  // = the slot of age W, overwritten now
            ovf |= Y[si] >= Pn && i - W >= 1;  // an older split point may still be in the window
            F[si] = best;
            Y[si] = Pn + Q;
            if (i == n) fin = best;
            P = Pn;
        }
    }
    if (!live) return;
    if (bad) cost[s] = INFINITY;
    else if (ovf) list[atomicAdd(count, 1u)] = s;
    else cost[s] = fin;
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

static size_t f32_table_bytes(int32_t n) { return align_up(sizeof(F32Pos) * (size_t)(n + 1 + kF32Pf), 256); }
static size_t f32_band_bytes(int32_t n) { return align_up(sizeof(float) * (size_t)(n + 1) * kF32W, 256); }
static size_t f32_list_bytes(int64_t S) { return align_up(sizeof(int64_t) * (size_t)S, 256) + 256; }

}  // namespace spdp

using namespace spdp;

extern "C" size_t spdp_f32_workspace_bytes(int32_t n, int64_t S) {
    if (n < 1 || S < 1) return 0;
    return f32_table_bytes(n) + f32_band_bytes(n) + f32_list_bytes(S) +
           align_up(sizeof(float) * (size_t)(n + 1) * (size_t)S, 256);
}

extern "C" spdp_status spdp_split_eval_f32(const int32_t* tour, const double* dist, int32_t n, const uint16_t* demand,
                                           int64_t ld, int64_t S, int32_t Q, float* cost, void* ws, size_t ws_bytes,
                                           spdp_stream_t stream) {
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
    float* tb = reinterpret_cast<float*>(w + f32_table_bytes(n));
    int64_t* list = reinterpret_cast<int64_t*>(w + f32_table_bytes(n) + f32_band_bytes(n));
    unsigned* count = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(list) + align_up(sizeof(int64_t) * (size_t)S, 256));
    float* fsc = reinterpret_cast<float*>(w + f32_table_bytes(n) + f32_band_bytes(n) + f32_list_bytes(S));
    f32_prep_kernel<<<1, 32, 0, st>>>(tour, n, dist, ld, tab);
    spdp_status rc = last_launch("f32_prep_kernel");
    if (rc) return rc;
    const int64_t nb = (int64_t)(n + 1) * kF32W;
    f32_band_kernel<<<(unsigned)ceil_div(nb, 256), 256, 0, st>>>(tab, n, kF32W, tb);
    if ((rc = last_launch("f32_band_kernel"))) return rc;
    if ((rc = cuda_check(cudaMemsetAsync(count, 0, sizeof(unsigned), st), "cudaMemsetAsync(count)"))) return rc;
    const int Qe = (int)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    const bool bsm = n <= kF32BandSmemMaxN;
    prof_begin(st);
    // (1) the ring kernel for every scenario; (2) the general kernel for the ones it deferred
    split_f32_ring_kernel<<<(unsigned)ceil_div(S, 256), 256,
                            bsm ? sizeof(float) * (size_t)nb + sizeof(uint32_t) * (size_t)(n + 1 + kF32Pf) : 0, st>>>(
        tab, tb, n, demand, S, Qe, cost, list, count, bsm ? 1 : 0);
    if ((rc = last_launch("split_f32_ring_kernel"))) return rc;
    const bool tsm = n <= kF32SmemMaxN;
    if ((rc = kernel_setup((const void*)split_f32_kernel, (int)(sizeof(F32Pos) * (kF32SmemMaxN + 1)), -1, 0, 0, nullptr,
                           "split_f32_kernel setup")))
        return rc;
    split_f32_kernel<<<(unsigned)ceil_div(S, 256), 256, tsm ? sizeof(F32Pos) * (size_t)(n + 1) : 0, st>>>(
        tab, n, demand, S, Qe, fsc, cost, tsm ? 1 : 0, list, count);
    prof_end(st);
    set_last_kernel("split_f32_ring_kernel<%d>", kF32W);
    return last_launch("split_f32_kernel");
}

extern "C" spdp_status spdp_split_eval_batch_f32(const int32_t* tours, int32_t T, const double* dist, int32_t n,
                                                 const uint16_t* demand, int64_t ld, int64_t S, int32_t Q, float* cost,
                                                 void* ws, size_t ws_bytes, spdp_stream_t stream) {
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
