// limits.cu -- f4: the split with a route-duration limit and a
// fleet limit (DESIGN R24; "route length/duration constraints, if
// applicable"; "three vehicles available"):
//   a route (p, i] is admissible iff  sum_{k=p+1}^{i} q <= Q  (Eq. (2)) and
//   t(p, i) = A[p] + B[i] <= Lmax  (duration = route cost, scenario-invariant);
//   F_0(0) = 0,  F_k(i) = min_{admissible (p, i]} F_{k-1}(p) + t(p, i),
//   cost = min_{k <= K} F_k(n)   (K <= 0: no fleet limit -> one pass of Eq. (3)).
// The fleet limit adds the vehicle-count layer dimension to the layered DAG: K
// passes of the Eq. (3) sweep, pass k reading F_{k-1}.  The masks mask(i) of
// Eq. (2) do not depend on k: they are computed once per scenario (two pointers)
// and reused by every pass.
#include <climits>

#include "common.cuh"
#include "split_ws.cuh"

namespace spdp {

constexpr int kLimBig = 1 << 30;  // no admissible split (above every finite value, R17 range bound)
constexpr int kLimThreads = 64;
constexpr int kLimGlobalBlocksPerSm = 4;  // persistent grid of the workspace-scratch variant

// One scenario per thread, grid-stride over scenarios.  Per-thread arrays of n+1 ints
// (mask, F_a, F_b; element p of thread r at base[p * stride + r], conflict-free /
// coalesced) live in shared memory (use_smem) or in the workspace.  The tour's
// position table {row, A, B, row offset} is staged in shared memory.
__global__ void __launch_bounds__(kLimThreads) split_limits_kernel(const int4* __restrict__ e, int n,
                                                                  const uint16_t* __restrict__ demand, int64_t S, int Q,
                                                                  int Lmax, int K, int32_t* __restrict__ cost,
                                                                  spdp_saa_partial* __restrict__ partial, int* gscratch,
                                                                  int use_smem) {
    extern __shared__ int4 sm4[];
    __shared__ Part red[kLimThreads / 32];
    int4* tb = sm4;
    for (int i = threadIdx.x; i <= n; i += blockDim.x) tb[i] = e[i];
    __syncthreads();
    int* arr;
    int64_t stride;
    int64_t r;
    if (use_smem) {
        arr = reinterpret_cast<int*>(sm4 + (n + 1));
        stride = blockDim.x;
        r = threadIdx.x;
    } else {
        arr = gscratch;
        stride = (int64_t)gridDim.x * blockDim.x;
        r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    }
    int* Mk = arr + r;
    int* Fa = arr + (int64_t)(n + 1) * stride + r;
    int* Fb = arr + 2 * (int64_t)(n + 1) * stride + r;
    const bool fleet = K > 0 && K < n;
    Part acc{0, 0, 0, 0, 0};
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
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
            int m = 0, Pm = 0;
            for (int i = 1; i <= n; ++i) {
                const int Pi = Fb[(int64_t)i * stride];
                while (Pi - Pm > Q) Pm = Fb[(int64_t)(++m) * stride];
                Mk[(int64_t)i * stride] = m;
            }
            // one pass of the layered sweep: cur[i] = min_{admissible p} prev[p] + A[p] + B[i]
            auto pass = [&](const int* prev, int* cur) -> bool {
                bool any = false;
                for (int i = 1; i <= n; ++i) {
                    const int Bi = tb[i].z;
                    const int thr = Lmax - Bi;  // duration: A[p] <= Lmax - B[i]
                    const int lo = Mk[(int64_t)i * stride];
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
            } else {
                Fa[0] = 0;
                for (int i = 1; i <= n; ++i) Fa[(int64_t)i * stride] = kLimBig;  // F_0
                int* prev = Fa;
                int* cur = Fb;  // (the prefix loads are no longer needed)
                res = kLimBig;
                for (int k = 1; k <= K; ++k) {
                    cur[0] = kLimBig;
                    const bool any = pass(prev, cur);
                    res = min(res, cur[(int64_t)n * stride]);
                    int* tmp = prev;
                    prev = cur;
                    cur = tmp;
                    if (!any) break;
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

static int lim_num_sms() {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

static size_t lim_table_bytes(int32_t n) { return align_up(sizeof(int4) * (size_t)(n + 1), 256); }
static size_t lim_smem_bytes(int32_t n, bool arrays) {
    return sizeof(int4) * (size_t)(n + 1) + (arrays ? 3 * sizeof(int) * (size_t)(n + 1) * kLimThreads : 0);
}
constexpr size_t kLimSmemCap = 200 * 1024;

}  // namespace spdp

using namespace spdp;

extern "C" size_t spdp_limits_workspace_bytes(int32_t n) {
    if (n < 1) return 0;
    const size_t threads = (size_t)lim_num_sms() * kLimGlobalBlocksPerSm * kLimThreads;
    return lim_table_bytes(n) + align_up(3 * sizeof(int) * (size_t)(n + 1) * threads, 256);
}

extern "C" spdp_status spdp_split_eval_limits(const int32_t* tour, const int32_t* dist, int32_t n,
                                              const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                              int32_t max_duration, int32_t max_routes, int32_t* cost,
                                              spdp_saa_partial* partial, void* ws, size_t ws_bytes, uint32_t flags,
                                              spdp_stream_t stream) {
    const char* fn = "spdp_split_eval_limits";
    if (n < 1) return fail(SPDP_E_USAGE, "%s: n=%d < 1", fn, n);
    if (n > SPDP_MAX_N) return fail(SPDP_E_RESOURCE, "%s: n=%d > SPDP_MAX_N=%d", fn, n, SPDP_MAX_N);
    if (S < 1) return fail(SPDP_E_USAGE, "%s: S=%lld < 1", fn, (long long)S);
    if (Q < 1) return fail(SPDP_E_USAGE, "%s: Q=%d < 1 (SPEC:34)", fn, Q);
    if (ld < S || (ld % 8) != 0) return fail(SPDP_E_USAGE, "%s: ld=%lld must be >= S and a multiple of 8", fn, (long long)ld);
    if (!tour || !dist || !demand || !ws) return fail(SPDP_E_USAGE, "%s: NULL required pointer", fn);
    if (((uintptr_t)demand & 15u) != 0) return fail(SPDP_E_USAGE, "%s: demand must be 16-byte aligned", fn);
    if (ws_bytes < spdp_limits_workspace_bytes(n)) return fail(SPDP_E_USAGE, "%s: workspace too small", fn);
    if ((uint64_t)n * (uint64_t)ld >= (1ull << 32)) return fail(SPDP_E_RESOURCE, "%s: n ld must stay below 2^32", fn);
    cudaStream_t st = (cudaStream_t)stream;
    char* w = static_cast<char*>(ws);
    int4* e = reinterpret_cast<int4*>(w);
    int* scratch = reinterpret_cast<int*>(w + lim_table_bytes(n));
    spdp_status rc = launch_tour_table(tour, 1, nullptr, n, dist, ld, e, nullptr, st);
    if (rc) return rc;
    if (partial && (rc = cuda_check(cudaMemsetAsync(partial, 0, sizeof(spdp_saa_partial), st), "cudaMemsetAsync(partial)")))
        return rc;
    const int Qe = (int)((int64_t)Q > (int64_t)n * 65535 ? (int64_t)n * 65535 : Q);
    const int Lmax = max_duration < 0 ? INT_MAX / 2 : max_duration;
    const bool smem_ok = lim_smem_bytes(n, true) <= kLimSmemCap && !(flags & SPDP_F_SCRATCH_GLOBAL);
    const size_t smem = lim_smem_bytes(n, smem_ok);
    if (smem > kLimSmemCap) return fail(SPDP_E_RESOURCE, "%s: n=%d too large for the staged table", fn, n);
    static bool attr = false;
    if (!attr) {
        cudaError_t err = cudaFuncSetAttribute(split_limits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kLimSmemCap);
        if (err != cudaSuccess) return cuda_check(err, "cudaFuncSetAttribute(split_limits_kernel)");
        attr = true;
    }
    int per_sm = kLimGlobalBlocksPerSm;
    if (smem_ok) {
        int occ = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, split_limits_kernel, kLimThreads, smem) != cudaSuccess ||
            occ < 1)
            occ = 1;
        per_sm = occ;
    }
    int64_t grid = (int64_t)lim_num_sms() * per_sm;
    const int64_t need = ceil_div(S, kLimThreads);
    if (grid > need) grid = need;
    prof_begin(st);
    split_limits_kernel<<<(unsigned)grid, kLimThreads, smem, st>>>(e, n, demand, S, Qe, Lmax, max_routes, cost, partial,
                                                                  scratch, smem_ok ? 1 : 0);
    prof_end(st);
    set_last_kernel("split_limits_kernel<%s>", smem_ok ? "smem" : "global");
    return last_launch("split_limits_kernel");
}
