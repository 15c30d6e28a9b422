// order.cu -- scenario ordering for the batched / repeated evaluation (DESIGN §"scenario order").
//
// The Eq. (3) window of a scenario at layer i is set by its loads, and a warp runs
// every layer at the deepest window among its lanes (the divergence the paper's mask formulation
// is there to bound).  Scenarios with a larger total demand have shorter windows
// everywhere, so sorting the columns of the demand matrix by total demand puts scenarios with
// similar windows into the same warp: the sweep then evaluates fewer masked candidates per layer
// (C3: -12 % sweep time; the costs, per scenario, and the SAA sums are unchanged -- a permutation).
// The order is a preprocessing of a scenario set that many tours are evaluated on (HGS, batched
// mode); it is done once per set.
//
//   key(s)    = sum_c demand[c][s]                  (exact, uint32: n * 65535 < 2^32)
//   bucket(s) = floor(key(s) * kOrdBuckets / (kmax + 1)),   kmax = max_s key(s)
//   perm      = per segment of kOrdSeg consecutive scenarios, the segment's scenarios in
//               increasing bucket order, increasing index within a bucket (a stable counting
//               sort per segment: deterministic; the segments stay in place, so the gather
//               below reads each row within a 128 KB window: L2-resident, not scattered over
//               the matrix -- and a warp's 64 scenarios come from one segment anyway)
//   out[c][j] = demand[c][perm[j]]
#include "common.cuh"

namespace spdp {

constexpr int kOrdBuckets = 1024;
constexpr int kOrdChunk = 4096;  // scenarios per block of the histogram / scatter passes
constexpr int kOrdSeg = 65536;   // scenarios per sorted segment (a multiple of kOrdChunk)
constexpr int kOrdCps = kOrdSeg / kOrdChunk;  // chunks per segment

// key(s) and the maximum key
__global__ void __launch_bounds__(256) order_keys_kernel(const uint16_t* __restrict__ demand, int64_t ld, int n,
                                                         int64_t S, uint32_t* __restrict__ key,
                                                         unsigned* __restrict__ kmax) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t k = 0u;
    if (s < S) {
        for (int c = 0; c < n; ++c) k += demand[(int64_t)c * ld + s];
        key[s] = k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) k = max(k, __shfl_xor_sync(kFull, k, o));
    if ((threadIdx.x & 31) == 0) atomicMax(kmax, k);
}

__device__ __forceinline__ int order_bucket(uint32_t k, uint32_t kmax) {
    return (int)(((uint64_t)k * kOrdBuckets) / ((uint64_t)kmax + 1u));
}

// per block (a chunk of kOrdChunk scenarios): the bucket histogram, into hist[seg][b][chunk in seg]
__global__ void __launch_bounds__(256) order_hist_kernel(const uint32_t* __restrict__ key, int64_t S,
                                                         const unsigned* __restrict__ kmax, unsigned* __restrict__ hist,
                                                         int nblocks) {
    __shared__ unsigned h[kOrdBuckets];
    for (int b = threadIdx.x; b < kOrdBuckets; b += blockDim.x) h[b] = 0u;
    __syncthreads();
    const uint32_t km = *kmax;
    const int64_t s0 = (int64_t)blockIdx.x * kOrdChunk;
    for (int i = threadIdx.x; i < kOrdChunk; i += blockDim.x) {
        const int64_t s = s0 + i;
        if (s < S) atomicAdd(&h[order_bucket(key[s], km)], 1u);
    }
    __syncthreads();
    const int64_t seg = blockIdx.x / kOrdCps, cin = blockIdx.x % kOrdCps;
    for (int b = threadIdx.x; b < kOrdBuckets; b += blockDim.x) hist[(seg * kOrdBuckets + b) * kOrdCps + cin] = h[b];
}

// exclusive scan of each segment's histogram (kOrdBuckets * kOrdCps entries, bucket-major) in place,
// offset by the segment's first column: one block per segment
__global__ void __launch_bounds__(1024) order_scan_kernel(unsigned* __restrict__ hist_all) {
    const int64_t len = (int64_t)kOrdBuckets * kOrdCps;
    unsigned* hist = hist_all + (int64_t)blockIdx.x * len;
    __shared__ unsigned warp_tot[32];
    __shared__ unsigned carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = (unsigned)blockIdx.x * (unsigned)kOrdSeg;
    __syncthreads();
    for (int64_t base = 0; base < len; base += 1024) {
        const int64_t i = base + tid;
        const unsigned v = i < len ? hist[i] : 0u;
        unsigned x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            unsigned t = warp_tot[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, t, o);
                if (lane >= o) t += y;
            }
            warp_tot[lane] = t;  // inclusive warp totals
        }
        __syncthreads();
        const unsigned excl = carry + (wid ? warp_tot[wid - 1] : 0u) + x - v;
        if (i < len) hist[i] = excl;
        __syncthreads();
        if (tid == 0) carry += warp_tot[31];
        __syncthreads();
    }
}

// stable scatter: one warp per chunk walks its scenarios in index order, 32 at a time; a lane's slot
// is its bucket's running offset plus its rank among the lanes of the same bucket before it
__global__ void __launch_bounds__(32) order_scatter_kernel(const uint32_t* __restrict__ key, int64_t S,
                                                           const unsigned* __restrict__ kmax,
                                                           const unsigned* __restrict__ hist, int nblocks,
                                                           int32_t* __restrict__ perm) {
    __shared__ unsigned off[kOrdBuckets];
    const int lane = threadIdx.x;
    const int64_t seg = blockIdx.x / kOrdCps, cin = blockIdx.x % kOrdCps;
    for (int b = lane; b < kOrdBuckets; b += 32) off[b] = hist[(seg * kOrdBuckets + b) * kOrdCps + cin];
    __syncwarp();
    const uint32_t km = *kmax;
    const int64_t s0 = (int64_t)blockIdx.x * kOrdChunk;
    for (int i0 = 0; i0 < kOrdChunk; i0 += 32) {
        const int64_t s = s0 + i0 + lane;
        const bool live = s < S;
        const int b = live ? order_bucket(key[s], km) : -1 - lane;  // (dead lanes: distinct, never matched)
        const unsigned grp = __match_any_sync(kFull, b);
        const unsigned rank = __popc(grp & ((1u << lane) - 1u));
        const unsigned base = live ? off[b] : 0u;
        if (live) perm[base + rank] = (int32_t)s;
        __syncwarp();
        if (live && rank == 0u) off[b] = base + __popc(grp);
        __syncwarp();
    }
}

// out[c][j] = demand[c][perm[j]]
__global__ void __launch_bounds__(256) order_permute_kernel(const uint16_t* __restrict__ demand, int64_t ld, int n,
                                                            int64_t S, const int32_t* __restrict__ perm,
                                                            uint16_t* __restrict__ out, int64_t ld_out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    const int64_t s = perm[j];
    for (int c = 0; c < n; ++c) out[(int64_t)c * ld_out + j] = demand[(int64_t)c * ld + s];
}

static int64_t ord_blocks(int64_t S) { return ceil_div(S, kOrdChunk); }
static int64_t ord_segs(int64_t S) { return ceil_div(S, kOrdSeg); }

}  // namespace spdp

using namespace spdp;

extern "C" size_t spdp_order_workspace_bytes(int64_t S) {
    if (S < 1) return 0;
    return align_up(sizeof(uint32_t) * (size_t)S, 256) + 256 +
           align_up(sizeof(unsigned) * (size_t)kOrdBuckets * kOrdCps * (size_t)ord_segs(S), 256);
}

extern "C" spdp_status spdp_order_scenarios(const uint16_t* demand, int64_t ld, int32_t n, int64_t S, uint16_t* out,
                                            int64_t ld_out, int32_t* perm, void* ws, size_t ws_bytes,
                                            spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_order_scenarios");
    const char* fn = "spdp_order_scenarios";
    if (n < 1 || S < 1) return fail(SPDP_E_USAGE, "%s: n and S must be >= 1", fn);
    if (n > SPDP_MAX_N) return fail(SPDP_E_RESOURCE, "%s: n=%d > SPDP_MAX_N=%d", fn, n, SPDP_MAX_N);
    if (!demand || !perm || !ws) return fail(SPDP_E_USAGE, "%s: NULL required pointer", fn);
    if (ld < S || (out && ld_out < S)) return fail(SPDP_E_USAGE, "%s: ld < S", fn);
    if (S >= (1LL << 31)) return fail(SPDP_E_RESOURCE, "%s: S >= 2^31", fn);
    if (out == demand) return fail(SPDP_E_USAGE, "%s: out must not alias demand", fn);
    if (ws_bytes < spdp_order_workspace_bytes(S)) return fail(SPDP_E_USAGE, "%s: workspace too small", fn);
    cudaStream_t st = (cudaStream_t)stream;
    char* w = static_cast<char*>(ws);
    uint32_t* key = reinterpret_cast<uint32_t*>(w);
    unsigned* kmax = reinterpret_cast<unsigned*>(w + align_up(sizeof(uint32_t) * (size_t)S, 256));
    unsigned* hist = kmax + 64;
    const int nb = (int)ord_blocks(S);
    spdp_status rc = cuda_check(cudaMemsetAsync(kmax, 0, sizeof(unsigned), st), "cudaMemsetAsync(kmax)");
    if (rc) return rc;
    order_keys_kernel<<<(unsigned)ceil_div(S, 256), 256, 0, st>>>(demand, ld, n, S, key, kmax);
    if ((rc = last_launch("order_keys_kernel"))) return rc;
    if ((rc = cuda_check(cudaMemsetAsync(hist, 0, sizeof(unsigned) * (size_t)kOrdBuckets * kOrdCps * ord_segs(S), st),
                         "cudaMemsetAsync(hist)")))
        return rc;  // (the last segment's missing chunks count zero)
    order_hist_kernel<<<(unsigned)nb, 256, 0, st>>>(key, S, kmax, hist, nb);
    if ((rc = last_launch("order_hist_kernel"))) return rc;
    order_scan_kernel<<<(unsigned)ord_segs(S), 1024, 0, st>>>(hist);
    if ((rc = last_launch("order_scan_kernel"))) return rc;
    order_scatter_kernel<<<(unsigned)nb, 32, 0, st>>>(key, S, kmax, hist, nb, perm);
    if ((rc = last_launch("order_scatter_kernel"))) return rc;
    if (out) {
        order_permute_kernel<<<(unsigned)ceil_div(S, 256), 256, 0, st>>>(demand, ld, n, S, perm, out, ld_out);
        if ((rc = last_launch("order_permute_kernel"))) return rc;
    }
    return SPDP_OK;
}
