// common.cuh -- shared device/host helpers of libspdp (product code; never
// includes or links anything under oracle/).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <utility>

#include "../../include/spdp.h"

namespace spdp {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// NVTX range around every C-ABI entry point (SURVEY §5 tracing: the calls show up by name on an
// Nsight Systems timeline; header-only NVTX v3, a no-op without an attached tool).
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
    NvtxScope(const NvtxScope&) = delete;
    NvtxScope& operator=(const NvtxScope&) = delete;
};

// Thread-local error message (spdp_last_error).
void set_error(const char* fmt, ...);
spdp_status fail(spdp_status st, const char* fmt, ...);
spdp_status cuda_check(cudaError_t e, const char* what);
spdp_status last_launch(const char* what);

// spdp_set_profile_events hook: record around the dominant kernel if set.
void prof_begin(cudaStream_t st);
void prof_end(cudaStream_t st);
// spdp_last_kernel(): record the name of the sweep kernel just enqueued.
void set_last_kernel(const char* fmt, ...);

// One-time setup per (kernel, device), thread-safe: raise the kernel's dynamic shared
// memory limit to smem_max bytes and (carveout >= 0) set the preferred shared-memory
// carveout in percent; with threads > 0 also return the resident CTAs per SM for
// `threads` threads and `smem` bytes (>= 1) in *blocks_per_sm.
spdp_status kernel_setup(const void* func, int smem_max, int carveout, int threads, size_t smem, int* blocks_per_sm,
                         const char* what);
// The SM count of the current device (cached per device).
int device_sms();

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Streaming 16-bit load that does not allocate in L1 (each demand row is
// read once per tour by a given warp).
__device__ __forceinline__ uint32_t ld_stream_u16(const uint16_t* p) {
    unsigned short v;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return (uint32_t)v;
}

// ---- programmatic dependent launch (PDL) ------------------------------------
// A kernel launched with launch_pdl() may start while its stream predecessor is
// still running; pdl_wait() blocks until the predecessor grid has completed and
// its memory is visible, pdl_trigger() lets the successor start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- bulk-async copy (TMA engine, cp.async.bulk) + mbarrier helpers -------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// generic-proxy accesses of shared memory ordered before later async-proxy (bulk copy) writes
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// global -> shared bulk copy (size multiple of 16, both addresses 16-byte aligned), completion
// reported to `bar` as transaction bytes, with an L2 cache policy
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- shared-memory access by 32-bit shared address --------------------------------
__device__ __forceinline__ int lds_s32(uint32_t a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ int2 lds_s32x2(uint32_t a) {
    int2 v;
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_s32x2(uint32_t a, int x, int y) {
    asm volatile("st.shared.v2.s32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}

// ---- cp.async (LDGSTS): per-thread 16-byte global -> shared copies, L2-only (.cg) ----
// (no L2 cache-policy operand: ptxas 12.9 can place the policy descriptor in a misaligned
// uniform register pair for LDGSTS, which traps as an illegal instruction)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Warp + block reduction of the SAA partial fields.
struct Part {
    long long n_feas, n_infeas, sum, sq_lo, sq_hi;
};

__device__ __forceinline__ void part_add_cost(Part& p, long long c, bool feasible) {
    if (feasible) {
        unsigned long long sq = (unsigned long long)c * (unsigned long long)c;
        p.n_feas += 1;
        p.sum += c;
        p.sq_lo += (long long)(sq & 0xffffffffull);
        p.sq_hi += (long long)(sq >> 32);
    } else {
        p.n_infeas += 1;
    }
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ Part warp_sum(Part p) {
    p.n_feas = warp_sum_ll(p.n_feas);
    p.n_infeas = warp_sum_ll(p.n_infeas);
    p.sum = warp_sum_ll(p.sum);
    p.sq_lo = warp_sum_ll(p.sq_lo);
    p.sq_hi = warp_sum_ll(p.sq_hi);
    return p;
}

// Block-wide sum; result valid in thread 0.  smem must hold blockDim/32 Parts.
__device__ __forceinline__ Part block_sum(Part p, Part* smem) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    p = warp_sum(p);
    if (lane == 0) smem[wid] = p;
    __syncthreads();
    Part r{0, 0, 0, 0, 0};
    if (wid == 0) {
        if (lane < nw) r = smem[lane];
        r = warp_sum(r);
    }
    return r;
}

__device__ __forceinline__ void part_store(spdp_saa_partial* dst, const Part& p) {
    dst->n_feas = p.n_feas;
    dst->n_infeas = p.n_infeas;
    dst->sum = p.sum;
    dst->sumsq_lo = p.sq_lo;
    dst->sumsq_hi = p.sq_hi;
    dst->reserved = 0;
}

}  // namespace spdp
