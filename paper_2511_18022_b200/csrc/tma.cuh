// tma.cuh -- TMA (cp.async.bulk.tensor) / mbarrier helpers shared by the warp-specialised
// sweeps (split_u16.cu, f32.cu): a producer warp gathers tour-ordered demand rows into a
// shared-memory stage ring with tile::gather4, consumers wait on "full" and release "empty".
#pragma once

#include <cudaTypedefs.h>

#include "common.cuh"

namespace spdp {

// d = a * b + c on the FMA pipe (b is a runtime multiplier, so ptxas cannot turn the multiply-add
// into an IADD3 on the ALU pipe, which the candidate LOP3 / VIMNMX3 already load)
__device__ __forceinline__ uint32_t imad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// 4 rows r0..r3 x box columns starting at col of the 2-D demand tensor -> 4 consecutive boxes in
// shared memory; completion as transaction bytes on bar
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// wait for the phase with the given parity to complete, the warp suspended in the barrier unit
// meanwhile (a suspend-time hint instead of the default short limit: no spinning instructions
// steal the consumers' issue slots)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(10000000u)
        : "memory");
}
// one try of the same wait (true: the phase has completed); a warp loops on it through a vote,
// so the compiler knows the warp leaves the loop converged (no divergence checks, BRA.DIV, on the
// warp votes that follow)
__device__ __forceinline__ bool mbar_try_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(10000000u)
        : "memory");
    return ok != 0;
}
// Every lane polls the barrier itself (try_wait has acquire semantics per thread; the phase it
// waits for completes once, for all of them), then the warp reconverges.  (Polling behind a warp
// vote -- all lanes loop until all saw it -- cost the C2 sweep 5 us of 66: 7 %.)
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_sleep(bar, parity)) {
    }
    __syncwarp();
}
// Stage release through a named hardware barrier (ids 1 .. NS, one per stage): the consumer warps
// arrive without waiting (bar.arrive), the producer warp waits in bar.sync until all of them did;
// the waiting warp is parked by the barrier unit (no polling: an mbarrier wait with a suspend hint
// re-polls on every barrier event of the SM, and __nanosleep returns after a few ns -- measured
// 76 / 114 polls per chunk, 6 - 9 % of the kernel's issue slots, 33 % in the fp32 sweep).
// The consumers' last reads of the stage (LDS) completed before they arrive (their values were
// used), so the producer's TMA may overwrite it once bar.sync returns.
__device__ __forceinline__ void stage_release(int stage, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(1 + stage), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void stage_acquire(int stage, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + stage), "r"(nthreads) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// The 2-D demand tensor {S columns, n rows} (row stride ld) for the TMA gathers: boxes of
// box_cols scenarios x 1 row; out-of-range rows / columns read as zeros (split_u16.cu).
spdp_status make_demand_map(CUtensorMap* map, const uint16_t* demand, int64_t ld, int64_t S, int n, int box_cols);

}  // namespace spdp
