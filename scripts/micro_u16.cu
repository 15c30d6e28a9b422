// micro_u16.cu -- pipe rates of the instructions the packed-u16 sweep (split_sweep_u16_kernel) is
// built from, on this B200: which pipe each one issues to (ALU vs FMA) and whether two of them
// co-issue.  Each kernel runs CH independent chains per thread at full occupancy, no memory traffic,
// and reports warp-instructions per cycle per SM (4.0 = one per scheduler per cycle).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/micro_u16 scripts/micro_u16.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

constexpr int ITERS = 4096;
constexpr int CH = 8;

__device__ __forceinline__ unsigned imad(unsigned a, unsigned b, unsigned c) {
    unsigned d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ unsigned lop3(unsigned a, unsigned b, unsigned c) {  // a | (~b & c)
    unsigned d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0xF4;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ unsigned iadd3(unsigned a, unsigned b, unsigned c) {
    unsigned d;
    asm volatile("add.u32 %0, %1, %2;\n\tadd.u32 %0, %0, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

#define KERNEL(name, INIT, BODY, FIN)                                    \
    __global__ void name(unsigned* out, unsigned m1, unsigned seed) {     \
        unsigned x[CH], y[CH];                                           \
        float f[CH];                                                     \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) {                 \
            x[c] = seed * (c + 1) + threadIdx.x;                         \
            y[c] = seed ^ (c * 0x9E3779B9u);                             \
            f[c] = (float)c;                                             \
        }                                                                \
        INIT;                                                            \
        for (int i = 0; i < ITERS; ++i) {                                \
            _Pragma("unroll") for (int c = 0; c < CH; ++c) { BODY; }     \
        }                                                                \
        unsigned s = 0;                                                  \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) s ^= x[c] ^ __float_as_uint(f[c]); \
        FIN;                                                             \
        if (s == 0x12345u) out[0] = s;                                   \
    }

KERNEL(k_imad, , x[c] = imad(x[c], m1, y[c]), )
KERNEL(k_lop3, , x[c] = lop3(x[c], y[c], 0x80008000u), )
KERNEL(k_iadd3, , x[c] = iadd3(x[c], y[c], m1), )
KERNEL(k_vmin3, , x[c] = __vimin3_u16x2(x[c], y[c], y[(c + 1) % CH]), )
KERNEL(k_vadd2, , x[c] = __vadd2(x[c], y[c]), )
KERNEL(k_vaddmin, , x[c] = __viaddmin_u16x2(x[c], y[c], y[(c + 3) % CH]), )
KERNEL(k_vmnmx, , { x[c] = __vminu2(x[c], y[c]); y[c] = __vmaxu2(y[c], x[(c + 3) % CH]); }, )
KERNEL(k_hmin2, , { __half2 a = *reinterpret_cast<__half2*>(&x[c]); __half2 b = *reinterpret_cast<__half2*>(&y[c]);
                    a = __hmin2(a, b); b = __hmax2(b, a); x[c] = *reinterpret_cast<unsigned*>(&a);
                    y[c] = *reinterpret_cast<unsigned*>(&b); }, )
KERNEL(k_imad_lop3, , { x[c] = imad(x[c], m1, y[c]); y[c] = lop3(y[c], x[(c + 4) % CH], 0x80008000u); }, )
KERNEL(k_lop3_ffma, , { x[c] = lop3(x[c], y[c], 0x80008000u); f[c] = fmaf(f[c], 0.999f, f[(c + 1) % CH]); }, )
KERNEL(k_imad_ffma, , { x[c] = imad(x[c], m1, y[c]); f[c] = fmaf(f[c], 0.999f, f[(c + 1) % CH]); }, )
KERNEL(k_hmin2_lop3, , { __half2 a = *reinterpret_cast<__half2*>(&x[c]); __half2 b = *reinterpret_cast<__half2*>(&y[c]);
                    a = __hmax2(a, b); x[c] = *reinterpret_cast<unsigned*>(&a); y[c] = lop3(y[c], x[(c + 4) % CH], 0x80008000u); }, )
KERNEL(k_hmin2_imad, , { __half2 a = *reinterpret_cast<__half2*>(&x[c]); __half2 b = *reinterpret_cast<__half2*>(&y[c]);
                    a = __hmax2(a, b); x[c] = *reinterpret_cast<unsigned*>(&a); y[c] = imad(y[c], m1, x[(c + 4) % CH]); }, )
KERNEL(k_vmin3_lop3, , { x[c] = __vimin3_u16x2(x[c], y[c], y[(c + 1) % CH]); y[c] = lop3(y[c], x[(c + 5) % CH], 0x80008000u); }, )
KERNEL(k_vmin3_imad, , { x[c] = __vimin3_u16x2(x[c], y[c], y[(c + 1) % CH]); y[c] = imad(y[c], m1, x[(c + 5) % CH]); }, )
// the candidate idiom of the packed-u16 sweep, per candidate PAIR of one scenario pair:
// d = Yg - P (IMAD), key = G | (~d & 0x80008000) (LOP3), best = min3(best, key0, key1) (VIMNMX3.U16x2)
__global__ void k_cand(unsigned* out, unsigned m1, unsigned seed) {
    unsigned Yg[CH], G[CH], best[CH / 2];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        Yg[c] = seed * (c + 1) + threadIdx.x;
        G[c] = seed ^ (c * 0x9E3779B9u);
    }
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) best[c] = 0xffffffffu;
    unsigned P = seed;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) {
            const unsigned d0 = imad(P, m1, Yg[2 * c]);
            const unsigned d1 = imad(P, m1, Yg[2 * c + 1]);
            best[c] = __vimin3_u16x2(best[c], lop3(G[2 * c], d0, 0x80008000u), lop3(G[2 * c + 1], d1, 0x80008000u));
        }
        P += 0x00010001u;
    }
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) s ^= best[c];
    if (s == 0x12345u) out[0] = s;
}


// warp vote + uniform branch (the deep-group guard of the sweep): VOTE.ANY + BRA per iteration,
// with 6 independent ALU ops between votes
__global__ void k_vote(unsigned* out, unsigned m1, unsigned seed) {
    unsigned x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = seed * (c + 1) + threadIdx.x;
    unsigned acc = 0;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = lop3(x[c], x[(c + 1) % CH], 0x80008000u);
        if (__any_sync(0xffffffffu, (x[0] & 0x40000000u) != 0u)) acc += x[1];  // rarely true
    }
    unsigned s = acc;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= x[c];
    if (s == 0x12345u) out[0] = s;
}
// the same loop without the vote (branch on a lane-uniform kernel argument)
__global__ void k_novote(unsigned* out, unsigned m1, unsigned seed) {
    unsigned x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = seed * (c + 1) + threadIdx.x;
    unsigned acc = 0;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = lop3(x[c], x[(c + 1) % CH], 0x80008000u);
        if (m1 == 7u) acc += x[1];
    }
    unsigned s = acc;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= x[c];
    if (s == 0x12345u) out[0] = s;
}


// candidate idiom variants (per pair of candidates of one scenario pair):
//  (b) 2 IMAD + 2 LOP3 + 2 VIMNMX.U16x2 (2-input folds)
__global__ void k_cand2(unsigned* out, unsigned m1, unsigned seed) {
    unsigned Yg[CH], G[CH], best[CH / 2];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        Yg[c] = seed * (c + 1) + threadIdx.x;
        G[c] = seed ^ (c * 0x9E3779B9u);
    }
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) best[c] = 0xffffffffu;
    unsigned P = seed;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) {
            const unsigned d0 = imad(P, m1, Yg[2 * c]);
            const unsigned d1 = imad(P, m1, Yg[2 * c + 1]);
            best[c] = __vminu2(__vminu2(best[c], lop3(G[2 * c], d0, 0x80008000u)), lop3(G[2 * c + 1], d1, 0x80008000u));
        }
        P += 0x00010001u;
    }
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) s ^= best[c];
    if (s == 0x12345u) out[0] = s;
}
//  (c) tree fold: 6 keys -> min3(min3(k0,k1,k2), min3(k3,k4,k5)) + accumulate: 6 IMAD + 6 LOP3 + 3 VIMNMX3
__global__ void k_cand3(unsigned* out, unsigned m1, unsigned seed) {
    unsigned Yg[6], G[6], best = 0xffffffffu;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
        Yg[c] = seed * (c + 1) + threadIdx.x;
        G[c] = seed ^ (c * 0x9E3779B9u);
    }
    unsigned P = seed;
    for (int i = 0; i < ITERS; ++i) {
        unsigned k[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) k[c] = lop3(G[c], imad(P, m1, Yg[c]), 0x80008000u);
        best = __vimin3_u16x2(best, __vimin3_u16x2(k[0], k[1], k[2]), __vimin3_u16x2(k[3], k[4], k[5]));
        P += 0x00010001u;
    }
    if (best == 0x12345u) out[0] = best;
}

template <typename K>
static void run(K kern, const char* name, double instr_per_iter_per_thread, unsigned* d, double clk_ghz) {
    const int blocks = 148 * 8, threads = 256;
    kern<<<blocks, threads>>>(d, 0xffffffffu, 1u);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) kern<<<blocks, threads>>>(d, 0xffffffffu, (unsigned)r + 2u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_instr = (double)blocks * threads / 32.0 * ITERS * instr_per_iter_per_thread * reps;
    const double per_clk_sm = warp_instr / (ms * 1e-3) / 148.0 / (clk_ghz * 1e9);
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"warp_instr_per_clk_per_sm\": %.3f}\n", name, ms / reps, per_clk_sm);
}

int main() {
    unsigned* d;
    cudaMalloc(&d, 16);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ghz = khz / 1e6;
    printf("{\"clock_ghz_nominal\": %.3f}\n", ghz);
    run(k_imad, "IMAD (mad.lo.u32, reg multiplier)", CH, d, ghz);
    run(k_lop3, "LOP3", CH, d, ghz);
    run(k_iadd3, "IADD3", CH, d, ghz);
    run(k_vmin3, "VIMNMX3.U16x2", CH, d, ghz);
    run(k_vadd2, "VIADD.16x2", CH, d, ghz);
    run(k_vaddmin, "VIADDMNMX.U16x2", CH, d, ghz);
    run(k_vmnmx, "VIMNMX.U16x2 (min/max alternating)", 2 * CH, d, ghz);
    run(k_hmin2, "HMNMX2 (min/max alternating)", 2 * CH, d, ghz);
    run(k_imad_lop3, "IMAD + LOP3 interleaved (per instr)", 2 * CH, d, ghz);
    run(k_lop3_ffma, "LOP3 + FFMA interleaved (per instr)", 2 * CH, d, ghz);
    run(k_imad_ffma, "IMAD + FFMA interleaved (per instr)", 2 * CH, d, ghz);
    run(k_hmin2_lop3, "HMNMX2 + LOP3 interleaved (per instr)", 2 * CH, d, ghz);
    run(k_hmin2_imad, "HMNMX2 + IMAD interleaved (per instr)", 2 * CH, d, ghz);
    run(k_vmin3_lop3, "VIMNMX3.U16x2 + LOP3 interleaved (per instr)", 2 * CH, d, ghz);
    run(k_vmin3_imad, "VIMNMX3.U16x2 + IMAD interleaved (per instr)", 2 * CH, d, ghz);
    run(k_cand, "candidate pair idiom: IMAD+LOP3 x2 + VIMNMX3 (per instr)", 5.0 * CH / 2 + 1.0, d, ghz);
    run(k_cand2, "candidate pair: IMAD+LOP3 x2 + 2 VIMNMX.U16x2 (per instr)", 6.0 * CH / 2 + 1.0, d, ghz);
    run(k_cand3, "6 candidates: 6 IMAD + 6 LOP3 + 3 VIMNMX3 tree (per instr)", 16.0, d, ghz);
    run(k_vote, "8 LOP3 + VOTE.ANY + BRA per iteration (per LOP3)", CH, d, ghz);
    run(k_novote, "8 LOP3 + uniform BRA per iteration (per LOP3)", CH, d, ghz);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
