// micro_alu.cu -- measured peak rates of the Eq. (3) candidate idioms on this B200
// (the ALU roofline denominators).  Each kernel runs many
// independent candidate chains per thread (no memory traffic) at full occupancy
// and reports candidates/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_alu scripts/micro_alu.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

// (1) fused add-min: best = min(best + a, c)  (VIADDMNMX), one op per candidate
__global__ void k_viaddmin(int* out, int seed) {
    int b[CH], a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { b[c] = seed + c + threadIdx.x; a[c] = (seed ^ c) & 7; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) b[c] = __viaddmin_s32(b[c], a[c], b[(c + 1) % CH]);
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= b[c];
    if (s == 0x12345) out[0] = s;
}

// (2) predicated min: if (Y >= P) best = min(best, G)  (ISETP + @P VIMNMX)
__global__ void k_predmin(int* out, int seed) {
    int best[CH];
    unsigned Y[CH];
    int G[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { best[c] = 1 << 30; Y[c] = seed * c + threadIdx.x; G[c] = seed + c; }
    unsigned P = seed;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (Y[c] >= P) best[c] = min(best[c], G[c]);
            G[c] += 1;
        }
        P += 3;
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= best[c];
    if (s == 0x12345) out[0] = s;
}

// (3) plain min (VIMNMX), one op per candidate
__global__ void k_min(int* out, int seed) {
    int b[CH], a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { b[c] = seed + c + threadIdx.x; a[c] = seed ^ (c * 77); }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) { b[c] = min(b[c], a[c]); a[c] = min(a[c], b[(c + 3) % CH]); }
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= b[c] ^ a[c];
    if (s == 0x12345) out[0] = s;
}

// (4) float saturate masking: s = sat(P - Y); c = sat(G + s); best = min3(best, c0, c1)
__global__ void k_fsat(int* out, int seed) {
    float best[CH / 2], Y[CH], G[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { Y[c] = (float)(seed * c + threadIdx.x); G[c] = (float)(c) * 1e-3f; }
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) best[c] = 1.0f;
    float P = (float)seed;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) {
            const float s0 = __saturatef(P - Y[2 * c]), s1 = __saturatef(P - Y[2 * c + 1]);
            const float c0 = __saturatef(G[2 * c] + s0), c1 = __saturatef(G[2 * c + 1] + s1);
            best[c] = fminf(best[c], fminf(c0, c1));
        }
        P += 1.0f;
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) s += best[c];
    if (s == 12345.f) out[0] = (int)s;
}

// (5) float max-min masking: u = P*B + Z (FFMA); c = max(G, u); best = min3(best, c0, c1)
__global__ void k_fmaxmin(int* out, int seed) {
    float best[CH / 2], Z[CH], G[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { Z[c] = -(float)(seed * c + threadIdx.x) * 16777216.f; G[c] = (float)c; }
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) best[c] = 3e38f;
    float P = (float)seed;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) {
            const float c0 = fmaxf(G[2 * c], fmaf(P, 16777216.f, Z[2 * c]));
            const float c1 = fmaxf(G[2 * c + 1], fmaf(P, 16777216.f, Z[2 * c + 1]));
            best[c] = fminf(best[c], fminf(c0, c1));
        }
        P += 1.0f;
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) s += best[c];
    if (s == 12345.f) out[0] = (int)s;
}

// (6) integer max-min masking: c = max(PB + Z, G) (VIADDMNMX), best = min3(best, c0, c1) (VIMNMX3)
__global__ void k_imaxmin(int* out, int seed) {
    int best[CH / 2], Z[CH], G[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { Z[c] = -(seed * c + (int)threadIdx.x) << 8; G[c] = c; }
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) best[c] = 1 << 30;
    int PB = seed << 8;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) {
            const int c0 = __viaddmax_s32(PB, Z[2 * c], G[2 * c]);
            const int c1 = __viaddmax_s32(PB, Z[2 * c + 1], G[2 * c + 1]);
            best[c] = __vimin3_s32(best[c], c0, c1);
        }
        PB += 256;
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) s ^= best[c];
    if (s == 0x12345) out[0] = s;
}

// (7) HBM-free issue ceiling: FFMA chains (fma pipe)
__global__ void k_ffma(int* out, int seed) {
    float a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = (float)(seed + c);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = fmaf(a[c], 0.999f, 0.5f);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += a[c];
    if (s == 12345.f) out[0] = (int)s;
}

// (8) packed candidate idiom of split_sweep_f2_kernel: s = sat(P - Y) x2 (FADD.SAT), c = G + s (FADD2),
//     best = min3(best, c.x, c.y) (FMNMX3)
__global__ void k_f2(int* out, int seed) {
    float best[CH / 2], Y[CH];
    float2 G[CH / 2];
#pragma unroll
    for (int c = 0; c < CH; ++c) Y[c] = (float)(seed * c + threadIdx.x);
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) { best[c] = 1.0f; G[c] = make_float2(c * 1e-3f, c * 2e-3f); }
    float P = (float)seed;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) {
            const float2 s = make_float2(__saturatef(P - Y[2 * c]), __saturatef(P - Y[2 * c + 1]));
            const float2 v = __fadd2_rn(G[c], s);
            best[c] = fminf(best[c], fminf(v.x, v.y));
        }
        P += 1.0f;
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) s += best[c];
    if (s == 12345.f) out[0] = (int)s;
}

// (9) FADD2 alone (2 adds per instruction)
__global__ void k_fadd2(int* out, int seed) {
    float2 a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = make_float2((float)(seed + c), (float)(seed - c));
    const float2 b = make_float2(0.5f, 0.25f);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __fadd2_rn(a[c], b);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += a[c].x + a[c].y;
    if (s == 12345.f) out[0] = (int)s;
}

// (10) FADD.SAT alone (register operands)
__global__ void k_fsat1(int* out, int seed) {
    float a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = (float)(seed + c) * 1e-3f;
    float b = (float)seed * 1e-4f;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __saturatef(a[c] - b);
        b = b * 0.5f;
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += a[c];
    if (s == 12345.f) out[0] = (int)s;
}

template <typename K>
static double run(K kern, const char* name, double cand_per_iter_per_thread, int* d) {
    int blocks = 148 * 8, threads = 256;
    kern<<<blocks, threads>>>(d, 1);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) kern<<<blocks, threads>>>(d, r + 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double cands = (double)blocks * threads * ITERS * cand_per_iter_per_thread * reps;
    double rate = cands / (ms / 1e3);
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"rate_per_s\": %.4e}\n", name, ms / reps, rate);
    return rate;
}

int main() {
    int* d;
    cudaMalloc(&d, 16);
    run(k_viaddmin, "viaddmin (1 op/cand)", CH, d);
    run(k_min, "vimnmx (1 op/cand, 2 per iter)", 2 * CH, d);
    run(k_predmin, "isetp+@p vimnmx (+iadd)", CH, d);
    run(k_fsat, "fadd.sat x2 + fmnmx3/2 (float sat mask)", CH, d);
    run(k_fmaxmin, "ffma + fmnmx + fmnmx3/2 (float max mask)", CH, d);
    run(k_imaxmin, "viaddmax + vimnmx3/2 (int max mask)", CH, d);
    run(k_ffma, "ffma (fma pipe)", CH, d);
    run(k_f2, "fadd.sat x2 + fadd2 + fmnmx3 (packed, per cand)", CH, d);
    run(k_fadd2, "fadd2 (per instruction)", CH, d);
    run(k_fsat1, "fadd.sat (per instruction)", CH, d);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
