// Launch overhead of a persistent grid shaped like the C2 sweep (592 CTAs x 160 threads, 31 KB
// dynamic shared memory, max carveout): an empty kernel and one that only initialises mbarriers
// and syncs, timed with CUDA events back to back (median of 200) -- the floor under the sweep's
// kernel time that no change inside the kernel can remove.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__global__ void empty_k() {}
__global__ void sync_k(int* out) {
    extern __shared__ unsigned long long sm[];
    if (threadIdx.x == 0) sm[0] = 0;
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 100000) out[0] = (int)sm[0];
}
template <typename F>
float timeit_b2b(F f) {  // 200 launches back to back, per launch
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < 200; ++i) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / 200;
}
template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    std::vector<float> v;
    for (int i = 0; i < 220; ++i) {
        cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 20) v.push_back(ms);
    }
    std::sort(v.begin(), v.end());
    return v[v.size() / 2] * 1e3f;
}
int main() {
    int* d; cudaMalloc(&d, 4);
    const int smem = 31152;
    cudaFuncSetAttribute(sync_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sync_k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    printf("empty kernel <<<1, 32>>>:            %.2f us\n", timeit([&] { empty_k<<<1, 32>>>(); }));
    printf("empty kernel <<<592, 160>>>:         %.2f us\n", timeit([&] { empty_k<<<592, 160>>>(); }));
    printf("smem+sync kernel <<<592, 160, 31KB>>>: %.2f us\n", timeit([&] { sync_k<<<592, 160, smem>>>(d); }));
    printf("back to back, per launch: empty <<<592,160>>> %.2f us, smem+sync <<<592,160,31KB>>> %.2f us\n",
           timeit_b2b([&] { empty_k<<<592, 160>>>(); }), timeit_b2b([&] { sync_k<<<592, 160, smem>>>(d); }));
    return 0;
}
