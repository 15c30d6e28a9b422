// gen.cu -- a1: counter-based scenario generator (DESIGN R14).
//
// One thread per scenario column; for each customer row c the thread draws
// one Philox4x32-10 block keyed by (seed) at counter (s, c, stream_tag) and
// maps it to an integer demand with integer-only arithmetic, so the host
// definition in spdp.h reproduces every value bit for bit.  Stores are
// coalesced along the scenario-minor rows.
#include "common.cuh"

namespace spdp {

struct DevModel {
    int32_t kind, n, lo_pm, hi_pm, q_cap;
    uint32_t stream_tag, key0, key1;
    int64_t A_fx, B_fx;
};

__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t a0 = 0xD2511F53u * c.x, h0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t a1 = 0xCD9E8D57u * c.z, h1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(h1 ^ c.y ^ k0, a1, h0 ^ c.w ^ k1, a0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ int64_t ih4(uint4 u) {
    return (int64_t)(u.x >> 16) + (u.y >> 16) + (u.z >> 16) + (u.w >> 16) - 131070;
}

__device__ __forceinline__ int64_t fdiv(int64_t a, int64_t b) {  // floor(a/b), b > 0
    int64_t q = a / b;
    return (a % b != 0 && a < 0) ? q - 1 : q;
}

__global__ void __launch_bounds__(256) gen_demands_kernel(DevModel m, const uint16_t* __restrict__ nominal,
                                                          int64_t s_begin, int64_t S,
                                                          uint16_t* __restrict__ demand, int64_t ld) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    const uint64_t s = (uint64_t)(s_begin + j);
    const uint32_t slo = (uint32_t)s, shi = (uint32_t)(s >> 32);
    int64_t zs = 0;
    if (m.kind == 2) zs = ih4(philox10(make_uint4(slo, shi, 0u, m.stream_tag), m.key0, m.key1));
    constexpr int64_t D = 37837LL * 65536LL;
#pragma unroll 4  // (several customers' Philox chains in flight: 0.55 -> 0.50 ms at C2; 8 measured the same)
    for (int c = 1; c <= m.n; ++c) {
        const int64_t mu = nominal[c - 1];
        int64_t q;
        if (m.kind == 0) {
            q = mu;
        } else {
            const uint4 u = philox10(make_uint4(slo, shi, (uint32_t)c, m.stream_tag), m.key0, m.key1);
            if (m.kind == 1) {
                const int64_t lo = mu * m.lo_pm / 1000;
                int64_t hi = mu * m.hi_pm / 1000;
                if (hi < lo) hi = lo;
                q = lo + (int64_t)(((uint64_t)u.x * (uint64_t)(hi - lo + 1)) >> 32);
            } else {
                q = mu + fdiv(mu * (m.A_fx * zs + m.B_fx * ih4(u)) + D / 2, D);
            }
        }
        q = q < 0 ? 0 : (q > m.q_cap ? m.q_cap : q);
        demand[(int64_t)(c - 1) * ld + j] = (uint16_t)q;
    }
}

}  // namespace spdp

using namespace spdp;

extern "C" spdp_status spdp_gen_demands(const spdp_demand_model* model, int64_t s_begin, int64_t S,
                                        uint16_t* demand, int64_t ld, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_gen_demands");
    if (!model) return fail(SPDP_E_USAGE, "spdp_gen_demands: model is NULL");
    if (model->n < 1) return fail(SPDP_E_USAGE, "spdp_gen_demands: n=%d < 1", model->n);
    if (S < 0 || s_begin < 0) return fail(SPDP_E_USAGE, "spdp_gen_demands: negative S or s_begin");
    if (ld < S) return fail(SPDP_E_USAGE, "spdp_gen_demands: ld=%lld < S=%lld", (long long)ld, (long long)S);
    if (model->kind < 0 || model->kind > 2) return fail(SPDP_E_USAGE, "spdp_gen_demands: kind=%d", model->kind);
    if (model->q_cap < 0) return fail(SPDP_E_USAGE, "spdp_gen_demands: q_cap < 0");
    if (S == 0) return SPDP_OK;
    if (!demand || !model->nominal) return fail(SPDP_E_USAGE, "spdp_gen_demands: NULL array");
    DevModel m;
    m.kind = model->kind;
    m.n = model->n;
    m.lo_pm = model->lo_pm;
    m.hi_pm = model->hi_pm;
    m.q_cap = model->q_cap > 65535 ? 65535 : model->q_cap;
    m.stream_tag = model->stream_tag;
    m.key0 = (uint32_t)(model->seed & 0xffffffffu);
    m.key1 = (uint32_t)(model->seed >> 32);
    m.A_fx = model->A_fx;
    m.B_fx = model->B_fx;
    const int threads = 256;
    const int64_t blocks = ceil_div(S, threads);
    gen_demands_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(m, model->nominal, s_begin, S,
                                                                               demand, ld);
    return last_launch("gen_demands_kernel");
}
