// api.cu -- error plumbing, SAA finalize (host) and the host-buffer
// end-to-end entry of libspdp.
#include <cmath>
#include <cstdarg>
#include <cstdio>

#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "split_ws.cuh"

namespace spdp {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

spdp_status fail(spdp_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

spdp_status cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return SPDP_OK;
    return fail(SPDP_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

spdp_status last_launch(const char* what) { return cuda_check(cudaGetLastError(), what); }

static thread_local char g_kernel[128] = "";

void set_last_kernel(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_kernel, sizeof(g_kernel), fmt, ap);
    va_end(ap);
}

static thread_local cudaEvent_t g_prof_start = nullptr, g_prof_stop = nullptr;

void prof_begin(cudaStream_t st) {
    if (g_prof_start && g_prof_stop) cudaEventRecord(g_prof_start, st);
}

void prof_end(cudaStream_t st) {
    if (g_prof_start && g_prof_stop) cudaEventRecord(g_prof_stop, st);
}

}  // namespace spdp

using namespace spdp;

static std::mutex g_setup_mu;
static std::map<std::tuple<const void*, int, int, int, int, size_t>, int> g_setup;  // (func, dev, smem_max, carveout, threads, smem)
static std::map<int, int> g_sms;

spdp_status spdp::kernel_setup(const void* func, int smem_max, int carveout, int threads, size_t smem, int* blocks_per_sm,
                         const char* what) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_check(e, what);
    const auto key = std::make_tuple(func, dev, smem_max, carveout, threads, smem);
    std::lock_guard<std::mutex> lock(g_setup_mu);
    auto it = g_setup.find(key);
    if (it != g_setup.end()) {
        if (blocks_per_sm) *blocks_per_sm = it->second;
        return SPDP_OK;
    }
    if (smem_max > 0) {
        e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
        if (e != cudaSuccess) return cuda_check(e, what);
    }
    if (carveout >= 0) {
        e = cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
        if (e != cudaSuccess) return cuda_check(e, what);
    }
    int b = 1;
    if (threads > 0) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, func, threads, smem);
        if (e != cudaSuccess) return cuda_check(e, what);
        if (b < 1) b = 1;
    }
    g_setup[key] = b;
    if (blocks_per_sm) *blocks_per_sm = b;
    return SPDP_OK;
}

int spdp::device_sms() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lock(g_setup_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = v;
    return v;
}

extern "C" int spdp_version(void) { return 100; }  // 0.1.0

extern "C" void spdp_set_profile_events(void* start_event, void* stop_event) {
    g_prof_start = static_cast<cudaEvent_t>(start_event);
    g_prof_stop = static_cast<cudaEvent_t>(stop_event);
}

extern "C" const char* spdp_last_error(void) { return g_err; }

extern "C" const char* spdp_last_kernel(void) { return g_kernel; }

extern "C" spdp_status spdp_debug_timeline(void* buffer) { return spdp::debug_timeline(buffer); }

// a6 finalize.  Exact integer moments, one rounding
// per reported statistic: mean = sum / m, var = (m sumsq - sum^2) / (m (m-1)).
extern "C" spdp_status spdp_saa_mean(const spdp_saa_partial* p, spdp_saa_estimate* out) {
    NvtxScope nvtx_("spdp_saa_mean");
    if (!p || !out) return fail(SPDP_E_USAGE, "spdp_saa_mean: NULL pointer");
    if (p->n_feas < 0 || p->n_infeas < 0) return fail(SPDP_E_USAGE, "spdp_saa_mean: negative counts");
    out->m = p->n_feas;
    out->infeasible = p->n_infeas;
    if (p->n_feas == 0) {
        out->mean = out->var = out->std_err = out->ci95_lo = out->ci95_hi = NAN;
        return fail(SPDP_E_DATA, "spdp_saa_mean: all scenarios infeasible (SPEC:287)");
    }
    const __int128 m = p->n_feas;
    const __int128 sum = p->sum;
    const __int128 sq = ((__int128)p->sumsq_hi << 32) + (__int128)p->sumsq_lo;
    out->mean = (double)p->sum / (double)p->n_feas;
    if (p->n_feas >= 2) {
        const __int128 num = m * sq - sum * sum;
        out->var = (double)num / ((double)p->n_feas * (double)(p->n_feas - 1));
    } else {
        out->var = 0.0;
    }
    out->std_err = std::sqrt(out->var / (double)p->n_feas);
    out->ci95_lo = out->mean - 1.96 * out->std_err;
    out->ci95_hi = out->mean + 1.96 * out->std_err;
    return SPDP_OK;
}

// ---------------------------------------------------------------- host-buffer e2e
namespace {
struct HostWs {
    size_t tour, dist, demand, cost, partial, split, total;
    int64_t ldd;
};
HostWs host_ws(int32_t n, int64_t S) {
    HostWs h;
    size_t off = 0;
    h.ldd = (S + 7) / 8 * 8;
    h.tour = off; off = align_up(off + sizeof(int32_t) * (size_t)n, 256);
    h.dist = off; off = align_up(off + sizeof(int32_t) * (size_t)(n + 1) * (size_t)(n + 1), 256);
    h.demand = off; off = align_up(off + sizeof(uint16_t) * (size_t)n * (size_t)h.ldd, 256);
    h.cost = off; off = align_up(off + sizeof(int32_t) * (size_t)S, 256);
    h.partial = off; off = align_up(off + sizeof(spdp_saa_partial), 256);
    h.split = off; off += spdp_workspace_bytes(n, S, 1);
    h.total = off;
    return h;
}
}  // namespace

extern "C" size_t spdp_host_workspace_bytes(int32_t n, int64_t S) {
    if (n < 1 || S < 1) return 0;
    return host_ws(n, S).total;
}

extern "C" spdp_status spdp_split_eval_host(const int32_t* tour_h, const int32_t* dist_h, int32_t n,
                                            const uint16_t* demand_h, int64_t ld_h, int64_t S, int32_t Q,
                                            int32_t* cost_h, spdp_saa_estimate* est_h, int32_t window_hint, void* ws,
                                            size_t ws_bytes, spdp_stream_t stream) {
    NvtxScope nvtx_("spdp_split_eval_host");
    if (n < 1 || S < 1) return fail(SPDP_E_USAGE, "spdp_split_eval_host: n and S must be >= 1");
    if (!tour_h || !dist_h || !demand_h || !est_h || !ws) return fail(SPDP_E_USAGE, "spdp_split_eval_host: NULL pointer");
    if (ld_h < S) return fail(SPDP_E_USAGE, "spdp_split_eval_host: ld_h < S");
    const HostWs h = host_ws(n, S);
    if (ws_bytes < h.total) return fail(SPDP_E_USAGE, "spdp_split_eval_host: workspace %zu < %zu", ws_bytes, h.total);
    cudaStream_t st = (cudaStream_t)stream;
    char* w = static_cast<char*>(ws);
    int32_t* tour = reinterpret_cast<int32_t*>(w + h.tour);
    int32_t* dist = reinterpret_cast<int32_t*>(w + h.dist);
    uint16_t* demand = reinterpret_cast<uint16_t*>(w + h.demand);
    int32_t* cost = reinterpret_cast<int32_t*>(w + h.cost);
    spdp_saa_partial* partial = reinterpret_cast<spdp_saa_partial*>(w + h.partial);
    spdp_status rc;
    if ((rc = cuda_check(cudaMemcpyAsync(tour, tour_h, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st), "H2D tour"))) return rc;
    if ((rc = cuda_check(cudaMemcpyAsync(dist, dist_h, sizeof(int32_t) * (size_t)(n + 1) * (n + 1), cudaMemcpyHostToDevice, st),
                         "H2D dist")))
        return rc;
    if (ld_h == h.ldd) {
        rc = cuda_check(cudaMemcpyAsync(demand, demand_h, sizeof(uint16_t) * (size_t)n * (size_t)ld_h, cudaMemcpyHostToDevice, st),
                        "H2D demand");
    } else {
        rc = cuda_check(cudaMemcpy2DAsync(demand, sizeof(uint16_t) * (size_t)h.ldd, demand_h, sizeof(uint16_t) * (size_t)ld_h,
                                          sizeof(uint16_t) * (size_t)S, (size_t)n, cudaMemcpyHostToDevice, st),
                        "H2D demand (2D)");
    }
    if (rc) return rc;
    rc = spdp_split_eval(tour, dist, n, demand, h.ldd, S, Q, cost_h ? cost : nullptr, partial, window_hint, w + h.split,
                         ws_bytes - h.split, 0u, stream);
    if (rc) return rc;
    spdp_saa_partial p;
    if ((rc = cuda_check(cudaMemcpyAsync(&p, partial, sizeof(p), cudaMemcpyDeviceToHost, st), "D2H partial"))) return rc;
    if (cost_h && (rc = cuda_check(cudaMemcpyAsync(cost_h, cost, sizeof(int32_t) * (size_t)S, cudaMemcpyDeviceToHost, st), "D2H cost")))
        return rc;
    if ((rc = cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
    return spdp_saa_mean(&p, est_h);
}
