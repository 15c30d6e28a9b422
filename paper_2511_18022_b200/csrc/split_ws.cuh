// split_ws.cuh -- the split workspace layout and the host-side launchers of
// split.cu that other translation units (nbr.cu, limits.cu) reuse.
#pragma once

#include "common.cuh"

namespace spdp {

// ---------------------------------------------------------------- workspace
// Per-tour info for the fp32 sweep: g0f = (g(0) + OFF) / 2^24 (float bits),
// off = OFF = D[n] (makes every g(p) + OFF >= 0), ok = every value the fp32
// sweep forms is an integer (times 2^-24) below 2^24, hence exact.
// The packed-u16 sweep (split_u16.cu) keeps g relative to a per-scenario base in 15 bits:
// ns16 = NS = sum of max(0, -Cg) over the tour's layers (the most the window minimum can ever
// fall, DESIGN §6 "packed-u16"), thr16 = 0x7FFF - (largest sum of max(0, Cg) over kU16Check
// consecutive layers): a value at or below thr16 at a range check stays below 2^15 until the
// next check; ok16 = every value the sweep forms fits (NS + max Cg + that sum <= 0x7FFF).
// bn = B[n] = D[n] + c_{s_n,0} (added in int32 at the end).
struct TourInfo {
    int32_t g0f_bits, off, ok, ns16, thr16, ok16, bn, pad;
};

// Range-check interval of the packed-u16 sweep (layers); tour_prep_kernel's thr16 assumes it.
constexpr int kU16Check = 12;

constexpr int kTabPad = 64;       // padding rows after each tour table
constexpr int kSlots = 32;  // SAA partial slots per tour (spread the sweep's atomics)

// Cg planes: per tour [kCgPlanes][cg_stride(n)] int32 (plane 0 int Cg, plane 1 fp32 Cg / 2^24 bits,
// plane 2 the packed-u16 pair Cg * 0x10001 (0 at layer n and in the padding)), zero padded;
// the stride keeps every chunk's W-entry slice 16-byte aligned for the bulk copies.
__host__ __device__ inline int cg_stride(int n) { return (n + kTabPad + 7) & ~7; }
constexpr int kCgPlanes = 3;

// Demand row of every tour position for the TMA sweep (split_u16.cu): per tour trow_stride(n)
// int32 entries, row of sigma_{i+1} at i < n, then n (a row outside the demand tensor: reads as
// zeros); 16-byte aligned rows of the table, so a producer reads 4 positions per load.
__host__ __device__ inline int trow_stride(int n) { return (n + kTabPad + 3) & ~3; }

struct WsLayout {
    size_t hdr, g0, tinfo, tabs, rowp, cgs, trow, slots, ovf, total;
};

inline WsLayout ws_layout(int32_t n, int64_t S, int32_t T) {
    WsLayout L;
    size_t off = 0;
    L.hdr = off; off += 256;
    L.g0 = off; off = align_up(off + sizeof(int32_t) * (size_t)T, 256);
    L.tinfo = off; off = align_up(off + sizeof(TourInfo) * (size_t)T, 256);
    L.tabs = off; off = align_up(off + sizeof(int2) * (size_t)T * (size_t)(n + kTabPad), 256);
    L.rowp = off; off = align_up(off + sizeof(uint64_t) * (size_t)T * (size_t)(n + kTabPad), 256);
    L.cgs = off; off = align_up(off + sizeof(int32_t) * kCgPlanes * (size_t)T * (size_t)cg_stride(n), 256);
    L.trow = off; off = align_up(off + sizeof(int32_t) * (size_t)T * (size_t)trow_stride(n), 256);
    L.slots = off; off = align_up(off + sizeof(spdp_saa_partial) * (size_t)T * (size_t)kSlots, 256);
    L.ovf = off; off = align_up(off + sizeof(unsigned long long) * (size_t)T * (size_t)S, 256);
    L.total = off;
    return L;
}

// header words
enum { HDR_OVF_COUNT = 0, HDR_STATUS = 1, HDR_SAMPLE_W = 2, HDR_TILE = 3, HDR_SAMPLE_SUM = 4 /* u64 */, HDR_SAMPLE_CNT = 6 };
enum { ST_NOT_PERM = 1, ST_NEG_DIST = 2, ST_RANGE = 4 };

// Claim order of a tour's scenario blocks (longest first): spdp_order_scenarios sorts each segment of
// kOrderSeg scenarios by increasing total demand, i.e. decreasing window length and tile time, so
// block-claim k takes position p = k / nseg of segment k % nseg: every segment's slowest tiles are
// claimed first and the persistent schedule ends on the fastest (a ragged last segment of r tiles
// takes part in the first r positions).  A permutation of 0 .. nb - 1 for any nb; on an unordered
// set it only changes which CTA takes which tile.
constexpr uint32_t kOrderSeg = 65536;  // = order.cu kOrdSeg (tile must divide it)
__device__ __forceinline__ uint32_t lpt_block(uint32_t k, uint32_t nb, int tile) {
    const uint32_t per = kOrderSeg / (uint32_t)tile;   // tiles per segment
    const uint32_t full = nb / per, rem = nb % per;     // full segments, tiles of the ragged last one
    const uint32_t nseg = full + (rem != 0u);
    if (k < rem * nseg) return (k % nseg) * per + k / nseg;
    if (full == 0u) return k;
    const uint32_t k2 = k - rem * nseg;
    return (k2 % full) * per + rem + k2 / full;
}

// Arguments of the sweep launchers (split.cu, split_u16.cu).
struct SweepArgs {
    const int32_t* tours;  // [T][n] (the u16 sweep reads its first tile's rows from it before the PDL wait)
    const uint16_t* const* rowp;
    const int2* tabs;
    const int32_t* trows;
    const int32_t* cgs;
    const int32_t* g0;
    const TourInfo* tinfo;
    int n, T;
    const uint16_t* demand;
    int64_t ld, S;
    uint32_t Q;
    int32_t* cost;
    spdp_saa_partial* slots;
    unsigned long long* ovf;
    unsigned* hdr;
};

// split_u16.cu: the packed-u16 sweep (two scenarios per lane).  u16_loads_ok(): its load
// range check (host side); launch_sweep_u16: W in {16, 20, 24, 32}, mean_w picks the grouping.
bool u16_loads_ok(int n, uint32_t Q);
spdp_status launch_sweep_u16(int W, int mean_w, cudaStream_t st, const SweepArgs& a);
spdp_status debug_timeline(void* p);  // spdp_debug_timeline

// Host launchers (split.cu).
// tour_prep_kernel over T tours into the workspace (tables, g0, row pointers, Cg
// planes; zeroes the SAA slots (if zero_slots), partial[0..T) (if non-NULL) and
// the overflow counter).
spdp_status launch_tour_prep(const int32_t* tours, int32_t T, int32_t n, const int32_t* dist,
                             const uint16_t* demand, int64_t ld, char* ws, const WsLayout& L,
                             spdp_saa_partial* partial, bool zero_slots, bool validate, cudaStream_t st);
// split_finish_kernel: SAA slots -> partial, then the overflow list (full
// recomputation of every listed (tour, scenario) pair from the tour tables).
spdp_status launch_finish(char* ws, const WsLayout& L, int32_t T, int32_t n, const uint16_t* demand, int64_t ld,
                          int64_t S, uint32_t Qe, int32_t* cost, spdp_saa_partial* partial, bool pdl,
                          cudaStream_t st);

// Position tables of nbr.cu / limits.cu: n + 1 entries per tour plus kTourTabPad padding entries
// (row offset 0: a valid demand row) so prefetches past position n need no bounds check.
constexpr int kTourTabPad = 8;
__host__ __device__ inline int tour_tab_stride(int n) { return n + 1 + kTourTabPad; }

// nbr.cu: per-tour position tables e[t][i] = {row of sigma_i, A[i], B[i], row * ld (uint32)},
// i = 0..n, for T tours [T][n]; with parent != NULL also info[t] = {common prefix length,
// n - common suffix length} against the parent.  One warp per tour.
spdp_status launch_tour_table(const int32_t* tours, int32_t T, const int32_t* parent, int32_t n, const int32_t* dist,
                              int64_t ld, int4* etabs, int4* info, cudaStream_t st);

}  // namespace spdp
