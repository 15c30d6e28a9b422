/*
 * spdp.h -- C-ABI of the B200-native scenario-parallel Split DP library
 * (libspdp.so), the hot path of arXiv 2511.18022:
 *   second-stage evaluation of a first-stage giant tour over up to millions of
 *   demand scenarios (§2), by the masked Split DP of Eq. (1)-(3)
 *   (§3), reduced to the sample-average-approximation (SAA)
 *   statistics of the expected recourse cost.
 *
 * Citations: PAPER:n = line n of the paper text; SPEC:n = line n of the
 * companion spec; SURVEY §x = /root/repo/SURVEY.md; DESIGN Rk = reading k in
 * DESIGN.md.
 *
 * Conventions (all entry points)
 *  - Plain C types only.  Array arguments are caller-owned DEVICE pointers
 *    unless the name ends in _h (host pointer).  The library never allocates
 *    or frees caller memory; scratch comes from the caller's workspace `ws`
 *    (size from spdp_workspace_bytes), which must not be used concurrently by
 *    two calls.
 *  - All device work is enqueued asynchronously on `stream` (a cudaStream_t;
 *    NULL = legacy default stream).  Exceptions: spdp_saa_mean (host only),
 *    spdp_split_eval_host (synchronizes `stream` before returning) and any
 *    call with SPDP_F_VALIDATE (synchronizes to read back the check).
 *  - Return value: SPDP_OK, or an error code; spdp_last_error() then returns a
 *    thread-local message.  Usage errors are detected on the host before
 *    anything is enqueued.
 *  - Index conventions: customers are 1..n, node 0 is the depot, node n+1 (the
 *    return depot) is node 0 (DESIGN R6).  A tour is a permutation
 *    sigma_1..sigma_n of 1..n (int32 [n]).  dist is int32 [(n+1)*(n+1)]
 *    row-major, dist[a*(n+1)+b] = c_{a,b} >= 0.
 *  - Demand matrix: uint16 [n][ld], row c-1 holds customer c, column j holds
 *    scenario j (scenario-minor so a warp's loads are coalesced, PAPER:151;
 *    DESIGN R19).  ld >= S, ld % 8 == 0, pointer 16-byte aligned.  The DP
 *    reads q^omega_{sigma_k} = demand[(sigma_k - 1)*ld + j] (tour order,
 *    PAPER:92; DESIGN R1).
 *  - Costs are exact integers (int32); an infeasible scenario (some single
 *    demand > Q, so Eq. (2)'s set is empty, DESIGN R4) gets SPDP_INFEASIBLE.
 *    Results are bit-identical for every launch configuration and shard
 *    count.
 */
#ifndef SPDP_H
#define SPDP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SPDP_API __attribute__((visibility("default")))
#else
#define SPDP_API
#endif

typedef struct CUstream_st* spdp_stream_t; /* == cudaStream_t */

typedef enum {
    SPDP_OK = 0,
    SPDP_E_USAGE = 2,    /* bad argument (null pointer, size, alignment, workspace too small) */
    SPDP_E_DATA = 3,     /* bad data: tour not a permutation, negative/oversized costs,
                            SAA over zero feasible scenarios */
    SPDP_E_RESOURCE = 4, /* problem too large for the kernels (e.g. n > SPDP_MAX_N) */
    SPDP_E_CUDA = 5      /* CUDA launch / runtime error */
} spdp_status;

#define SPDP_INFEASIBLE INT32_MAX   /* cost sentinel */
#define SPDP_MAX_N 16384            /* largest tour length the sweep kernels accept */

/* flags */
#define SPDP_F_VALIDATE 1u          /* check tour permutation, dist >= 0 and the int32 range
                                       bound on the device; synchronizes; E_DATA on failure */
/* sweep algorithm (spdp_split_eval / _batch); all give bit-identical results.
 * Default (none set): the packed-u16 register ring for windows <= 32 when its load check passes
 * (else the packed-fp32 or int ring), the deque for wider windows. */
#define SPDP_F_SWEEP_INT   2u       /* register ring, exact int32, predicated min per candidate */
#define SPDP_F_SWEEP_F32   4u       /* register ring, exact integer-valued fp32, FMA-pipe masking */
#define SPDP_F_SWEEP_DEQUE 8u       /* monotone-deque sliding-window minimum, O(1) amortised */
#define SPDP_F_SWEEP_U16 128u       /* register ring, two scenarios per lane in packed u16 halves
                                       (windows 9..32, 14 (Q + 1) <= 2^15; else as the default) */
#define SPDP_F_SCRATCH_GLOBAL 16u  /* spdp_split_eval_limits: every scenario through the general kernel
                                       with its DP arrays in the workspace (same results; tests both paths) */
#define SPDP_F_NBR_SMEM 32u        /* spdp_split_eval_neighbours: the shared-memory-ring kernel instead of
                                       the register ring (same results) */
#define SPDP_F_NBR_AUTO 64u        /* spdp_split_eval_neighbours(_multi): read the candidates' changed spans
                                       back (synchronizes) and run spdp_split_eval_batch instead when they
                                       average more than 40 % of the tour (the measured crossover) */
#define SPDP_F_IRP_EAGER 65536u    /* spdp_irp_dp: the eager-shift lane kernel instead of the lazily shifted
                                       value functions (same results) */
#define SPDP_F_IRP_STATES 131072u  /* spdp_irp_dp: the state-parallel kernel (lanes = inventory states, the
                                       delivery band a warp prefix-min scan; the general kernel for
                                       0 < X < U) for every band shape (same results) */
/* bits 8..15 of flags: the expected MEAN window width i - mask(i) (0 = unknown; with
 * window_hint = 0 it is sampled).  A tuning hint like window_hint: it picks how many
 * candidates the sweep evaluates before its first warp vote, never the result. */
#define SPDP_F_MEAN_WINDOW_SHIFT 8
#define SPDP_F_MEAN_WINDOW(w) ((uint32_t)((w) < 255 ? (w) : 255) << SPDP_F_MEAN_WINDOW_SHIFT)

/* Summable SAA partial.  Every field is an int64 that adds
 * elementwise, so partials of disjoint scenario sets combine by a plain SUM
 * (e.g. an NCCL all-reduce over ranks) and the result is exact and
 * independent of the summation order.  sum = sum of feasible costs;
 * sum of squares = sumsq_hi * 2^32 + sumsq_lo where sumsq_lo / sumsq_hi are
 * the sums of the low / high 32-bit halves of each cost^2.  48 bytes. */
typedef struct {
    int64_t n_feas, n_infeas, sum, sumsq_lo, sumsq_hi, reserved;
} spdp_saa_partial;

/* SAA estimate (PAPER:264 z_m): mean and unbiased variance of
 * the feasible scenario costs, std_err = sqrt(var/m), ci95 = mean -+ 1.96 std_err. */
typedef struct {
    int64_t m, infeasible;
    double mean, var, std_err, ci95_lo, ci95_hi;
} spdp_saa_estimate;

/* Counter-based demand model (DESIGN R14).  For global
 * scenario s and customer c (1..n), u = Philox4x32-10(ctr = (lo32 s, hi32 s,
 * c, stream_tag), key = (lo32 seed, hi32 seed)):
 *   kind 0 fixed:       q = mu_c
 *   kind 1 uniform-int: q = lo + ((u0 * (hi - lo + 1)) >> 32), lo = mu*lo_pm/1000, hi = mu*hi_pm/1000
 *   kind 2 correlated:  q = mu + floor((mu*(A_fx*z_s + B_fx*z_sc) + D/2) / D), D = 37837*2^16,
 *                       z = sum_j (u_j >> 16) - 131070 (Irwin-Hall(4)); z_s uses counter c = 0
 * then q = clamp(q, 0, q_cap).  `nominal` is a DEVICE pointer [n]. */
typedef struct {
    int32_t kind;
    int32_t n;
    const uint16_t* nominal;
    int32_t lo_pm, hi_pm;
    int64_t A_fx, B_fx;
    int32_t q_cap;
    uint32_t stream_tag;
    uint64_t seed;
} spdp_demand_model;

/* IRP customer parameters (DESIGN R21): capacity U, max
 * delivery X per visit, initial inventory I0, holding h, lost-sale b and
 * per-unit delivery c costs; all >= 0 and I0 <= U. */
typedef struct {
    int32_t U, X, I0, h, b, c;
} spdp_irp_customer;

/* Library version (major*10000 + minor*100 + patch). */
SPDP_API int spdp_version(void);

/* Thread-local message for the last non-OK status of this thread. */
SPDP_API const char* spdp_last_error(void);

/* Measurement hook (bench.py): when both are non-NULL, every subsequent
 * spdp_split_eval / _batch / _penalized / _neighbours / _limits, spdp_split_values
 * or spdp_irp_dp call made by THIS thread records `start_event` immediately
 * before and `stop_event` immediately after its dominant kernel(s) (the sweep /
 * neighbour / limits / values / IRP kernels), on the call's stream.  Both are cudaEvent_t.  Pass NULL, NULL to clear.  Thread-local. */
SPDP_API void spdp_set_profile_events(void* start_event, void* stop_event);

/* Name of the dominant kernel (variant and ring width) that the last split call
 * on this thread enqueued, e.g. "split_sweep_f2_kernel<20,3,1,0,20,0>" or
 * "split_nbr_kernel<16,1>"; "" before the first call.  Thread-local,
 * owned by the library, valid until the next call on this thread.  For
 * reports (bench.py's roofline line); never needed for correctness. */
SPDP_API const char* spdp_last_kernel(void);

/* Debug timeline of the packed-u16 sweep (measurement only): with a non-NULL
 * DEVICE pointer to a zeroed u64 buffer, every later split_sweep_u16_kernel appends, per tile
 * and consumer warp, {sm << 16 | warp slot, tile, start ns, end ns} (global timer) as 4 u64
 * after a u64 record counter at [0] (records start at [2]); the caller sizes the buffer
 * (2 + 4 x tiles x 4 u64).  NULL switches it off.  Process-wide; returns SPDP_E_CUDA on a
 * failed symbol copy. */
SPDP_API spdp_status spdp_debug_timeline(void* buffer);

/* Workspace bytes needed by spdp_split_eval / spdp_split_eval_batch for T tours
 * of n customers over S scenarios (T = 1 for spdp_split_eval). */
SPDP_API size_t spdp_workspace_bytes(int32_t n, int64_t S, int32_t T);

/* a1. Scenario generation: demand[(c-1)*ld + j] = q of customer c in global
 * scenario s_begin + j, j in [0, S).  Bit-identical to the host definition
 * above for any (s_begin, S) split, so ranks generate their own shards.
 * model: HOST pointer to the struct (its `nominal` is a device pointer). */
SPDP_API spdp_status spdp_gen_demands(const spdp_demand_model* model, int64_t s_begin, int64_t S,
                             uint16_t* demand, int64_t ld, spdp_stream_t stream);

/* a1 (layout). Scenario ordering for repeated / batched evaluation of one scenario set
 * (DESIGN §"scenario order"; a warp runs each layer at the deepest Eq. (3)
 * window among its lanes, so scenarios with similar loads belong in the same warp).
 *   key(s) = sum_c demand[c][s];  bucket(s) = floor(key(s) * 1024 / (max_s key(s) + 1));
 *   perm[j] = within each segment of 65536 consecutive scenarios, the segment's scenarios in
 *             increasing bucket order, increasing index within a bucket (stable: deterministic);
 *   out[c][j] = demand[c][perm[j]]  (out may be NULL).
 * Every evaluation of `out` equals the evaluation of `demand` with its scenarios permuted:
 * costs[j] belong to scenario perm[j]; SAA partials are identical.  demand, out, perm
 * (int32 [S]) are DEVICE pointers, out must not alias demand; ws: spdp_order_workspace_bytes(S)
 * bytes of device scratch.  Asynchronous on `stream`.  Errors: E_USAGE (sizes, NULL, aliasing,
 * small workspace), E_RESOURCE (n > SPDP_MAX_N, S >= 2^31), E_CUDA. */
SPDP_API size_t spdp_order_workspace_bytes(int64_t S);
SPDP_API spdp_status spdp_order_scenarios(const uint16_t* demand, int64_t ld, int32_t n, int64_t S, uint16_t* out,
                                          int64_t ld_out, int32_t* perm, void* ws, size_t ws_bytes,
                                          spdp_stream_t stream);

/* a3. Tour-order demand prefix sums ("prefix-sum operations";
 * SPEC:127-135): prefix[i*S + j] = sum_{k<=i} q^j_{sigma_k}, i = 0..n
 * (uint32 [n+1][S], scenario-minor). */
SPDP_API spdp_status spdp_demand_prefix(const int32_t* tour, int32_t n, const uint16_t* demand, int64_t ld,
                               int64_t S, uint32_t* prefix, spdp_stream_t stream);

/* a4. Masks, Eq. (2): mask[(i-1)*S + j] = min{p < i : sum_{k=p+1}^{i}
 * q^j_{sigma_k} <= Q}, or -1 when q^j_{sigma_i} > Q (DESIGN R4).  int32 [n][S]. */
SPDP_API spdp_status spdp_split_mask(const int32_t* tour, int32_t n, const uint16_t* demand, int64_t ld,
                            int64_t S, int32_t Q, int32_t* mask, spdp_stream_t stream);

/* a2+a5+a6. Split evaluation of one giant tour over S scenarios:
 *   f(0) = 0,  f(i) = min_{mask(i) <= p <= i-1} f(p) + c_{0,sigma_{p+1}}
 *                     + sum_{k=p+1}^{i-1} c_{sigma_k,sigma_{k+1}} + c_{sigma_i,0}
 *   cost[j] = f(n) of scenario j  (int32 [S], may be NULL)
 *   partial = SAA partial over the S scenarios (DEVICE pointer to ONE
 *             spdp_saa_partial, may be NULL), overwritten (not accumulated).
 * Q >= 1.  window_hint: expected maximum window width i - mask(i) (0 = sample
 * the data to choose); it only selects the kernel variant, never the result:
 * scenarios whose window exceeds the variant's register ring are finished by
 * a general transition-parallel kernel.  The int32 range bound is
 * 3*n*max(dist) + max(dist) < 2^31 (checked with SPDP_F_VALIDATE). */
SPDP_API spdp_status spdp_split_eval(const int32_t* tour, const int32_t* dist, int32_t n,
                            const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                            int32_t* cost, spdp_saa_partial* partial, int32_t window_hint,
                            void* ws, size_t ws_bytes, uint32_t flags, spdp_stream_t stream);

/* a8. Batched tours (tour x scenario x transition parallelism): T tours
 * [T][n] over the same demand set.  cost [T][S] (may be NULL), partial [T]
 * (may be NULL), one SAA partial per tour. */
SPDP_API spdp_status spdp_split_eval_batch(const int32_t* tours, int32_t T, const int32_t* dist, int32_t n,
                                  const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                  int32_t* cost, spdp_saa_partial* partial, int32_t window_hint,
                                  void* ws, size_t ws_bytes, uint32_t flags, spdp_stream_t stream);

/* f2. Penalized split (DESIGN R22): the split of spdp_split_eval
 * with EVERY p admissible and a linear overload penalty (the paper
 * reports "penalized cost" only, without defining it):
 *   f(i) = min_{0 <= p <= i-1} f(p) + t(p,i) + lambda * max(0, sum_{k=p+1}^{i} q - Q)
 * lambda >= 0 (cost units per unit of overload).  Every scenario is feasible
 * (partial->n_infeas = 0).  lambda = 0 is the split without capacity; a lambda
 * above every route-cost difference gives the strict split whenever that is
 * feasible.  Same workspace (spdp_workspace_bytes(n, S, 1)), layout and window_hint
 * semantics as spdp_split_eval; int32 results (scenarios whose lambda * load
 * reaches 2^29 are finished in int64 by a slower per-scenario kernel). */
SPDP_API spdp_status spdp_split_eval_penalized(const int32_t* tour, const int32_t* dist, int32_t n,
                                      const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                      int32_t lambda, int32_t* cost, spdp_saa_partial* partial,
                                      int32_t window_hint, void* ws, size_t ws_bytes, uint32_t flags,
                                      spdp_stream_t stream);

/* f1. Route recovery for K selected scenarios: the same DP as
 * spdp_split_eval (Eq. (1)-(3)), recording for every prefix i the
 * optimal last split point p = pred[k][i] (the route sigma_{p+1}..sigma_i is the
 * last one of the optimal split of the first i customers); ties keep the
 * LARGEST p (DESIGN R10), so pred equals the oracle's exactly.
 *   scen    [K] int64: scenario (column) indices, each in [0, S)      (device)
 *   pred    [K][n+1] int32: pred[k][0] = -1; -1 where f(i) is infinite (device)
 *   cost    [K] int32: f(n), SPDP_INFEASIBLE if a demand exceeds Q      (device)
 *   nroutes [K] int32 (may be NULL): routes of the optimal split of all n
 *   maxload [K] int32 (may be NULL): largest route load (<= Q: the capacity
 *           feasibility of every returned route, checked on the device)
 * Walking pred from i = n back to 0 lists the routes (tour positions
 * pred[i]..i-1, 0-based).  A warp per scenario for n <= 1024 (window start by ballot,
 * minimum and its largest argument by warp reductions, P and g in shared memory), one
 * thread per scenario above (latency-oriented: for inspecting a few thousand scenarios,
 * e.g. the worst ones of an SAA sample).  Ties go to the largest split point.
 * ws: spdp_routes_workspace_bytes(n, K) bytes of device memory. */
SPDP_API size_t spdp_routes_workspace_bytes(int32_t n, int32_t K);
SPDP_API spdp_status spdp_split_routes(const int32_t* tour, const int32_t* dist, int32_t n,
                              const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                              const int64_t* scen, int32_t K, int32_t* pred, int32_t* cost,
                              int32_t* nroutes, int32_t* maxload, void* ws, size_t ws_bytes,
                              spdp_stream_t stream);

/* f3 (DESIGN R23). Prefix and suffix split values of one tour,
 * the state that candidate tours sharing a prefix / suffix with it reuse
 * (evaluate many candidate first-stage tours):
 *   fwd[i*S + j] = Split(sigma_1..sigma_i)      of scenario j, i = 0..n (fwd[0] = 0)
 *   bwd[i*S + j] = Split(sigma_{i+1}..sigma_n)  of scenario j, i = 0..n (bwd[n] = 0)
 * (Split = Eq. (1), of the sub-tour as a standalone problem).
 * int32 [n+1][S] each (DEVICE, caller-owned), SPDP_INFEASIBLE where the prefix /
 * suffix holds a demand above Q.  fwd[n] = bwd[0] = the spdp_split_eval cost.
 * One thread per scenario: a 32-entry register ring per direction, scenarios whose
 * window outgrows it (or with a demand above Q) by a general kernel (any window).
 * ws: spdp_values_workspace_bytes(n, S) bytes of device memory.  Same argument
 * rules as spdp_split_eval; n ld < 2^32. */
SPDP_API size_t spdp_values_workspace_bytes(int32_t n, int64_t S);
SPDP_API spdp_status spdp_split_values(const int32_t* tour, const int32_t* dist, int32_t n,
                              const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                              int32_t* fwd, int32_t* bwd, void* ws, size_t ws_bytes,
                              spdp_stream_t stream);

/* f3. Neighbourhood evaluation: the split cost of T candidate tours [T][n] that
 * are permutations of the same customers as `parent`, from the parent's values
 * (fwd, bwd from spdp_split_values on the SAME demand, dist and Q).  A candidate
 * equal to the parent on positions 1..a and s0+1..n only re-runs the Eq. (3)
 * sweep from layer a+1 to the last layer a route starting before s0 can reach,
 * then takes cost = min_{s0 <= i <= E} f(i) + bwd[i] (every split has a route
 * boundary there).  Results (cost [T][S] int32, may be NULL; partial [T], may be
 * NULL, overwritten) are bit-identical to spdp_split_eval_batch on `tours`.
 * window_hint: 1..24 selects a 16-entry register ring, else 32 entries (with
 * SPDP_F_NBR_SMEM: a shared-memory ring of 32, or 64 entries for hints above 32);
 * wider windows are finished by the general kernel.  SPDP_F_VALIDATE checks the
 * candidates (not the parent).  ws: spdp_neighbour_workspace_bytes(n, S, T). */
SPDP_API size_t spdp_neighbour_workspace_bytes(int32_t n, int64_t S, int32_t T);
/* Several parents in one call (an HGS population's neighbourhoods): parents [P][n], fwd / bwd
 * [P][n+1][S] (spdp_split_values of each parent, stacked), parent_of [T] int32 (DEVICE; the
 * parent of candidate t, clamped to [0, P); may be NULL when P = 1).  Same results as P calls
 * of spdp_split_eval_neighbours; same workspace size. */
SPDP_API spdp_status spdp_split_eval_neighbours_multi(const int32_t* parents, int32_t P, const int32_t* parent_of,
                                             const int32_t* fwd, const int32_t* bwd, const int32_t* tours,
                                             int32_t T, const int32_t* dist, int32_t n, const uint16_t* demand,
                                             int64_t ld, int64_t S, int32_t Q, int32_t* cost,
                                             spdp_saa_partial* partial, int32_t window_hint, void* ws,
                                             size_t ws_bytes, uint32_t flags, spdp_stream_t stream);
SPDP_API spdp_status spdp_split_eval_neighbours(const int32_t* parent, const int32_t* fwd, const int32_t* bwd,
                                       const int32_t* tours, int32_t T, const int32_t* dist, int32_t n,
                                       const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                       int32_t* cost, spdp_saa_partial* partial, int32_t window_hint,
                                       void* ws, size_t ws_bytes, uint32_t flags, spdp_stream_t stream);

/* f4 (DESIGN R24). Split with a route-duration limit and a fleet
 * limit ("route length/duration constraints, if applicable"; PAPER:68
 * "three vehicles available"):
 *   route (p, i] admissible iff  sum_{k=p+1}^{i} q <= Q  and
 *     t(p, i) = c_{0,s_{p+1}} + sum_{k=p+1}^{i-1} c_{s_k,s_{k+1}} + c_{s_i,0} <= max_duration
 *   F_0(0) = 0, F_k(i) = min_{admissible (p, i]} F_{k-1}(p) + t(p, i),
 *   cost[j] = min_{1 <= k <= max_routes} F_k(n)  of scenario j
 * max_duration < 0: no duration limit; max_routes <= 0 (or >= n): no fleet limit
 * (one pass of Eq. (3)).  SPDP_INFEASIBLE when no admissible split exists (a
 * demand above Q, a customer whose out-and-back trip exceeds max_duration, or
 * more routes needed than max_routes).  cost [S] int32 (may be NULL), partial:
 * ONE spdp_saa_partial (may be NULL, overwritten).  One thread per scenario: without a
 * fleet limit a register-ring sweep with a per-layer duration bitmask; with one, a
 * 16-position shared-memory ring kernel keeps the vehicle-count dimension to the band
 * [kP(i), kP(i) + max_routes - kT] of the capacity bounds (kP = greedy route count
 * of the prefix, kT of the tour); scenarios whose window or band outgrows it go to
 * a general kernel (K passes, arrays of n+1 per scenario; SPDP_F_SCRATCH_GLOBAL
 * sends every scenario there).  n ld < 2^32, S < 2^31; the int32 range bound of
 * spdp_split_eval applies.  ws: spdp_limits_workspace_bytes(n, S) bytes of device
 * memory. */
SPDP_API size_t spdp_limits_workspace_bytes(int32_t n, int64_t S);
SPDP_API spdp_status spdp_split_eval_limits(const int32_t* tour, const int32_t* dist, int32_t n,
                                   const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                   int32_t max_duration, int32_t max_routes, int32_t* cost,
                                   spdp_saa_partial* partial, void* ws, size_t ws_bytes, uint32_t flags,
                                   spdp_stream_t stream);

/* a5 fp32 mode (DESIGN R25): real-valued route costs.
 * dist: DEVICE fp64 [(n+1)*(n+1)] row-major (c_{a,b} >= 0).  With the fp64 prefix
 * Dd[1] = 0, Dd[i] = Dd[i-1] + c_{s_{i-1},s_i} (sequential) and the route cost of
 * Eq. (1) rounded once, T32(p,i) = fl32((c_{0,s_{p+1}} + (Dd[i] - Dd[p+1])) + c_{s_i,0}):
 *   f(0) = 0,  f(i) = min_{mask(i) <= p <= i-1} fl32(f(p) + T32(p,i))
 *   cost[j] = f(n) of scenario j (float [S], +INFINITY when a demand exceeds Q).
 * One IEEE single add per candidate and an exact min: bit-identical for every launch
 * configuration.  One thread per scenario on a 32-entry register ring with the band table
 * T32(i-k, i), k <= 32, formed once per call; scenarios with wider windows by a general
 * kernel (any window).  ws: spdp_f32_workspace_bytes(n, S) bytes (the f rows [n+1][S] fp32
 * of the general kernel, the tables, a deferral list).  n ld < 2^32. */
SPDP_API size_t spdp_f32_workspace_bytes(int32_t n, int64_t S);
SPDP_API spdp_status spdp_split_eval_f32(const int32_t* tour, const double* dist, int32_t n,
                                const uint16_t* demand, int64_t ld, int64_t S, int32_t Q,
                                float* cost, void* ws, size_t ws_bytes, spdp_stream_t stream);

/* a8 in fp32 mode: T tours [T][n] over the same demand set, cost [T][S] float (the tours run
 * one after the other on `stream`, sharing the workspace of spdp_f32_workspace_bytes(n, S)). */
SPDP_API spdp_status spdp_split_eval_batch_f32(const int32_t* tours, int32_t T, const double* dist, int32_t n,
                                      const uint16_t* demand, int64_t ld, int64_t S, int32_t Q, float* cost,
                                      void* ws, size_t ws_bytes, spdp_stream_t stream);

/* SAA estimate of fp32 costs (SURVEY §8(c5) fp32 mode): over the finite costs, fp64 sums
 * in two passes (mean, then the squared deviations), agreeing with a sequential fp64
 * evaluation within 1e-9 relative.  cost: DEVICE float [S]; ws: 64 bytes of device
 * memory; synchronizes `stream`; E_DATA when every cost is infinite. */
SPDP_API spdp_status spdp_saa_estimate_f32(const float* cost, int64_t S, spdp_saa_estimate* out_h,
                                  void* ws, size_t ws_bytes, spdp_stream_t stream);

/* The moments behind it, for a multi-rank estimate (asynchronous): moments (DEVICE double[4],
 * overwritten) = {m, sum c, sum (c - center)^2, infeasible} over the finite costs.  Two passes
 * across ranks (paper_2511_18022_b200.dist.saa_estimate_f32): all-reduce(SUM) of the pass with
 * center 0 gives the global mean, all-reduce of the pass centred on it the squared deviations. */
SPDP_API spdp_status spdp_saa_f32_moments(const float* cost, int64_t S, double center, double* moments,
                                 spdp_stream_t stream);

/* fp32-mode SAA finalize (host, synchronous): from the SUMMED pass-1 moments m1
 * (HOST double[4], spdp_saa_f32_moments with center 0, all-reduced over ranks) the count,
 * infeasible count and mean -- the centre of pass 2 -- and, when m2 (HOST double[4], the summed
 * pass centred on that mean) is non-NULL, also var (m - 1 denominator), std_err and the 95 %
 * interval; with m2 NULL those stay NaN.  E_DATA when no cost is finite. */
SPDP_API spdp_status spdp_saa_finalize_f32(const double* m1, const double* m2, spdp_saa_estimate* out_h);

/* a6 standalone: SAA partial of a cost vector (SPDP_INFEASIBLE entries are
 * counted in n_infeas and excluded).  partial: DEVICE pointer to one struct. */
SPDP_API spdp_status spdp_saa_reduce(const int32_t* cost, int64_t S, spdp_saa_partial* partial,
                            spdp_stream_t stream);

/* a6 finalize (host, synchronous): estimate from a (possibly all-reduced)
 * partial.  E_DATA when n_feas == 0. */
SPDP_API spdp_status spdp_saa_mean(const spdp_saa_partial* partial_h, spdp_saa_estimate* out_h);

/* End-to-end entry with HOST buffers: copies tour/dist/demand host->device
 * (pinned host memory recommended), runs spdp_split_eval, copies the partial
 * (and cost_h if non-NULL) back and finalizes the estimate.  Synchronizes
 * `stream`.  demand_h is [n][ld_h] uint16 (ld_h >= S).  ws must hold
 * spdp_host_workspace_bytes(n, S) bytes of DEVICE memory. */
SPDP_API size_t spdp_host_workspace_bytes(int32_t n, int64_t S);
SPDP_API spdp_status spdp_split_eval_host(const int32_t* tour_h, const int32_t* dist_h, int32_t n,
                                 const uint16_t* demand_h, int64_t ld_h, int64_t S, int32_t Q,
                                 int32_t* cost_h, spdp_saa_estimate* est_h, int32_t window_hint,
                                 void* ws, size_t ws_bytes, spdp_stream_t stream);

/* a9+a10. Inventory-routing recourse DP (model SURVEY §8(c6), DESIGN R21):
 * per scenario j and customer m, V_0[I0] = 0, and for t = 0..H-1
 *   W_t[y]     = min_{I in [max(0, y - z_{m,t} X), y]} V_t[I] + c (y - I)          (delivery)
 *   V_{t+1}[J] = W_t[J + d] + h J                       for J >= 1, J + d <= U     (demand d)
 *   V_{t+1}[0] = min_{y <= min(d, U)} W_t[y] + b (d - y)
 * cost[j] = sum_m min_J V_H[J] (int64 [S], overwritten).  visit_h: HOST uint8 [M][H]
 * (z_{m,t}); cust_h: HOST array [M]; both are copied into `ws` (size from
 * spdp_irp_workspace_bytes).  demand: uint16 [H*M][ld], row t*M + m.
 * U <= 1023 and H (c X + h U + b 65535) < 2^29 per customer (else E_RESOURCE).
 * partial (may be NULL): SAA partial of the S costs (DEVICE pointer); needs the sum of those
 * per-customer bounds below 2^31 (cost^2 must fit the summable int64 halves), else E_RESOURCE.
 * flags: SPDP_F_IRP_EAGER selects the eager-shift kernel, SPDP_F_IRP_STATES the state-parallel
 * one (same results; the default for X == 0 or X >= U is the lazy affine-tail lane kernel). */
SPDP_API size_t spdp_irp_workspace_bytes(int32_t H, int32_t M, int64_t S);
SPDP_API spdp_status spdp_irp_dp(const uint8_t* visit_h, const spdp_irp_customer* cust_h, int32_t H, int32_t M,
                        const uint16_t* demand, int64_t ld, int64_t S, int64_t* cost,
                        spdp_saa_partial* partial, void* ws, size_t ws_bytes, uint32_t flags,
                        spdp_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SPDP_H */
