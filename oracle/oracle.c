/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 2511.18022 ("GPU-accelerated DP for scenario-based stochastic
 * combinatorial optimization").
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2511_18022_b200/) may include, link or call this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg load it.  It shares no code, header, table or constant
 * generator with the CUDA path.
 *
 * Citations: PAPER:n = line n of the paper text; SPEC:n = line n
 * of SPEC.md; SURVEY §x = /root/repo/SURVEY.md; DESIGN Rk = reading k in
 * DESIGN.md section "Readings of the paper".
 *
 * Arithmetic: integers throughout (int64 DP values, __int128 for SAA
 * second moments), so every result is exact.  No blocking, no fusion, no
 * reordering beyond what the definitions state.
 *
 * Functions and their pins (tests/test_oracle_*.py):
 *   oracle_philox4x32_10     Random123 known-answer vectors (tests/golden/philox_kat.txt)
 *   oracle_gen_demands       fixed/cv=0 identities, determinism, shard invariance,
 *                            moments and correlation within 3-4 standard errors
 *   oracle_tour_prefix       SPEC:68 collinear D=[0,1,2]; direct arc sums
 *   oracle_demand_prefix     SPEC:133 [14,15,8,1,8] -> [0,14,29,37,38,46]
 *   oracle_mask              SPEC:199-200 Example-1 masks; definitional scan
 *   oracle_split_eq1         brute force over all 2^(n-1) partitions (pure Python,
 *                            in the test); PAPER:64-66 Example 1(i) routes; closed forms
 *   oracle_split_scan        == oracle_split_eq1 on random cases; O(n) deque split
 *                            (independent algorithm, in the test) for deterministic demand
 *   oracle_split_values      brute force over the partitions of every prefix / suffix;
 *                            b(i) of a tour = f(n-i) of the reversed tour under the
 *                            transposed costs; f(i) + b(i) >= cost, = at optimal boundaries
 *   oracle_split_limits      brute force over partitions with <= K routes of duration
 *                            <= Lmax; no limits = plain split; monotone in K and Lmax
 *   oracle_split_f32         integer-valued costs = oracle_split exactly; real costs within the
 *                            fp32 rounding bound of an fp64 brute force over partitions
 *   oracle_saa               Python statistics.fmean/variance (exact Fractions) on costs
 *   oracle_saa_f32           Python statistics on exact Fractions within 1e-12 relative
 *   oracle_irp               brute force over all action sequences (pure Python, in
 *                            the test); two closed forms
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <stdlib.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_INF INT64_MAX

/* ------------------------------------------------------------------------ */
/* a1. Counter-based scenario generator (DESIGN R14).         */
/* Philox4x32-10 (Salmon et al., SC'11), written from its definition: ten    */
/* rounds of  (L,R) <- (hi(R0*M0) ^ k0 ^ L1, lo(R0*M0), ...) with a Weyl key  */
/* schedule.                                                                  */
/* ------------------------------------------------------------------------ */
static const uint32_t PHILOX_M0 = 0xD2511F53u, PHILOX_M1 = 0xCD9E8D57u;
static const uint32_t PHILOX_W0 = 0x9E3779B9u, PHILOX_W1 = 0xBB67AE85u;

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += PHILOX_W0; k1 += PHILOX_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* floor(a / b) for b > 0 (C division truncates toward zero). */
static int64_t floor_div_i64(int64_t a, int64_t b)
{
    int64_t q = a / b;
    if ((a % b != 0) && (a < 0)) q -= 1;
    return q;
}

/* Irwin-Hall(4) on the 16-bit high halves of one Philox block, centred:
 * z = sum_j (u_j >> 16) - 131070  (mean of four U{0..65535} is 131070). */
static int64_t irwin_hall4_centred(const uint32_t u[4])
{
    int64_t z = 0;
    for (int j = 0; j < 4; ++j) z += (int64_t)(u[j] >> 16);
    return z - 131070;
}

/* Demand of customer c (1-based) in global scenario s.
 * kind 0 fixed: q = mu_c                                      ("fixed")
 * kind 1 uniform-int: q = lo + floor(u0 * (hi-lo+1) / 2^32),  lo = mu*lo_pm/1000, hi = mu*hi_pm/1000
 * kind 2 correlated: q = mu + floor((mu*(A*z_s + B*z_sc) + D/2) / D),  D = 37837 * 2^16
 *        z_s from counter c=0 (scenario-level common factor), z_sc from counter c.
 * then clamp to [0, q_cap]. */
static uint16_t oracle_demand_one(int32_t kind, uint16_t mu, int32_t lo_pm, int32_t hi_pm,
                                  int64_t A_fx, int64_t B_fx, int32_t q_cap,
                                  uint64_t seed, uint32_t stream_tag, int64_t s, int32_t c)
{
    int64_t q;
    uint32_t key[2] = { (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32) };
    if (kind == 0) {
        q = mu;
    } else if (kind == 1) {
        uint32_t ctr[4] = { (uint32_t)((uint64_t)s & 0xffffffffu), (uint32_t)((uint64_t)s >> 32),
                            (uint32_t)c, stream_tag };
        uint32_t u[4];
        oracle_philox4x32_10(ctr, key, u);
        int64_t lo = ((int64_t)mu * lo_pm) / 1000;
        int64_t hi = ((int64_t)mu * hi_pm) / 1000;
        if (hi < lo) hi = lo;
        q = lo + (int64_t)(((uint64_t)u[0] * (uint64_t)(hi - lo + 1)) >> 32);
    } else {
        uint32_t ctr0[4] = { (uint32_t)((uint64_t)s & 0xffffffffu), (uint32_t)((uint64_t)s >> 32),
                             0u, stream_tag };
        uint32_t ctrc[4] = { ctr0[0], ctr0[1], (uint32_t)c, stream_tag };
        uint32_t u0[4], uc[4];
        oracle_philox4x32_10(ctr0, key, u0);
        oracle_philox4x32_10(ctrc, key, uc);
        int64_t zs = irwin_hall4_centred(u0);
        int64_t zc = irwin_hall4_centred(uc);
        const int64_t D = 37837LL * 65536LL;
        int64_t num = (int64_t)mu * (A_fx * zs + B_fx * zc) + D / 2;
        q = (int64_t)mu + floor_div_i64(num, D);
    }
    if (q < 0) q = 0;
    if (q > q_cap) q = q_cap;
    return (uint16_t)q;
}

/* demand[(c-1)*ld + j] = demand of customer c in global scenario s_begin + j. */
int oracle_gen_demands(int32_t kind, const uint16_t* nominal, int32_t n,
                       int32_t lo_pm, int32_t hi_pm, int64_t A_fx, int64_t B_fx, int32_t q_cap,
                       uint64_t seed, uint32_t stream_tag,
                       int64_t s_begin, int64_t S, uint16_t* demand, int64_t ld, int threads)
{
    if (n < 1 || S < 0 || ld < S) return 2;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t j = 0; j < S; ++j)
        for (int32_t c = 1; c <= n; ++c)
            demand[(int64_t)(c - 1) * ld + j] =
                oracle_demand_one(kind, nominal[c - 1], lo_pm, hi_pm, A_fx, B_fx, q_cap,
                                  seed, stream_tag, s_begin + j, c);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* a2. Tour distance prefix D: D[1]=0, D[i]=D[i-1]+c[s_{i-1}][s_i]. */
/* Output D[0..n] with D[0] := 0 unused.                                     */
/* ------------------------------------------------------------------------ */
void oracle_tour_prefix(int32_t n, const int32_t* tour, const int32_t* dist, int64_t* D)
{
    const int64_t N1 = (int64_t)n + 1;
    D[0] = 0;
    if (n >= 1) D[1] = 0;
    for (int32_t i = 2; i <= n; ++i)
        D[i] = D[i - 1] + dist[(int64_t)tour[i - 2] * N1 + tour[i - 1]];
}

/* ------------------------------------------------------------------------ */
/* a3. Tour-order demand prefix:               */
/*     P[s][0]=0, P[s][i] = sum_{k<=i} q_{sigma_k}^s.  Output [n+1][S].     */
/* ------------------------------------------------------------------------ */
void oracle_demand_prefix(int32_t n, const int32_t* tour, const uint16_t* demand, int64_t ld,
                          int64_t S, int64_t* P)
{
    for (int64_t s = 0; s < S; ++s) {
        int64_t acc = 0;
        P[s] = 0;
        for (int32_t i = 1; i <= n; ++i) {
            acc += demand[(int64_t)(tour[i - 1] - 1) * ld + s];
            P[(int64_t)i * S + s] = acc;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* a4. Mask, Eq. (2): mask(i) = min{p : 0<=p<i,              */
/*     sum_{k=p+1}^{i} q_{sigma_k} <= Q}; -1 (INFEASIBLE) if the set is      */
/*     empty (DESIGN R4).  Written as the definition: for each p from 0 up,  */
/*     sum the segment directly.  Output [n][S], row i-1 = position i.       */
/* ------------------------------------------------------------------------ */
void oracle_mask(int32_t n, const int32_t* tour, const uint16_t* demand, int64_t ld, int64_t S,
                 int32_t Q, int32_t* mask)
{
    for (int64_t s = 0; s < S; ++s) {
        for (int32_t i = 1; i <= n; ++i) {
            int32_t m = -1;
            for (int32_t p = 0; p < i; ++p) {
                int64_t load = 0;
                for (int32_t k = p + 1; k <= i; ++k) load += demand[(int64_t)(tour[k - 1] - 1) * ld + s];
                if (load <= Q) { m = p; break; }
            }
            mask[(int64_t)(i - 1) * S + s] = m;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* a5. Split, Eq. (1) written out literally:                   */
/*   f(0)=0; f(i) = min_{0<=p<=i-1} f(p) + c_{0,s_{p+1}}                      */
/*                  + sum_{k=p+1}^{i-1} c_{s_k,s_{k+1}} + c_{s_i,n+1}        */
/*   subject to sum_{k=p+1}^{i} q_{s_k} <= Q  (inclusive, PAPER:66 load 17=Q).*/
/* Node n+1 is the depot 0 (DESIGN R6).  Every segment sum is       */
/* recomputed from scratch: O(n^3) per scenario -- for small n only.         */
/* Ties: p ascending with "<=" keeps the LARGEST p (DESIGN R10).   */
/* q: the n demands of ONE scenario in TOUR order (DESIGN R1).     */
/* ------------------------------------------------------------------------ */
static int64_t split_eq1_one(int32_t n, const int32_t* tour, const int32_t* dist, int32_t Q,
                             const int64_t* q, int64_t* f, int32_t* pred)
{
    const int64_t N1 = (int64_t)n + 1;
    f[0] = 0;
    for (int32_t i = 1; i <= n; ++i) {
        int64_t best = ORACLE_INF;
        int32_t arg = -1;
        for (int32_t p = 0; p <= i - 1; ++p) {
            int64_t load = 0;
            for (int32_t k = p + 1; k <= i; ++k) load += q[k - 1];
            if (load > Q) continue;
            if (f[p] == ORACLE_INF) continue;
            int64_t chain = 0;
            for (int32_t k = p + 1; k <= i - 1; ++k)
                chain += dist[(int64_t)tour[k - 1] * N1 + tour[k]];
            int64_t cand = f[p] + dist[0 * N1 + tour[p]] + chain + dist[(int64_t)tour[i - 1] * N1 + 0];
            if (cand <= best) { best = cand; arg = p; }
        }
        f[i] = best;
        if (pred) pred[i] = arg;
    }
    if (pred) pred[0] = -1;
    return f[n];
}

/* ------------------------------------------------------------------------ */
/* a5. Split, Eq. (1) as a descending scan over p:           */
/*   for p = i-1 down to 0: load += q_{p+1}; if load > Q break;              */
/* The break is exact because q >= 0 makes the segment load nondecreasing as */
/* p decreases (DESIGN R5), so the last accepted p is mask(i) of Eq. (2) and */
/* the loop visits exactly the candidates of Eq. (3).  The chain */
/* term sum_{k=p+1}^{i-1} c is accumulated right-to-left as p decreases.     */
/* Ties: strict "<" while p decreases keeps the LARGEST p (DESIGN R10).      */
/* Also returns sum_i w(i), w(i) = i - mask(i): the Eq. (3) candidate count. */
/* ------------------------------------------------------------------------ */
/* (N1 = the row stride of dist: n + 1 for a whole tour, larger for a sub-tour.) */
static int64_t split_scan_sub(int32_t n, const int32_t* tour, const int32_t* dist, int64_t N1, int32_t Q,
                              const int64_t* q, int64_t* f, int32_t* pred, int64_t* wsum)
{
    int64_t cnt = 0;
    f[0] = 0;
    for (int32_t i = 1; i <= n; ++i) {
        int64_t best = ORACLE_INF;
        int32_t arg = -1;
        int64_t load = 0, chain = 0;
        for (int32_t p = i - 1; p >= 0; --p) {
            load += q[p];                         /* q_{sigma_{p+1}} */
            if (load > Q) break;
            if (p + 1 <= i - 1) chain += dist[(int64_t)tour[p] * N1 + tour[p + 1]];
            cnt += 1;
            if (f[p] == ORACLE_INF) continue;
            int64_t cand = f[p] + dist[0 * N1 + tour[p]] + chain + dist[(int64_t)tour[i - 1] * N1 + 0];
            if (cand < best) { best = cand; arg = p; }
        }
        f[i] = best;
        if (pred) pred[i] = arg;
    }
    if (pred) pred[0] = -1;
    if (wsum) *wsum = cnt;
    return f[n];
}

static int64_t split_scan_one(int32_t n, const int32_t* tour, const int32_t* dist, int32_t Q,
                              const int64_t* q, int64_t* f, int32_t* pred, int64_t* wsum)
{
    return split_scan_sub(n, tour, dist, (int64_t)n + 1, Q, q, f, pred, wsum);
}

/* Batch driver: scenario s of demand[n][ld] (customer-id rows, DESIGN R1),
 * gathered to tour order, then one of the two single-scenario routines.
 * cost[s] = f(n) or ORACLE_INF (infeasible, DESIGN R4).
 * pred (nullable) is [S][n+1]; wsum (nullable) is [S].
 * method 0 = scan (O(n w)), 1 = literal Eq. (1) (O(n^3)). */
int oracle_split_batch(int32_t n, const int32_t* tour, const int32_t* dist, int32_t Q,
                       const uint16_t* demand, int64_t ld, int64_t S, int32_t method,
                       int64_t* cost, int32_t* pred, int64_t* wsum, int threads)
{
    if (n < 1 || S < 0 || Q < 1 || ld < S) return 2;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        int64_t* f = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t s = 0; s < S; ++s) {
            for (int32_t k = 1; k <= n; ++k) q[k - 1] = demand[(int64_t)(tour[k - 1] - 1) * ld + s];
            int32_t* pr = pred ? pred + s * (int64_t)(n + 1) : NULL;
            int64_t w = 0;
            int64_t c = (method == 1) ? split_eq1_one(n, tour, dist, Q, q, f, pr)
                                      : split_scan_one(n, tour, dist, Q, q, f, pr, &w);
            cost[s] = c;
            if (wsum) wsum[s] = w;
        }
        free(q);
        free(f);
    }
    return 0;
}

/* Batched tours (BASELINE configs[2]): cost[t*S + s] for T tours [T][n]. */
int oracle_split_batch_tours(int32_t n, int32_t T, const int32_t* tours, const int32_t* dist, int32_t Q,
                             const uint16_t* demand, int64_t ld, int64_t S,
                             int64_t* cost, int threads)
{
    for (int32_t t = 0; t < T; ++t) {
        int rc = oracle_split_batch(n, tours + (int64_t)t * n, dist, Q, demand, ld, S, 0,
                                    cost + (int64_t)t * S, NULL, NULL, threads);
        if (rc) return rc;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* f3. Prefix and suffix split values of one tour, the   */
/* state that candidate tours sharing a prefix / suffix with it reuse        */
/* ("explore many more candidate first-stage tours"; DESIGN    */
/* R23).  Written as the definitions, not as a recursion over each other:    */
/*   fwd[i] = Split(sigma_1..sigma_i)      i = 0..n  (fwd[0] = 0)            */
/*   bwd[i] = Split(sigma_{i+1}..sigma_n)  i = 0..n  (bwd[n] = 0)            */
/* where Split(.) is Eq. (1) of the sub-tour as a standalone problem         */
/* (PAPER:98-101): fwd[i] is f(i) of the scan (Eq. (1) restricted to the      */
/* first i customers is the same recursion), bwd[i] is one more call of the  */
/* scan on the suffix.  O(n^2 w) per scenario: small cases only.            */
/* ORACLE_INF where the sub-tour holds a demand above Q (DESIGN R4).          */
/* fwd, bwd: [S][n+1] (row per scenario).                                     */
/* ------------------------------------------------------------------------ */
int oracle_split_values(int32_t n, const int32_t* tour, const int32_t* dist, int32_t Q,
                        const uint16_t* demand, int64_t ld, int64_t S,
                        int64_t* fwd, int64_t* bwd, int threads)
{
    if (n < 1 || S < 0 || Q < 1 || ld < S) return 2;
    const int64_t N1 = (int64_t)n + 1;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        int64_t* f = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t s = 0; s < S; ++s) {
            for (int32_t k = 1; k <= n; ++k) q[k - 1] = demand[(int64_t)(tour[k - 1] - 1) * ld + s];
            split_scan_one(n, tour, dist, Q, q, f, NULL, NULL);
            for (int32_t i = 0; i <= n; ++i) fwd[s * N1 + i] = f[i];
            bwd[s * N1 + n] = 0;
            for (int32_t i = 0; i < n; ++i)   /* the suffix sigma_{i+1..n}: n - i customers */
                bwd[s * N1 + i] = split_scan_sub(n - i, tour + i, dist, N1, Q, q + i, f, NULL, NULL);
        }
        free(q);
        free(f);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* f4. Split with a route-duration limit and a fleet     */
/* limit (DESIGN R24; "route length/duration constraints, if         */
/* applicable", "three vehicles available"):                         */
/*   a route (p, i] is admissible iff  sum_{k=p+1}^{i} q <= Q  and           */
/*   t(p, i) = c_{0,s_{p+1}} + sum_{k=p+1}^{i-1} c_{s_k,s_{k+1}} + c_{s_i,0}  */
/*   <= Lmax  (route duration = route cost; Lmax < 0: no limit);             */
/*   F_0(0) = 0, F_0(i>0) = inf,                                             */
/*   F_k(i) = min_{admissible (p,i]} F_{k-1}(p) + t(p, i)   (k = 1..K)        */
/*   cost = min_{1 <= k <= K} F_k(n)          (K <= 0: no fleet limit, K = n) */
/* The Eq. (1) layered DAG with a vehicle-count layer dimension.  Descending */
/* scan: the load break is exact (R5); the duration test only skips (t need  */
/* not be monotone in p without the triangle inequality).  Ties: the         */
/* smallest k, then (strict "<" while p decreases) the largest p.            */
/* pred (nullable) [S][n+1]: the last split point of the chosen layer's      */
/* path, k_used (nullable) [S]: the route count of the optimum.              */
/* ------------------------------------------------------------------------ */
int oracle_split_limits(int32_t n, const int32_t* tour, const int32_t* dist, int32_t Q,
                        int64_t Lmax, int32_t K, const uint16_t* demand, int64_t ld, int64_t S,
                        int64_t* cost, int32_t* pred, int32_t* k_used, int threads)
{
    if (n < 1 || S < 0 || Q < 1 || ld < S) return 2;
    const int64_t N1 = (int64_t)n + 1;
    const int32_t KK = (K <= 0 || K > n) ? n : K;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        int64_t* F = (int64_t*)malloc(sizeof(int64_t) * (size_t)(KK + 1) * (size_t)N1);
        int32_t* arg = (int32_t*)malloc(sizeof(int32_t) * (size_t)(KK + 1) * (size_t)N1);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t s = 0; s < S; ++s) {
            for (int32_t k = 1; k <= n; ++k) q[k - 1] = demand[(int64_t)(tour[k - 1] - 1) * ld + s];
            for (int32_t i = 0; i <= n; ++i) { F[i] = ORACLE_INF; arg[i] = -1; }
            F[0] = 0;
            for (int32_t k = 1; k <= KK; ++k) {
                int64_t* Fk = F + (int64_t)k * N1;
                const int64_t* Fp = F + (int64_t)(k - 1) * N1;
                Fk[0] = ORACLE_INF;
                arg[(int64_t)k * N1] = -1;
                for (int32_t i = 1; i <= n; ++i) {
                    int64_t best = ORACLE_INF, load = 0, chain = 0;
                    int32_t a = -1;
                    for (int32_t p = i - 1; p >= 0; --p) {
                        load += q[p];                               /* q_{sigma_{p+1}} */
                        if (load > Q) break;
                        if (p + 1 <= i - 1) chain += dist[(int64_t)tour[p] * N1 + tour[p + 1]];
                        const int64_t t = dist[0 * N1 + tour[p]] + chain + dist[(int64_t)tour[i - 1] * N1 + 0];
                        if (Lmax >= 0 && t > Lmax) continue;
                        if (Fp[p] == ORACLE_INF) continue;
                        const int64_t cand = Fp[p] + t;
                        if (cand < best) { best = cand; a = p; }
                    }
                    Fk[i] = best;
                    arg[(int64_t)k * N1 + i] = a;
                }
            }
            int64_t best = ORACLE_INF;
            int32_t kb = 0;
            for (int32_t k = 1; k <= KK; ++k)
                if (F[(int64_t)k * N1 + n] < best) { best = F[(int64_t)k * N1 + n]; kb = k; }
            cost[s] = best;
            if (k_used) k_used[s] = best == ORACLE_INF ? 0 : kb;
            if (pred) {
                int32_t* pr = pred + s * N1;
                for (int32_t i = 0; i <= n; ++i) pr[i] = -1;
                if (best != ORACLE_INF) {       /* the optimum's path: layer kb at n, kb-1 at its pred, ... */
                    int32_t i = n, k = kb;
                    while (i > 0 && k > 0) {
                        const int32_t p = arg[(int64_t)k * N1 + i];
                        pr[i] = p;
                        i = p;
                        --k;
                    }
                }
            }
        }
        free(q);
        free(F);
        free(arg);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* f2. Penalized split, DESIGN R22 (the paper names a      */
/* "penalized cost" only; SPEC:206 widens the window to every p    */
/* and adds lambda * max(0, load - Q), SPEC:252 keeps single-customer routes  */
/* admissible):                                                              */
/*   f(0) = 0,                                                               */
/*   f(i) = min_{0<=p<=i-1} f(p) + c_{0,s_{p+1}} + sum_{k=p+1}^{i-1}          */
/*          c_{s_k,s_{k+1}} + c_{s_i,0} + lambda * max(0, sum_{k=p+1}^{i} q - Q) */
/* Literal O(n^2) descending scan (load and chain accumulated right-to-left). */
/* Ties keep the largest p.  Every scenario is feasible.                     */
/* ------------------------------------------------------------------------ */
int oracle_split_penalized(int32_t n, const int32_t* tour, const int32_t* dist, int32_t Q, int64_t lambda,
                           const uint16_t* demand, int64_t ld, int64_t S, int64_t* cost, int32_t* pred,
                           int threads)
{
    if (n < 1 || S < 0 || Q < 1 || ld < S || lambda < 0) return 2;
    const int64_t N1 = (int64_t)n + 1;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        int64_t* f = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t s = 0; s < S; ++s) {
            for (int32_t k = 1; k <= n; ++k) q[k - 1] = demand[(int64_t)(tour[k - 1] - 1) * ld + s];
            int32_t* pr = pred ? pred + s * N1 : NULL;
            f[0] = 0;
            for (int32_t i = 1; i <= n; ++i) {
                int64_t best = ORACLE_INF, load = 0, chain = 0;
                int32_t arg = -1;
                for (int32_t p = i - 1; p >= 0; --p) {
                    load += q[p];                                   /* q_{sigma_{p+1}} */
                    if (p + 1 <= i - 1) chain += dist[(int64_t)tour[p] * N1 + tour[p + 1]];
                    const int64_t over = load - Q > 0 ? load - Q : 0;
                    int64_t cand = f[p] + dist[0 * N1 + tour[p]] + chain + dist[(int64_t)tour[i - 1] * N1 + 0]
                                   + lambda * over;
                    if (cand < best) { best = cand; arg = p; }
                }
                f[i] = best;
                if (pr) pr[i] = arg;
            }
            if (pr) pr[0] = -1;
            cost[s] = f[n];
        }
        free(q);
        free(f);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* a6. SAA estimate (PAPER:48, 264 (P_m)).                      */
/* Over feasible scenarios (cost != ORACLE_INF):                              */
/*   m = #feasible, mean = (1/m) sum c,                                      */
/*   var = (m sum c^2 - (sum c)^2) / (m (m-1))   (unbiased sample variance), */
/*   stderr = sqrt(var/m), ci95 = mean +- 1.96 stderr.                       */
/* Sums are exact (__int128); only the final divisions round.                */
/* out: [0]=m, [1]=infeasible, [2]=mean, [3]=var, [4]=stderr, [5]=lo, [6]=hi */
/* sums_out (nullable): exact sum and sum of squares as decimal-free int128  */
/* halves {sum_lo, sum_hi, sq_lo, sq_hi} (unsigned 64-bit limbs).            */
/* ------------------------------------------------------------------------ */
int oracle_saa(const int64_t* cost, int64_t S, double* out, uint64_t* sums_out)
{
    __int128 sum = 0, sq = 0;
    int64_t m = 0, inf = 0;
    for (int64_t s = 0; s < S; ++s) {
        if (cost[s] == ORACLE_INF) { inf++; continue; }
        m++;
        sum += (__int128)cost[s];
        sq += (__int128)cost[s] * (__int128)cost[s];
    }
    out[0] = (double)m;
    out[1] = (double)inf;
    if (sums_out) {
        sums_out[0] = (uint64_t)sum; sums_out[1] = (uint64_t)(sum >> 64);
        sums_out[2] = (uint64_t)sq;  sums_out[3] = (uint64_t)(sq >> 64);
    }
    if (m == 0) return 3;
    out[2] = (double)sum / (double)m;
    if (m >= 2) {
        __int128 num = (__int128)m * sq - sum * sum;        /* exact, >= 0 */
        out[3] = (double)num / ((double)m * (double)(m - 1));
    } else {
        out[3] = 0.0;
    }
    out[4] = sqrt(out[3] / (double)m);
    out[5] = out[2] - 1.96 * out[4];
    out[6] = out[2] + 1.96 * out[4];
    return 0;
}

/* ------------------------------------------------------------------------ */
/* a5 fp32 mode (SURVEY §8(a) a2/a5 "fp32 (one add + exact min)", §8(c3)    */
/* "fp32 mode (secondary)"; DESIGN R25): real-valued costs c (fp64 input).   */
/*   Dd[1] = 0, Dd[i] = Dd[i-1] + c[s_{i-1}][s_i]      (fp64, sequential)     */
/*   T32(p,i) = (float)((c[0][s_{p+1}] + (Dd[i] - Dd[p+1])) + c[s_i][0])     */
/*             (the route cost of Eq. (1), rounded ONCE to fp32)   */
/*   f(0) = 0, f(i) = min_{mask(i) <= p <= i-1} fl32(f(p) + T32(p,i))         */
/* Descending scan with the exact capacity break (as oracle_split_batch),    */
/* each candidate one IEEE single add (SSE, -ffp-contract=off), exact min.   */
/* cost[s] = f(n), +INFINITY when infeasible (a demand above Q, R4).          */
/* ------------------------------------------------------------------------ */
int oracle_split_f32(int32_t n, const int32_t* tour, const double* dist, int32_t Q,
                     const uint16_t* demand, int64_t ld, int64_t S, float* cost, int threads)
{
    if (n < 1 || S < 0 || Q < 1 || ld < S) return 2;
    const int64_t N1 = (int64_t)n + 1;
    double* Dd = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    Dd[0] = 0.0;
    Dd[1] = 0.0;
    for (int32_t i = 2; i <= n; ++i) Dd[i] = Dd[i - 1] + dist[(int64_t)tour[i - 2] * N1 + tour[i - 1]];
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        float* f = (float*)malloc(sizeof(float) * (size_t)(n + 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t s = 0; s < S; ++s) {
            for (int32_t k = 1; k <= n; ++k) q[k - 1] = demand[(int64_t)(tour[k - 1] - 1) * ld + s];
            f[0] = 0.0f;
            for (int32_t i = 1; i <= n; ++i) {
                float best = INFINITY;
                int64_t load = 0;
                for (int32_t p = i - 1; p >= 0; --p) {
                    load += q[p];                                   /* q_{sigma_{p+1}} */
                    if (load > Q) break;
                    const double t64 = (dist[0 * N1 + tour[p]] + (Dd[i] - Dd[p + 1])) + dist[(int64_t)tour[i - 1] * N1 + 0];
                    const float t32 = (float)t64;
                    const float cand = f[p] + t32;
                    if (cand < best) best = cand;
                }
                f[i] = best;
            }
            cost[s] = f[n];
        }
        free(q);
        free(f);
    }
    free(Dd);
    return 0;
}

/* SAA of fp32 costs (SURVEY §8(c5) fp32 mode): over the finite costs, sequential */
/* fp64 sums, two passes: mean = sum / m, var = sum (c - mean)^2 / (m - 1).       */
/* out: as oracle_saa.                                                             */
int oracle_saa_f32(const float* cost, int64_t S, double* out)
{
    int64_t m = 0, inf = 0;
    double sum = 0.0;
    for (int64_t s = 0; s < S; ++s) {
        if (isinf(cost[s])) { inf++; continue; }
        m++;
        sum += (double)cost[s];
    }
    out[0] = (double)m;
    out[1] = (double)inf;
    if (m == 0) return 3;
    const double mean = sum / (double)m;
    double ss = 0.0;
    for (int64_t s = 0; s < S; ++s)
        if (!isinf(cost[s])) ss += ((double)cost[s] - mean) * ((double)cost[s] - mean);
    out[2] = mean;
    out[3] = m >= 2 ? ss / (double)(m - 1) : 0.0;
    out[4] = sqrt(out[3] / (double)m);
    out[5] = out[2] - 1.96 * out[4];
    out[6] = out[2] + 1.96 * out[4];
    return 0;
}

/* ------------------------------------------------------------------------ */
/* a9/a10. Inventory-routing recourse DP (PAPER:7 names it only; the model   */
/* is SURVEY §8(c6), DESIGN R21).  Per scenario s and customer m:            */
/*   state I in [0,U]; action x in [0, z_{m,t} X] with I + x <= U;           */
/*   I' = max(0, I + x - d);  stage cost c x + h I' + b max(0, d - I - x).   */
/* V_0[I0] = 0, others +inf; V_{t+1}[I'] = min over every (I, x) pair.       */
/* cost_s = sum_m min_I V_H[I].  Every (I, x) pair is enumerated explicitly. */
/* visit: [M][H] u8; cust: [M][6] int32 = {U, X, I0, h, b, c};               */
/* demand: [H][M][ld] u16 (row t*M + m).  cost: [S] int64.                   */
/* ------------------------------------------------------------------------ */
int oracle_irp(int32_t H, int32_t M, const uint8_t* visit, const int32_t* cust,
               const uint16_t* demand, int64_t ld, int64_t S, int64_t* cost, int threads)
{
    if (H < 1 || M < 1 || S < 0 || ld < S) return 2;
    for (int32_t m = 0; m < M; ++m) {
        const int32_t* p = cust + 6 * m;
        if (p[0] < 0 || p[1] < 0 || p[2] < 0 || p[2] > p[0] || p[3] < 0 || p[4] < 0 || p[5] < 0) return 3;
    }
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        int32_t Umax = 0;
        for (int32_t m = 0; m < M; ++m) if (cust[6 * m] > Umax) Umax = cust[6 * m];
        int64_t* V = (int64_t*)malloc(sizeof(int64_t) * (size_t)(Umax + 1));
        int64_t* Vn = (int64_t*)malloc(sizeof(int64_t) * (size_t)(Umax + 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t s = 0; s < S; ++s) {
            int64_t total = 0;
            for (int32_t m = 0; m < M; ++m) {
                const int32_t U = cust[6 * m + 0], X = cust[6 * m + 1], I0 = cust[6 * m + 2];
                const int64_t h = cust[6 * m + 3], b = cust[6 * m + 4], c = cust[6 * m + 5];
                for (int32_t I = 0; I <= U; ++I) V[I] = ORACLE_INF;
                V[I0] = 0;
                for (int32_t t = 0; t < H; ++t) {
                    const int64_t d = demand[((int64_t)t * M + m) * ld + s];
                    const int32_t xmax = visit[(int64_t)m * H + t] ? X : 0;
                    for (int32_t I = 0; I <= U; ++I) Vn[I] = ORACLE_INF;
                    for (int32_t I = 0; I <= U; ++I) {
                        if (V[I] == ORACLE_INF) continue;
                        for (int32_t x = 0; x <= xmax && I + x <= U; ++x) {
                            int64_t y = I + x;
                            int64_t Ip = y - d > 0 ? y - d : 0;
                            int64_t lost = d - y > 0 ? d - y : 0;
                            int64_t v = V[I] + c * x + h * Ip + b * lost;
                            if (v < Vn[Ip]) Vn[Ip] = v;
                        }
                    }
                    for (int32_t I = 0; I <= U; ++I) V[I] = Vn[I];
                }
                int64_t best = ORACLE_INF;
                for (int32_t I = 0; I <= U; ++I) if (V[I] < best) best = V[I];
                total += best;
            }
            cost[s] = total;
        }
        free(V);
        free(Vn);
    }
    return 0;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
