"""Pins for the oracle's fp32 mode (DESIGN R25; SURVEY §8(c3) "fp32 mode") and its SAA.

Expected values: the integer-mode oracle on integer-valued costs (every fp32 value is then an
exact integer below 2^24, so the two modes must agree bit for bit), an fp64 brute force over
all contiguous partitions (pure Python) within the fp32 rounding bound, and exact-Fraction
statistics -- never the function itself.
"""
import itertools
import math
import statistics
from fractions import Fraction

import numpy as np

import oracle
import synth


def _case(rng, n, S, real, qmax=10, Qlo=8, Qhi=30):
    if real:
        xy = rng.uniform(0, 1000, size=(n + 1, 2))
        dist = np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1))
    else:
        dist = rng.integers(0, 60, size=(n + 1, n + 1)).astype(np.float64)
        np.fill_diagonal(dist, 0)
    tour = (rng.permutation(n) + 1).astype(np.int32)
    Q = int(rng.integers(Qlo, Qhi + 1))
    q = rng.integers(0, qmax + 1, size=(S, n))
    dem = np.zeros((n, (S + 7) // 8 * 8), dtype=np.uint16)
    for s in range(S):
        for k, c in enumerate(tour):
            dem[c - 1, s] = q[s, k]
    return tour, np.ascontiguousarray(dist), Q, q, dem


def _bf64(tour, q, dist, Q):
    n = len(tour)
    best = math.inf
    for cuts in itertools.product((0, 1), repeat=n - 1):
        routes, start = [], 0
        for k, cut in enumerate(cuts):
            if cut:
                routes.append(list(range(start, k + 1)))
                start = k + 1
        routes.append(list(range(start, n)))
        if any(sum(q[k] for k in r) > Q for r in routes):
            continue
        cost = 0.0
        for r in routes:
            cost += dist[0, tour[r[0]]] + sum(dist[tour[r[k]], tour[r[k + 1]]] for k in range(len(r) - 1)) \
                + dist[tour[r[-1]], 0]
        best = min(best, cost)
    return best


def test_f32_equals_integer_mode_on_integer_costs():
    rng = np.random.default_rng(51)
    for _ in range(30):
        n = int(rng.integers(1, 60))
        tour, dist, Q, q, dem = _case(rng, n, 16, real=False, qmax=12)
        c32 = oracle.split_f32(tour, dist, dem, Q, S=16)
        ci = oracle.split(tour, dist.astype(np.int32), dem, Q, S=16)
        want = np.where(ci == oracle.INF, np.inf, ci.astype(np.float64))
        assert np.array_equal(c32.astype(np.float64), want)


def test_f32_within_rounding_bound_of_fp64_brute_force():
    """Each route cost is rounded once (rel. error <= 2^-24) and each of the <= n DP adds rounds
    once more, so |c32 - c64| <= 2 n 2^-24 c64 (loose); the value is that of some partition."""
    rng = np.random.default_rng(52)
    checked = 0
    for _ in range(80):
        n = int(rng.integers(1, 10))
        tour, dist, Q, q, dem = _case(rng, n, 3, real=True, qmax=10)
        c32 = oracle.split_f32(tour, dist, dem, Q, S=3)
        for s in range(3):
            c64 = _bf64(tour, q[s], dist, Q)
            if math.isinf(c64):
                assert math.isinf(c32[s])
                continue
            assert abs(float(c32[s]) - c64) <= 2 * n * 2.0 ** -24 * c64 + 1e-9
            checked += 1
    assert checked > 150


def test_f32_closed_forms_and_infeasible():
    rng = np.random.default_rng(53)
    tour, dist, Q, q, dem = _case(rng, 1, 2, real=True)
    c = oracle.split_f32(tour, dist, dem, Q, S=2)
    assert (c == np.float32(np.float32(dist[0, tour[0]] + dist[tour[0], 0]))).all()  # n = 1
    tour, dist, Q, q, dem = _case(rng, 6, 2, real=True, qmax=5, Qlo=10, Qhi=10)
    dem[tour[2] - 1, 0] = Q + 1                                                         # a demand above Q
    c = oracle.split_f32(tour, dist, dem, Q, S=2)
    assert np.isinf(c[0]) and np.isfinite(c[1])


def test_saa_f32_against_exact_fractions():
    rng = np.random.default_rng(54)
    cost = (rng.uniform(1e4, 1e5, size=2001)).astype(np.float32)
    cost[::97] = np.inf
    got = oracle.saa_f32(cost)
    fin = [Fraction(float(v)) for v in cost if np.isfinite(v)]
    mean = sum(fin) / len(fin)
    var = sum((v - mean) ** 2 for v in fin) / (len(fin) - 1)
    assert got["m"] == len(fin) and got["infeasible"] == int(np.isinf(cost).sum())
    assert abs(got["mean"] - float(mean)) <= 1e-12 * float(mean)
    assert abs(got["var"] - float(var)) <= 1e-9 * float(var)
    assert abs(got["stderr"] - math.sqrt(float(var) / len(fin))) <= 1e-9 * got["stderr"]
    # identical costs: variance 0
    assert oracle.saa_f32(np.full(10, 3.5, dtype=np.float32))["var"] == 0.0
    assert statistics.fmean([1.0, 2.0]) == oracle.saa_f32(np.array([1.0, 2.0], dtype=np.float32))["mean"]


def _bf32_leftfold(tour, q, dist, Q):
    """R25 written out over every contiguous partition: each route's cost formed in fp64 from the
    sequential fp64 tour prefix Dd, c_{0,s_{p+1}} + (Dd[i] - Dd[p+1]) + c_{s_i,0} left to right,
    rounded once to fp32; the routes' costs summed left to right in fp32 (one rounding per add);
    the minimum over the capacity-feasible partitions.  Round-to-nearest is monotone, so this
    minimum is EXACTLY the value of the DP min_p fl32(f(p) + T32(p, i)) -- bit for bit."""
    n = len(tour)
    Dd = [0.0] * (n + 1)  # Dd[k], k = 1..n (1-based positions): arcs before position k
    for k in range(2, n + 1):
        Dd[k] = Dd[k - 1] + float(dist[tour[k - 2], tour[k - 1]])
    best = np.float32(np.inf)
    for cuts in itertools.product((0, 1), repeat=n - 1):
        bounds, start = [], 1
        for k, cut in enumerate(cuts, start=1):
            if cut:
                bounds.append((start, k))
                start = k + 1
        bounds.append((start, n))
        if any(sum(q[k - 1] for k in range(a, b + 1)) > Q for a, b in bounds):
            continue
        acc = np.float32(0.0)
        for a, b in bounds:  # route = positions a..b = p + 1..i
            t64 = (float(dist[0, tour[a - 1]]) + (Dd[b] - Dd[a])) + float(dist[tour[b - 1], 0])
            acc = np.float32(acc + np.float32(t64))
        best = min(best, acc)
    return best


def test_f32_bit_exact_against_fp32_left_fold_brute_force():
    rng = np.random.default_rng(55)
    checked = 0
    for _ in range(60):
        n = int(rng.integers(1, 10))
        tour, dist, Q, q, dem = _case(rng, n, 3, real=True, qmax=10)
        c32 = oracle.split_f32(tour, dist, dem, Q, S=3)
        for s in range(3):
            want = _bf32_leftfold(tour, q[s], dist, Q)
            assert np.float32(c32[s]).tobytes() == want.tobytes(), (n, s, c32[s], want)
            checked += np.isfinite(want)
    assert checked > 100
