"""Pins for the oracle's f3 prefix / suffix split values (DESIGN R23) and the
f4 duration- / fleet-limited split (DESIGN R24).  CPU only.

Expected values come from brute force over all contiguous partitions (pure
Python, tests/pyref.py), the reversal symmetry of the split (a different
call path: the forward DP of the reversed tour under the transposed costs),
the concatenation bound and closed forms -- never from the function itself.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth
import pyref

INF = oracle.INF


def _case(rng, n, S, triangle=False, qmax=10, Qlo=8, Qhi=30, sym=True):
    if triangle:
        dist = synth.cost_matrix(rng.integers(0, 10000, size=(n + 1, 2)), "ceil")
    else:
        dist = rng.integers(0, 60, size=(n + 1, n + 1)).astype(np.int32)
        if sym:
            dist = np.minimum(dist, dist.T)
        np.fill_diagonal(dist, 0)
    tour = (rng.permutation(n) + 1).astype(np.int32)
    Q = int(rng.integers(Qlo, Qhi + 1))
    q_tour = rng.integers(0, qmax + 1, size=(S, n))
    dem = np.zeros((n, (S + 7) // 8 * 8), dtype=np.uint16)
    for s in range(S):
        for k, c in enumerate(tour):
            dem[c - 1, s] = q_tour[s, k]
    return tour, np.ascontiguousarray(dist), Q, q_tour, dem


def _bf(tour, q, dist, Q):
    c, _ = pyref.brute_force_split(list(tour), list(q), dist.tolist(), Q)
    return INF if c is None else c


# ---------------------------------------------------------------- f3 values
def test_values_match_brute_force_on_every_prefix_and_suffix():
    rng = np.random.default_rng(31)
    for _ in range(40):
        n = int(rng.integers(1, 9))
        tour, dist, Q, q, dem = _case(rng, n, 3, qmax=12)
        fwd, bwd = oracle.split_values(tour, dist, dem, Q, S=3)
        for s in range(3):
            assert fwd[s, 0] == 0 and bwd[s, n] == 0
            for i in range(1, n + 1):
                assert fwd[s, i] == _bf(tour[:i], q[s, :i], dist, Q)
            for i in range(0, n):
                assert bwd[s, i] == _bf(tour[i:], q[s, i:], dist, Q)


def test_suffix_values_are_the_reversed_tour_prefix_values():
    """b(i) of sigma under c = f(n - i) of reversed sigma under c^T (route costs of a reversed
    route under the transposed matrix are equal term by term; a different computation)."""
    rng = np.random.default_rng(32)
    for _ in range(30):
        n = int(rng.integers(2, 40))
        tour, dist, Q, q, dem = _case(rng, n, 5, sym=False, qmax=10, Qlo=10, Qhi=40)
        fwd, bwd = oracle.split_values(tour, dist, dem, Q, S=5)
        rfwd, rbwd = oracle.split_values(tour[::-1].copy(), np.ascontiguousarray(dist.T), dem, Q, S=5)
        for i in range(n + 1):
            assert np.array_equal(bwd[:, i], rfwd[:, n - i])
            assert np.array_equal(fwd[:, i], rbwd[:, n - i])


def test_concatenation_bound_and_equality_at_optimal_boundaries():
    rng = np.random.default_rng(33)
    for _ in range(30):
        n = int(rng.integers(2, 60))
        tour, dist, Q, q, dem = _case(rng, n, 6, qmax=15, Qlo=15, Qhi=50)
        fwd, bwd = oracle.split_values(tour, dist, dem, Q, S=6)
        cost, pred = oracle.split(tour, dist, dem, Q, want_pred=True, S=6)
        for s in range(6):
            assert fwd[s, n] == cost[s] and bwd[s, 0] == cost[s]
            if cost[s] == INF:
                continue
            tot = fwd[s] + bwd[s]
            assert (tot >= cost[s]).all()
            i = n
            while i > 0:  # every boundary of the optimal split attains the bound
                assert tot[i] == cost[s]
                i = int(pred[s, i])
            assert tot[0] == cost[s]


def test_values_closed_forms_and_infeasible_positions():
    rng = np.random.default_rng(34)
    tour, dist, Q, q, dem = _case(rng, 7, 2, qmax=5, Qlo=20, Qhi=20)
    fwd, bwd = oracle.split_values(tour, dist, dem, Q, S=2)
    last = tour[-1]
    assert (bwd[:, 6] == dist[0, last] + dist[last, 0]).all()
    first = tour[0]
    assert (fwd[:, 1] == dist[0, first] + dist[first, 0]).all()
    # one demand above Q at tour position 4 (1-based): prefixes >= 4 and suffixes < 4 infeasible
    qq = q.copy()
    qq[0, 3] = Q + 1
    dem2 = np.zeros_like(dem)
    for k, c in enumerate(tour):
        dem2[c - 1, :2] = qq[:, k]
    fwd, bwd = oracle.split_values(tour, dist, dem2, Q, S=2)
    assert (fwd[0, 4:] == INF).all() and (fwd[0, :4] != INF).all()
    assert (bwd[0, :4] == INF).all() and (bwd[0, 4:] != INF).all()


# ---------------------------------------------------------------- f4 limits
def _bf_limits(tour, q, dist, Q, Lmax, K):
    n = len(tour)
    best = INF
    for cuts in itertools.product((0, 1), repeat=n - 1):
        routes, start = [], 0
        for k, cut in enumerate(cuts):
            if cut:
                routes.append(list(range(start, k + 1)))
                start = k + 1
        routes.append(list(range(start, n)))
        if K > 0 and len(routes) > K:
            continue
        ok, cost = True, 0
        for r in routes:
            if sum(q[k] for k in r) > Q:
                ok = False
                break
            rc = pyref.route_cost([int(tour[k]) for k in r], dist.tolist())
            if Lmax >= 0 and rc > Lmax:
                ok = False
                break
            cost += rc
        if ok and cost < best:
            best = cost
    return best


def test_limits_match_brute_force():
    rng = np.random.default_rng(41)
    checked = 0
    for _ in range(60):
        n = int(rng.integers(1, 9))
        tour, dist, Q, q, dem = _case(rng, n, 3, qmax=10, sym=bool(rng.integers(0, 2)))
        for Lmax, K in ((-1, 0), (int(rng.integers(20, 200)), 0), (-1, int(rng.integers(1, n + 1))),
                        (int(rng.integers(40, 250)), int(rng.integers(1, n + 1)))):
            got = oracle.split_limits(tour, dist, dem, Q, Lmax=Lmax, K=K, S=3)
            for s in range(3):
                assert got[s] == _bf_limits(tour, q[s], dist, Q, Lmax, K)
                checked += 1
    assert checked == 720


def test_limits_reduce_to_the_plain_split_and_are_monotone():
    rng = np.random.default_rng(42)
    for _ in range(20):
        n = int(rng.integers(3, 50))
        tour, dist, Q, q, dem = _case(rng, n, 8, qmax=12, Qlo=12, Qhi=40)
        plain = oracle.split(tour, dist, dem, Q, S=8)
        assert np.array_equal(oracle.split_limits(tour, dist, dem, Q, S=8), plain)
        assert np.array_equal(oracle.split_limits(tour, dist, dem, Q, K=n, S=8), plain)
        big = int(dist.max()) * (n + 2)
        assert np.array_equal(oracle.split_limits(tour, dist, dem, Q, Lmax=big, S=8), plain)
        prev = None
        for K in range(1, n + 1):  # nonincreasing in K
            c = oracle.split_limits(tour, dist, dem, Q, K=K, S=8)
            if prev is not None:
                assert (c <= prev).all()
            prev = c
        prev = None
        for L in np.linspace(0, big, 7).astype(int):  # nonincreasing in Lmax
            c = oracle.split_limits(tour, dist, dem, Q, Lmax=int(L), S=8)
            assert (c >= plain).all()
            if prev is not None:
                assert (c <= prev).all()
            prev = c


def test_limits_route_counts_and_durations_of_the_returned_path():
    rng = np.random.default_rng(43)
    for _ in range(20):
        n = int(rng.integers(3, 40))
        tour, dist, Q, q, dem = _case(rng, n, 6, triangle=True, qmax=12, Qlo=20, Qhi=60)
        Lmax = int(rng.integers(int(dist[0].max()) * 2, int(dist[0].max()) * 5))
        K = int(rng.integers(1, n + 1))
        cost, pred, kused = oracle.split_limits(tour, dist, dem, Q, Lmax=Lmax, K=K, want_pred=True, S=6)
        for s in range(6):
            if cost[s] == INF:
                assert kused[s] == 0
                continue
            routes = oracle.routes_from_pred(pred[s], tour)
            assert len(routes) == kused[s] <= K
            assert sum(pyref.route_cost(r, dist.tolist()) for r in routes) == cost[s]
            pos = {int(c): k for k, c in enumerate(tour)}
            for r in routes:
                assert pyref.route_cost(r, dist.tolist()) <= Lmax
                assert sum(q[s, pos[c]] for c in r) <= Q


def test_limits_closed_forms():
    rng = np.random.default_rng(44)
    tour, dist, Q, q, dem = _case(rng, 6, 4, triangle=True, qmax=3, Qlo=30, Qhi=30)
    single = int(dist[0, tour[0]]) + sum(int(dist[tour[k], tour[k + 1]]) for k in range(5)) + int(dist[tour[-1], 0])
    # K = 1 and every load fits: the single route (the only 1-route partition)
    assert (oracle.split_limits(tour, dist, dem, Q, K=1, S=4) == single).all()
    # K = 1 with Lmax just below it: infeasible
    assert (oracle.split_limits(tour, dist, dem, Q, K=1, Lmax=single - 1, S=4) == INF).all()
    # Lmax below every out-and-back trip: infeasible; at the largest one: feasible
    trips = [int(dist[0, c] + dist[c, 0]) for c in tour]
    assert (oracle.split_limits(tour, dist, dem, Q, Lmax=min(trips) - 1, S=4) == INF).all()
    assert (oracle.split_limits(tour, dist, dem, Q, Lmax=max(trips), S=4) != INF).all()
