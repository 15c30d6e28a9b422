"""Pins for the oracle's split (Eq. 1), mask (Eq. 2) and prefix (PAPER §3).

Everything here is CPU-only (-m "not gpu").  Expected values come from the
paper (tests/golden/*.txt, cited there), brute force, an independent O(n)
algorithm, closed forms and invariants -- never from the oracle itself.
"""
import numpy as np
import pytest

import oracle
import synth
import pyref


def _tour_order_to_customer_rows(tour, q_tour_rows):
    """Scenario vectors given in tour order -> u16 [n][S] rows by customer id."""
    tour = list(tour)
    n = len(tour)
    rows = []
    for q in q_tour_rows:
        cust = [0] * n
        for k, c in enumerate(tour):
            cust[c - 1] = q[k]
        rows.append(cust)
    return synth.explicit_demands(rows)


def _random_case(rng, n, triangle=False, qmax=10, Qlo=5, Qhi=30, S=1):
    if triangle:
        coords = rng.integers(0, 10000, size=(n + 1, 2))
        dist = synth.cost_matrix(coords, "ceil")
    else:
        dist = rng.integers(0, 50, size=(n + 1, n + 1)).astype(np.int32)
        np.fill_diagonal(dist, 0)
    tour = (rng.permutation(n) + 1).astype(np.int32)
    Q = int(rng.integers(Qlo, Qhi + 1))
    q_tour = rng.integers(0, qmax + 1, size=(S, n))
    return tour, dist, Q, q_tour


# ---------------------------------------------------------------- paper pins
def test_example1_masks_and_prefix():
    g = pyref.read_golden("example1.txt")
    tour, Q = g["tour"], g["Q"][0]
    dem = _tour_order_to_customer_rows(tour, [g["scenario1"], g["scenariom"]])
    m = oracle.mask(tour, dem, Q)
    assert m[:, 0].tolist() == g["scenario1_mask"]
    assert m[:, 1].tolist() == g["scenariom_mask"]
    P = oracle.demand_prefix(tour, dem)
    assert P[:, 0].tolist() == g["scenario1_prefix"]


def test_example1_scenario1_routes_forced_under_triangle_inequality():
    """(1),(2),(4,3,5).  Forced for any metric whose depot detours are
    strict (c[a][0] + c[0][b] > c[a][b]); geometries violating strictness are skipped."""
    g = pyref.read_golden("example1.txt")
    tour, Q = g["tour"], g["Q"][0]
    want = g["scenario1_routes"]
    rng = np.random.default_rng(7)
    checked = 0
    for _ in range(200):
        coords = rng.integers(0, 100000, size=(6, 2))
        dist = synth.cost_matrix(coords, "ceil")
        strict = all(dist[a, 0] + dist[0, b] > dist[a, b] for a in range(1, 6) for b in range(1, 6) if a != b)
        if not strict:
            continue
        dem = _tour_order_to_customer_rows(tour, [g["scenario1"]])
        cost, pred = oracle.split(tour, dist, dem, Q, want_pred=True)
        assert oracle.routes_from_pred(pred[0], tour) == want
        bf, bf_routes = pyref.brute_force_split(tour, g["scenario1"], dist.tolist(), Q)
        assert cost[0] == bf and bf_routes == want
        checked += 1
    assert checked > 100


def test_example1_scenario_m_partition_feasible_and_not_better_than_optimum():
    """(1),(2,4,3,5) is feasible (loads 8 and 15 <= 17); several optima may
    exist (DESIGN R3), so assert only that the oracle's optimum is <= its cost."""
    g = pyref.read_golden("example1.txt")
    tour, Q = g["tour"], g["Q"][0]
    rng = np.random.default_rng(11)
    qpos = {c: g["scenariom"][k] for k, c in enumerate(tour)}
    for routes in [g["scenariom_routes"]]:
        assert all(sum(qpos[c] for c in r) <= Q for r in routes)
    for _ in range(50):
        coords = rng.integers(0, 1000, size=(6, 2))
        dist = synth.cost_matrix(coords, "nint")
        dem = _tour_order_to_customer_rows(tour, [g["scenariom"]])
        cost = oracle.split(tour, dist, dem, Q)
        paper_cost = sum(pyref.route_cost(r, dist) for r in g["scenariom_routes"])
        assert cost[0] <= paper_cost


def test_collinear_worked_example():
    g = pyref.read_golden("collinear.txt")
    xs = g["xs"]
    dist = np.abs(np.subtract.outer(xs, xs)).astype(np.int32)
    tour, Q = g["tour"], g["Q"][0]
    dem = _tour_order_to_customer_rows(tour, [g["demand"]])
    cost, pred = oracle.split(tour, dist, dem, Q, want_pred=True)
    assert cost[0] == g["cost"][0]
    assert oracle.routes_from_pred(pred[0], tour) == g["routes"]
    assert oracle.tour_prefix(tour, dist)[1:].tolist() == g["D"]
    assert oracle.split(tour, dist, dem, Q, method="eq1")[0] == g["cost"][0]


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("seed", range(6))
def test_split_matches_brute_force(seed):
    rng = np.random.default_rng(1000 + seed)
    for trial in range(60):
        n = int(rng.integers(1, 10))
        tour, dist, Q, q_tour = _random_case(rng, n, triangle=bool(trial % 2), S=4)
        q_tour[0, rng.integers(0, n)] = Q          # a demand exactly at capacity
        if trial % 7 == 0:
            q_tour[1, rng.integers(0, n)] = Q + 1  # an infeasible scenario
        dem = _tour_order_to_customer_rows(tour, q_tour.tolist())
        scan = oracle.split(tour, dist, dem, Q, S=4)
        eq1 = oracle.split(tour, dist, dem, Q, method="eq1", S=4)
        for s in range(4):
            bf, _ = pyref.brute_force_split(tour.tolist(), q_tour[s].tolist(), dist.tolist(), Q)
            want = oracle.INF if bf is None else bf
            assert scan[s] == want and eq1[s] == want


def test_pred_routes_partition_and_respect_capacity():
    rng = np.random.default_rng(5)
    for _ in range(40):
        n = int(rng.integers(1, 30))
        tour, dist, Q, q_tour = _random_case(rng, n, triangle=True, qmax=12, S=8)
        q_tour = np.minimum(q_tour, Q)
        dem = _tour_order_to_customer_rows(tour, q_tour.tolist())
        cost, pred = oracle.split(tour, dist, dem, Q, want_pred=True)
        qpos = [{c: q_tour[s][k] for k, c in enumerate(tour)} for s in range(8)]
        for s in range(8):
            routes = oracle.routes_from_pred(pred[s], tour)
            assert [c for r in routes for c in r] == tour.tolist()
            assert all(sum(qpos[s][c] for c in r) <= Q for r in routes)
            assert sum(pyref.route_cost(r, dist) for r in routes) == cost[s]


# ---------------------------------------------------------------- independent algorithm
@pytest.mark.parametrize("n", [1, 2, 17, 100, 300])
def test_scan_matches_linear_deque_split(n):
    rng = np.random.default_rng(n)
    inst = synth.make_instance(n, seed=n, r=4.0)
    for kind in (synth.FIXED, synth.CORRELATED):
        model = synth.demand_model(inst["nominal"], inst["Q"], kind=kind, seed=99)
        dem = oracle.gen_demands(model, 0, 24)
        cost = oracle.split(inst["tour"], inst["dist"], dem, inst["Q"])
        for s in range(24):
            q_tour = [int(dem[c - 1, s]) for c in inst["tour"]]
            want = pyref.deque_split(inst["tour"].tolist(), q_tour, inst["dist"].tolist(), inst["Q"])
            assert cost[s] == want
        if kind == synth.FIXED:
            assert np.all(cost == cost[0])  # deterministic model: every scenario = classical split
    del rng


# ---------------------------------------------------------------- closed forms
def test_closed_forms():
    rng = np.random.default_rng(3)
    for _ in range(30):
        n = int(rng.integers(1, 40))
        coords = rng.integers(0, 1000, size=(n + 1, 2))
        dist = synth.cost_matrix(coords, "ceil")
        tour = (rng.permutation(n) + 1).astype(np.int32)
        D = oracle.tour_prefix(tour, dist)
        q = rng.integers(0, 20, size=n)
        # Q >= sum q and triangle inequality -> one route
        Q = int(q.sum()) + 1
        dem = _tour_order_to_customer_rows(tour, [q.tolist()])
        one = int(dist[0, tour[0]] + D[n] + dist[tour[-1], 0])
        assert oracle.split(tour, dist, dem, Q)[0] == one
        # q_k + q_{k+1} > Q for all k (q <= Q) -> all singletons
        Q2 = 10
        q2 = rng.integers(6, 11, size=n)
        dem2 = _tour_order_to_customer_rows(tour, [q2.tolist()])
        single = int(sum(dist[0, c] + dist[c, 0] for c in tour))
        assert oracle.split(tour, dist, dem2, Q2)[0] == single
        # n = 1 is covered by the first form with n = 1; lower bound
        c = oracle.split(tour, dist, _tour_order_to_customer_rows(tour, [np.minimum(q, 9).tolist()]), 9)[0]
        assert c >= dist[0, tour[0]] + dist[tour[-1], 0]


# ---------------------------------------------------------------- invariants
def test_monotone_in_demand_and_capacity():
    rng = np.random.default_rng(21)
    for _ in range(40):
        n = int(rng.integers(2, 25))
        tour, dist, Q, q_tour = _random_case(rng, n, triangle=False, qmax=8, Qlo=8, Qhi=20, S=1)
        q = q_tour[0]
        dem = _tour_order_to_customer_rows(tour, [q.tolist()])
        base = oracle.split(tour, dist, dem, Q)[0]
        k = int(rng.integers(0, n))
        q_up = q.copy()
        q_up[k] += int(rng.integers(1, 4))
        up = oracle.split(tour, dist, _tour_order_to_customer_rows(tour, [q_up.tolist()]), Q)[0]
        assert up >= base                                  # nondecreasing in each demand
        assert oracle.split(tour, dist, dem, Q + 3)[0] <= base  # nonincreasing in Q


def test_prefix_values_nondecreasing_under_triangle_inequality():
    """'V monotone' (BASELINE north_star) holds when c satisfies the triangle
    inequality (ceil rounding; SURVEY finding 5): f(i) <= f(i+1)."""
    rng = np.random.default_rng(8)
    for _ in range(30):
        n = int(rng.integers(2, 30))
        tour, dist, Q, q_tour = _random_case(rng, n, triangle=True, qmax=9, Qlo=10, Qhi=30, S=1)
        q = q_tour[0]
        fs = []
        for i in range(1, n + 1):
            sub_tour = tour[:i]
            # f(i) of the full tour == split cost of the tour prefix sigma_1..sigma_i
            dem = _tour_order_to_customer_rows(np.arange(1, i + 1), [q[:i].tolist()])
            sub = dist[np.ix_([0] + sub_tour.tolist(), [0] + sub_tour.tolist())]
            fs.append(int(oracle.split(np.arange(1, i + 1, dtype=np.int32), sub, dem, Q)[0]))
        assert all(a <= b for a, b in zip(fs, fs[1:]))


def test_mask_definition_two_pointer_and_window_count():
    rng = np.random.default_rng(13)
    for _ in range(30):
        n = int(rng.integers(1, 50))
        tour, dist, Q, q_tour = _random_case(rng, n, qmax=12, Qlo=6, Qhi=40, S=5)
        dem = _tour_order_to_customer_rows(tour, q_tour.tolist())
        m = oracle.mask(tour, dem, Q)
        _, wsum = oracle.split(tour, dist, dem, Q, want_windows=True)
        for s in range(5):
            tp = pyref.two_pointer_mask(q_tour[s].tolist(), Q)
            assert m[:, s].tolist() == tp
            feas = [x for x in tp if x >= 0]
            assert feas == sorted(feas)                       # monotone
            if all(x >= 0 for x in tp):
                assert wsum[s] == sum(i - tp[i - 1] for i in range(1, n + 1))  # Eq. (3) count
    # all fit -> zeros; single demand > Q -> INFEASIBLE
    t = np.array([1, 2, 3], dtype=np.int32)
    assert oracle.mask(t, synth.explicit_demands([[1, 2, 3]]), 17)[:, 0].tolist() == [0, 0, 0]
    assert oracle.mask(t, synth.explicit_demands([[1, 18, 3]]), 17)[:, 0].tolist() == [0, -1, 2]
