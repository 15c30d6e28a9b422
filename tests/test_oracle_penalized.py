"""Pins for the f2 penalized-split oracle (DESIGN R22: every p admissible, lam * max(0, load - Q)
per route).  Each pin is a different computation from oracle_split_penalized."""
import numpy as np
import pytest

import oracle
import synth
import pyref


def _inst(n, seed, rounding="nint"):
    return synth.make_instance(n, seed=seed, r=3.0, rounding=rounding)


@pytest.mark.parametrize("seed", range(6))
def test_penalized_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    for trial in range(20):
        n = int(rng.integers(1, 9))
        inst = _inst(n, 1000 * seed + trial)
        Q = inst["Q"]
        lam = int(rng.choice([0, 1, 3, 17, 1000]))
        rows = rng.integers(0, 2 * Q, size=(4, n))
        dem = synth.explicit_demands(rows.tolist())
        got = oracle.split_penalized(inst["tour"], inst["dist"], dem, Q, lam, S=4)
        for s in range(4):
            q_tour = [int(dem[c - 1, s]) for c in inst["tour"]]
            want = pyref.brute_force_penalized(inst["tour"].tolist(), q_tour, inst["dist"].tolist(), Q, lam)
            assert got[s] == want, (seed, trial, s, lam)


def test_penalized_limits_reduce_to_strict_split():
    """lam = 0: the capacity never binds -> the strict split with Q above every load.
    lam huge: overloading never pays (single-customer routes fit) -> the strict split."""
    cfg = synth.config_instance("C2", S=300)
    inst = cfg["inst"]
    dem = oracle.gen_demands(cfg["model"], 0, 300)
    Q, n = inst["Q"], cfg["n"]
    free = oracle.split(inst["tour"], inst["dist"], dem, n * 65535)
    assert np.array_equal(oracle.split_penalized(inst["tour"], inst["dist"], dem, Q, 0), free)
    strict = oracle.split(inst["tour"], inst["dist"], dem, Q)
    big = 10 ** 9  # > any route-cost difference (costs < 3 n max(dist) << 1e9)
    assert np.array_equal(oracle.split_penalized(inst["tour"], inst["dist"], dem, Q, big), strict)


def test_penalized_monotone_in_lambda_and_single_customer_closed_form():
    cfg = synth.config_instance("C1", S=100)
    inst = cfg["inst"]
    dem = oracle.gen_demands(cfg["model"], 0, 100)
    prev = None
    for lam in (0, 1, 2, 5, 20, 100, 10 ** 6):
        c = oracle.split_penalized(inst["tour"], inst["dist"], dem, inst["Q"], lam)
        if prev is not None:
            assert (c >= prev).all()
        prev = c
    # n = 1: one route, cost c_{0,s1} + c_{s1,0} + lam * max(0, q - Q) (also when q > Q)
    one = _inst(1, 5)
    dem1 = synth.explicit_demands([[0], [one["Q"]], [one["Q"] + 7]])
    d = one["dist"]
    c0 = int(d[0, one["tour"][0]] + d[one["tour"][0], 0])
    got = oracle.split_penalized(one["tour"], d, dem1, one["Q"], 3, S=3)
    assert list(got) == [c0, c0, c0 + 21]


def test_penalized_pred_walk_reproduces_the_cost():
    cfg = synth.config_instance("C1", S=50)
    inst = cfg["inst"]
    Q = inst["Q"] - 10  # some routes overloaded
    dem = oracle.gen_demands(cfg["model"], 0, 50)
    lam = 4
    cost, pred = oracle.split_penalized(inst["tour"], inst["dist"], dem, Q, lam, want_pred=True)
    for s in range(50):
        routes = oracle.routes_from_pred(pred[s], inst["tour"])
        assert [c for r in routes for c in r] == [int(c) for c in inst["tour"]]
        total = sum(pyref.route_cost(r, inst["dist"]) + lam * max(0, sum(int(dem[c - 1, s]) for c in r) - Q)
                    for r in routes)
        assert total == cost[s]
