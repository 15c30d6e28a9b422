"""Pins for the oracle's SAA statistics and IRP DP."""
import math
import statistics
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
import pyref


def test_saa_matches_exact_statistics():
    rng = np.random.default_rng(0)
    for S in (1, 2, 3, 10, 1000):
        c = rng.integers(0, 3_000_000, size=S).astype(np.int64)
        r = oracle.saa(c)
        xs = [int(v) for v in c]
        assert r["m"] == S and r["infeasible"] == 0
        assert r["mean"] == float(Fraction(sum(xs), S))
        if S >= 2:
            v = statistics.variance([Fraction(x) for x in xs])   # exact rational
            assert r["var"] == pytest.approx(float(v), rel=1e-15)
            assert r["stderr"] == pytest.approx(math.sqrt(float(v) / S), rel=1e-14)
        assert r["ci95_lo"] <= r["mean"] <= r["ci95_hi"]


def test_saa_special_cases():
    r = oracle.saa(np.full(100, 4242, dtype=np.int64))
    assert r["mean"] == 4242.0 and r["var"] == 0.0 and r["stderr"] == 0.0
    r = oracle.saa(np.array([8], dtype=np.int64))
    assert r["mean"] == 8.0
    a, b = 1234567, 7654321
    assert oracle.saa(np.array([a, b], dtype=np.int64))["mean"] == (a + b) / 2
    c = np.array([5, oracle.INF, 7, oracle.INF], dtype=np.int64)
    r = oracle.saa(c)
    assert r["m"] == 2 and r["infeasible"] == 2 and r["mean"] == 6.0        # excluded + counted
    assert "mean" not in oracle.saa(np.array([oracle.INF], dtype=np.int64))  # SPEC:287 error
    # concatenation: size-weighted mean, exact
    rng = np.random.default_rng(1)
    x = rng.integers(0, 10**6, size=300)
    y = rng.integers(0, 10**6, size=700)
    rx, ry, rxy = oracle.saa(x), oracle.saa(y), oracle.saa(np.concatenate([x, y]))
    assert rxy["sum"] == rx["sum"] + ry["sum"] and rxy["sumsq"] == rx["sumsq"] + ry["sumsq"]


def _irp_random(rng, H, M):
    visit = rng.integers(0, 2, size=(M, H)).astype(np.uint8)
    cust = []
    for _ in range(M):
        U = int(rng.integers(0, 6))
        cust.append([U, int(rng.integers(0, 5)), int(rng.integers(0, U + 1)), int(rng.integers(0, 4)),
                     int(rng.integers(0, 6)), int(rng.integers(0, 4))])
    return visit, np.array(cust, dtype=np.int32)


def test_irp_matches_brute_force():
    rng = np.random.default_rng(42)
    for _ in range(80):
        H, M, S = int(rng.integers(1, 5)), int(rng.integers(1, 3)), 3
        visit, cust = _irp_random(rng, H, M)
        dem = rng.integers(0, 7, size=(H * M, 8)).astype(np.uint16)
        cost = oracle.irp(H, M, visit, cust, dem, S=S)
        for s in range(S):
            want = 0
            for m in range(M):
                d_seq = [int(dem[t * M + m, s]) for t in range(H)]
                want += pyref.brute_force_irp(H, visit[m].tolist(), cust[m].tolist(), d_seq)
            assert cost[s] == want


def test_irp_closed_forms():
    rng = np.random.default_rng(9)
    for _ in range(30):
        H, M = int(rng.integers(1, 12)), int(rng.integers(1, 4))
        dem = rng.integers(0, 10, size=(H * M, 4)).astype(np.uint16)
        # (1) z == 1, X, U >= max d, I0 = 0, b >= c -> cost = c * sum d (order up to demand)
        c, h, b = int(rng.integers(0, 4)), int(rng.integers(0, 4)), 5
        cust = np.array([[12, 12, 0, h, b, c]] * M, dtype=np.int32)
        cost = oracle.irp(H, M, np.ones((M, H), np.uint8), cust, dem)
        for s in range(4):
            assert cost[s] == c * int(dem[:, s].astype(np.int64).sum())
        # (2) z == 0 -> natural depletion from I0
        I0 = int(rng.integers(0, 12))
        cust0 = np.array([[12, 12, I0, h, b, c]] * M, dtype=np.int32)
        cost0 = oracle.irp(H, M, np.zeros((M, H), np.uint8), cust0, dem)
        for s in range(4):
            want = 0
            for m in range(M):
                inv = I0
                for t in range(H):
                    d = int(dem[t * M + m, s])
                    want += h * max(0, inv - d) + b * max(0, d - inv)
                    inv = max(0, inv - d)
            assert cost0[s] == want


def test_irp_monotone_in_capacity_and_visits():
    rng = np.random.default_rng(17)
    H, M = 6, 2
    dem = rng.integers(0, 15, size=(H * M, 16)).astype(np.uint16)
    visit = rng.integers(0, 2, size=(M, H)).astype(np.uint8)
    base = np.array([[20, 8, 5, 1, 9, 2]] * M, dtype=np.int32)
    c0 = oracle.irp(H, M, visit, base, dem)
    bigger = base.copy(); bigger[:, 0] = 30; bigger[:, 1] = 12
    assert np.all(oracle.irp(H, M, visit, bigger, dem) <= c0)
    assert np.all(oracle.irp(H, M, np.ones_like(visit), base, dem) <= c0)
    pricier = base.copy(); pricier[:, 4] = 15
    assert np.all(oracle.irp(H, M, visit, pricier, dem) >= c0)
