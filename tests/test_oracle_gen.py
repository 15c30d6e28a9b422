"""Pins for the oracle's counter-based scenario generator."""
import math

import numpy as np

import oracle
import synth
import pyref


def test_philox_known_answers():
    g = pyref.read_golden("philox_kat.txt")
    # read_golden keys the lines by their first token; re-read all three rows
    rows = []
    with open(pyref.os.path.join(pyref.GOLDEN, "philox_kat.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                rows.append([int(v, 16) for v in line.split()])
    assert len(rows) == 3 and g
    for r in rows:
        out = oracle.philox4x32_10(r[0:4], r[4:6])
        assert out.tolist() == r[6:10]


def test_fixed_and_zero_cv_give_nominal():
    mu = np.array([5, 17, 100, 0, 65535], dtype=np.uint16)
    for kind, kw in ((synth.FIXED, {}), (synth.CORRELATED, dict(cv=0.0)),
                     (synth.UNIFORM, dict(lo_pm=1000, hi_pm=1000))):
        m = synth.demand_model(mu, 65535, kind=kind, seed=3, **kw)
        d = oracle.gen_demands(m, 0, 50)
        assert np.all(d == mu[:, None])


def test_determinism_and_shard_invariance():
    inst = synth.make_instance(30, seed=4)
    m = synth.demand_model(inst["nominal"], inst["Q"], seed=12345)
    full = oracle.gen_demands(m, 0, 1000)
    assert np.array_equal(full, oracle.gen_demands(m, 0, 1000))
    # shards [0,333), [333,1000) concatenated == single run; any prefix is stable
    a = oracle.gen_demands(m, 0, 333)
    b = oracle.gen_demands(m, 333, 667)
    assert np.array_equal(np.concatenate([a, b], axis=1), full)
    assert np.array_equal(oracle.gen_demands(m, 0, 100), full[:, :100])
    # a different seed or stream tag changes the data
    m2 = dict(m, seed=12346)
    assert not np.array_equal(oracle.gen_demands(m2, 0, 1000), full)
    m3 = dict(m, stream_tag=1)
    assert not np.array_equal(oracle.gen_demands(m3, 0, 1000), full)


def test_uniform_moments():
    """U{lo..hi} with lo = mu/2, hi = 3mu/2: mean (lo+hi)/2 and variance
    ((hi-lo+1)^2 - 1)/12 within 4 standard errors."""
    mu = np.array([100, 40], dtype=np.uint16)
    m = synth.demand_model(mu, 65535, kind=synth.UNIFORM, lo_pm=500, hi_pm=1500, seed=77)
    S = 200_000
    d = oracle.gen_demands(m, 0, S).astype(np.float64)
    for c, v in enumerate(mu):
        lo, hi = int(v) * 500 // 1000, int(v) * 1500 // 1000
        mean = (lo + hi) / 2
        var = ((hi - lo + 1) ** 2 - 1) / 12
        assert abs(d[c].mean() - mean) < 4 * math.sqrt(var / S)
        assert abs(d[c].var() - var) < 0.02 * var
        assert d[c].min() == lo and d[c].max() == hi


def test_correlated_moments():
    """q = mu (1 + cv (rho Z_s + sqrt(1-rho^2) Z_sc)) with Z ~ standardized Irwin-Hall(4):
    mean mu, sd cv mu, and correlation rho^2 between two customers."""
    mu = np.array([1000, 2000, 500], dtype=np.uint16)
    cv, rho = 0.3, 0.5
    m = synth.demand_model(mu, 65535, cv=cv, rho=rho, seed=2024)
    S = 200_000
    d = oracle.gen_demands(m, 0, S).astype(np.float64)
    for c, v in enumerate(mu):
        sd = cv * float(v)
        assert abs(d[c].mean() - float(v)) < 4 * sd / math.sqrt(S) + 0.5
        assert abs(d[c].std() / sd - 1.0) < 0.01
    r = np.corrcoef(d[0], d[1])[0, 1]
    assert abs(r - rho * rho) < 0.01
    # Irwin-Hall(4) is bounded: |Z| <= 131070 / 37837 ~ 3.464 sd, so
    # |q/mu - 1| <= cv (rho + sqrt(1 - rho^2)) 3.464 (+ rounding)
    zmax = cv * (rho + math.sqrt(1 - rho * rho)) * (131070 / 37837)
    assert d[0].max() <= 1000 * (1 + zmax) + 1 and d[0].min() >= 1000 * (1 - zmax) - 1


def test_clamp_to_capacity():
    mu = np.array([100], dtype=np.uint16)
    m = synth.demand_model(mu, 110, cv=0.5, rho=0.0, seed=1)
    d = oracle.gen_demands(m, 0, 10_000)
    assert d.max() == 110 and d.min() >= 0
