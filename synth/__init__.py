"""Seeded synthetic inputs shared by the tests, bench.py and smoke().

This module holds NONE of the method's arithmetic: it draws X-set-shaped
instances (coordinates, rounded Euclidean cost matrix, nominal demands,
capacity, giant tours, IRP parameters) and turns the demand-model knobs
(cv, rho) into the integer parameters that BOTH the CUDA generator and the
oracle's generator consume.  The recipe is DESIGN.md §"Input recipe"
(SURVEY §8(d)).
"""
from __future__ import annotations

import math

import numpy as np

# Demand-model kinds (mirrors spdp_demand_model.kind).
FIXED, UNIFORM, CORRELATED = 0, 1, 2


def isqrt_round(k: np.ndarray, mode: str) -> np.ndarray:
    """Exact rounding of sqrt(k) for nonnegative integer k.

    nint: floor(sqrt(k) + 1/2) (TSPLIB half-up);
    ceil: ceil(sqrt(k)) (satisfies the triangle inequality, SURVEY finding 5).
    """
    k = np.asarray(k, dtype=np.int64)
    r = np.floor(np.sqrt(k.astype(np.float64))).astype(np.int64)
    # fix the float estimate to the exact integer square root
    r = np.where(r * r > k, r - 1, r)
    r = np.where((r + 1) * (r + 1) <= k, r + 1, r)
    if mode == "nint":
        # sqrt(k) >= r + 1/2  <=>  k >= r^2 + r + 1/4  <=>  k >= r^2 + r + 1
        return np.where(k >= r * r + r + 1, r + 1, r)
    if mode == "ceil":
        return np.where(r * r == k, r, r + 1)
    if mode == "floor":
        return r
    raise ValueError(mode)


def cost_matrix(coords: np.ndarray, rounding: str = "nint") -> np.ndarray:
    """int32 [(n+1) x (n+1)] rounded Euclidean costs, node 0 = depot."""
    xy = np.asarray(coords, dtype=np.int64)
    dx = xy[:, None, 0] - xy[None, :, 0]
    dy = xy[:, None, 1] - xy[None, :, 1]
    return isqrt_round(dx * dx + dy * dy, rounding).astype(np.int32)


def make_instance(n: int, seed: int, r: float = 4.0, mu_lo: int = 1, mu_hi: int = 100,
                  coord_max: int = 1000, rounding: str = "nint", Q: int | None = None) -> dict:
    """X-set-shaped CVRP instance: integer coords on {0..coord_max}^2, depot at a
    random point, nominal demands U{mu_lo..mu_hi}, Q = ceil(r * sum(mu) / n),
    and a seeded random giant tour (a permutation of 1..n)."""
    rng = np.random.default_rng(seed)
    coords = rng.integers(0, coord_max + 1, size=(n + 1, 2), dtype=np.int64)
    nominal = rng.integers(mu_lo, mu_hi + 1, size=n, dtype=np.int64).astype(np.uint16)
    if Q is None:
        Q = int(math.ceil(r * float(nominal.sum()) / n))
    tour = (rng.permutation(n) + 1).astype(np.int32)
    return {"n": n, "coords": coords, "dist": cost_matrix(coords, rounding), "nominal": nominal,
            "Q": int(Q), "tour": tour, "seed": seed, "rounding": rounding}


def demand_model(nominal, Q: int, kind: int = CORRELATED, cv: float = 0.3, rho: float = 0.5,
                 seed: int = 0x5EED0000, stream_tag: int = 0, lo_pm: int = 500, hi_pm: int = 1500,
                 q_cap: int | None = None) -> dict:
    """Integer parameters of the counter-based demand model.

    A_fx = round(rho cv 2^16), B_fx = round(sqrt(1 - rho^2) cv 2^16) are computed
    here once, on the host, and passed as integers to both generators.
    q_cap defaults to min(Q, 65535) so every benchmark scenario is feasible.
    """
    nominal = np.ascontiguousarray(nominal, dtype=np.uint16)
    return {"kind": int(kind), "nominal": nominal, "lo_pm": int(lo_pm), "hi_pm": int(hi_pm),
            "A_fx": int(round(rho * cv * 65536.0)),
            "B_fx": int(round(math.sqrt(max(0.0, 1.0 - rho * rho)) * cv * 65536.0)),
            "q_cap": int(min(Q, 65535) if q_cap is None else q_cap),
            "seed": int(seed), "stream_tag": int(stream_tag)}


def perturb_tours(tour: np.ndarray, T: int, seed: int) -> np.ndarray:
    """T tours: tour 0 as given, tours 1..T-1 = tour 0 + 1..3 seeded relocate / 2-opt
    moves (HGS-offspring-like candidate population, BASELINE configs[2])."""
    rng = np.random.default_rng(seed)
    n = tour.shape[0]
    out = np.empty((T, n), dtype=np.int32)
    out[0] = tour
    for t in range(1, T):
        x = list(int(v) for v in tour)
        for _ in range(int(rng.integers(1, 4))):
            if n < 3:
                break
            if rng.random() < 0.5:  # relocate
                a = int(rng.integers(0, n))
                v = x.pop(a)
                b = int(rng.integers(0, n))
                x.insert(b, v)
            else:  # 2-opt segment reversal
                a, b = sorted(int(v) for v in rng.choice(n, size=2, replace=False))
                x[a:b + 1] = x[a:b + 1][::-1]
        out[t] = np.asarray(x, dtype=np.int32)
    return out


def local_move_tours(tour: np.ndarray, T: int, seed: int, radius: int = 10) -> np.ndarray:
    """T tours: tour 0 as given, tours 1..T-1 = tour 0 + ONE seeded granular move (relocate of a
    customer by at most `radius` positions, or a 2-opt reversal of at most radius + 1 positions),
    the bounded neighbourhoods of HGS local search (f3 workload, DESIGN R23)."""
    rng = np.random.default_rng(seed)
    n = tour.shape[0]
    out = np.empty((T, n), dtype=np.int32)
    out[0] = tour
    for t in range(1, T):
        x = list(int(v) for v in tour)
        if n >= 3:
            a = int(rng.integers(0, n))
            b = int(np.clip(a + rng.integers(-radius, radius + 1), 0, n - 1))
            if rng.random() < 0.5:  # relocate
                v = x.pop(a)
                x.insert(b, v)
            else:  # 2-opt
                lo, hi = min(a, b), max(a, b)
                x[lo:hi + 1] = x[lo:hi + 1][::-1]
        out[t] = np.asarray(x, dtype=np.int32)
    return out


def irp_instance(M: int = 10, H: int = 30, U: int = 100, X: int = 100, I0: int = 50,
                 h: int = 1, b: int = 20, c: int = 1, mu_lo: int = 5, mu_hi: int = 30,
                 seed: int = 105, period: int = 3) -> dict:
    """IRP instance of SURVEY §8(d) C5: z_{m,t} = [(t + m) mod period == 0]."""
    rng = np.random.default_rng(seed)
    mu = rng.integers(mu_lo, mu_hi + 1, size=M, dtype=np.int64).astype(np.uint16)
    visit = np.zeros((M, H), dtype=np.uint8)
    for m in range(M):
        for t in range(H):
            visit[m, t] = 1 if (t + m) % period == 0 else 0
    cust = np.tile(np.array([U, X, I0, h, b, c], dtype=np.int32), (M, 1))
    # demand rows are (t, m) pairs, row t*M + m, nominal mu_m (DESIGN R21)
    nominal_rows = np.tile(mu, H).astype(np.uint16)
    return {"M": M, "H": H, "visit": visit, "cust": cust, "mu": mu, "nominal_rows": nominal_rows}


# BASELINE.json configs.  Seeds: instance 100 + index, Philox key 0x5EED0000 + index.
CONFIGS = {
    "C1": dict(index=0, n=10, S=100, r=None, Q=30, mu_lo=1, mu_hi=10, T=1),
    "C2": dict(index=1, n=100, S=1_000_000, r=4.0, Q=None, mu_lo=1, mu_hi=100, T=1),
    "C3": dict(index=2, n=200, S=100_000, r=8.0, Q=None, mu_lo=1, mu_hi=100, T=256),
    "C4": dict(index=3, n=1000, S=1_000_000, r=23.0, Q=None, mu_lo=1, mu_hi=100, T=1),
}


def config_instance(name: str, S: int | None = None) -> dict:
    """Instance + demand model + tours of one BASELINE config (C1..C4)."""
    cfg = CONFIGS[name]
    inst = make_instance(cfg["n"], 100 + cfg["index"], r=cfg["r"] or 4.0, mu_lo=cfg["mu_lo"],
                         mu_hi=cfg["mu_hi"], Q=cfg["Q"])
    model = demand_model(inst["nominal"], inst["Q"], seed=0x5EED0000 + cfg["index"])
    tours = perturb_tours(inst["tour"], cfg["T"], 200 + cfg["index"]) if cfg["T"] > 1 else inst["tour"][None, :]
    return {"name": name, "inst": inst, "model": model, "tours": tours,
            "S": cfg["S"] if S is None else S, "n": cfg["n"], "Q": inst["Q"], "T": cfg["T"]}


def irp_config(S: int = 100_000) -> dict:
    inst = irp_instance()
    U = int(inst["cust"][0, 0])
    model = demand_model(inst["nominal_rows"], U, seed=0x5EED0000 + 4, q_cap=65535)
    return {"name": "C5", "irp": inst, "model": model, "S": S}


def explicit_demands(rows, S_pad: int | None = None) -> np.ndarray:
    """Hand-made demand matrix: rows = list of per-scenario customer-order vectors.
    Returns u16 [n][ld] (scenario-minor), ld padded to a multiple of 8."""
    a = np.asarray(rows, dtype=np.int64)
    S, n = a.shape
    ld = S if S_pad is None else S_pad
    ld = (ld + 7) // 8 * 8
    out = np.zeros((n, ld), dtype=np.uint16)
    out[:, :S] = a.T
    return out
