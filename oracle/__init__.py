"""CPU oracle for the hot path of arXiv 2511.18022 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product
(``paper_2511_18022_b200``) never imports it and shares no code with it.

``oracle.c`` holds the arithmetic (plain C, integer-exact, each function citing
the passage it follows); this module compiles it with gcc and marshals numpy
arrays through ctypes.  Every function is pinned by ``tests/test_oracle_*.py``
to something other than itself (paper examples, brute force, closed forms,
known-answer vectors, library statistics).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
INF = np.iinfo(np.int64).max

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, OpenMP, no fast-math)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    tmp = _LIB_PATH + ".tmp.%d" % os.getpid()
    cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
           "-o", tmp, _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, u32, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
        lib.oracle_philox4x32_10.argtypes = [P, P, P]
        lib.oracle_gen_demands.argtypes = [i32, P, i32, i32, i32, i64, i64, i32, u64, u32,
                                           i64, i64, P, i64, ctypes.c_int]
        lib.oracle_tour_prefix.argtypes = [i32, P, P, P]
        lib.oracle_demand_prefix.argtypes = [i32, P, P, i64, i64, P]
        lib.oracle_mask.argtypes = [i32, P, P, i64, i64, i32, P]
        lib.oracle_split_batch.argtypes = [i32, P, P, i32, P, i64, i64, i32, P, P, P, ctypes.c_int]
        lib.oracle_split_batch_tours.argtypes = [i32, i32, P, P, i32, P, i64, i64, P, ctypes.c_int]
        lib.oracle_saa.argtypes = [P, i64, P, P]
        lib.oracle_split_penalized.argtypes = [i32, P, P, i32, i64, P, i64, i64, P, P, ctypes.c_int]
        lib.oracle_split_values.argtypes = [i32, P, P, i32, P, i64, i64, P, P, ctypes.c_int]
        lib.oracle_split_limits.argtypes = [i32, P, P, i32, i64, i32, P, i64, i64, P, P, P, ctypes.c_int]
        lib.oracle_split_f32.argtypes = [i32, P, P, i32, P, i64, i64, P, ctypes.c_int]
        lib.oracle_saa_f32.argtypes = [P, i64, P]
        lib.oracle_irp.argtypes = [i32, i32, P, P, P, i64, i64, P, ctypes.c_int]
        for name in ("oracle_gen_demands", "oracle_split_batch", "oracle_split_batch_tours", "oracle_split_penalized",
                     "oracle_split_values", "oracle_split_limits", "oracle_split_f32", "oracle_saa_f32",
                     "oracle_saa", "oracle_irp", "oracle_num_threads"):
            getattr(lib, name).restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(_L().oracle_num_threads())


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    out = np.zeros(4, dtype=np.uint32)
    _L().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def gen_demands(model: dict, s_begin: int, S: int, ld: int | None = None, threads: int = 0) -> np.ndarray:
    """Host twin of the device generator: u16 [n][ld], row c-1 = customer c."""
    nominal = np.ascontiguousarray(model["nominal"], dtype=np.uint16)
    n = nominal.shape[0]
    ld = S if ld is None else ld
    out = np.zeros((n, ld), dtype=np.uint16)
    rc = _L().oracle_gen_demands(int(model["kind"]), _p(nominal), n, int(model.get("lo_pm", 0)),
                                 int(model.get("hi_pm", 0)), int(model.get("A_fx", 0)),
                                 int(model.get("B_fx", 0)), int(model["q_cap"]),
                                 int(model["seed"]), int(model.get("stream_tag", 0)),
                                 int(s_begin), int(S), _p(out), int(ld), int(threads))
    if rc:
        raise ValueError("oracle_gen_demands rc=%d" % rc)
    return out


def tour_prefix(tour, dist) -> np.ndarray:
    tour = np.ascontiguousarray(tour, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=np.int32)
    n = tour.shape[0]
    D = np.zeros(n + 1, dtype=np.int64)
    _L().oracle_tour_prefix(n, _p(tour), _p(dist), _p(D))
    return D


def demand_prefix(tour, demand) -> np.ndarray:
    tour = np.ascontiguousarray(tour, dtype=np.int32)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    n, S = tour.shape[0], demand.shape[1]
    P = np.zeros((n + 1, S), dtype=np.int64)
    _L().oracle_demand_prefix(n, _p(tour), _p(demand), demand.shape[1], S, _p(P))
    return P


def mask(tour, demand, Q) -> np.ndarray:
    """Eq. (2) masks, [n][S] int32, -1 = INFEASIBLE."""
    tour = np.ascontiguousarray(tour, dtype=np.int32)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    n, S = tour.shape[0], demand.shape[1]
    out = np.zeros((n, S), dtype=np.int32)
    _L().oracle_mask(n, _p(tour), _p(demand), demand.shape[1], S, int(Q), _p(out))
    return out


def split(tour, dist, demand, Q, method: str = "scan", want_pred: bool = False,
          want_windows: bool = False, S: int | None = None, threads: int = 0):
    """Per-scenario split cost (int64, INF = infeasible) for demand u16 [n][ld].

    method "scan" = Eq. (1) descending scan with exact capacity break;
    method "eq1"  = Eq. (1) literally with every segment recomputed (small n).
    Only the first S columns (default: all) are evaluated.
    """
    tour = np.ascontiguousarray(tour, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=np.int32)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    n = tour.shape[0]
    ld = demand.shape[1]
    S = ld if S is None else S
    cost = np.zeros(S, dtype=np.int64)
    pred = np.zeros((S, n + 1), dtype=np.int32) if want_pred else None
    wsum = np.zeros(S, dtype=np.int64) if want_windows else None
    rc = _L().oracle_split_batch(n, _p(tour), _p(dist), int(Q), _p(demand), ld, int(S),
                                 1 if method == "eq1" else 0, _p(cost),
                                 _p(pred) if pred is not None else None,
                                 _p(wsum) if wsum is not None else None, int(threads))
    if rc:
        raise ValueError("oracle_split_batch rc=%d" % rc)
    out = [cost]
    if want_pred:
        out.append(pred)
    if want_windows:
        out.append(wsum)
    return out[0] if len(out) == 1 else tuple(out)


def split_penalized(tour, dist, demand, Q, lam: int, want_pred: bool = False, S: int | None = None,
                    threads: int = 0):
    """f2 penalized split (DESIGN R22): every p admissible, lam * max(0, load - Q) added.
    int64 [S] costs (and [S][n+1] predecessors, ties -> largest p)."""
    tour = np.ascontiguousarray(tour, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=np.int32)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    n = tour.shape[0]
    ld = demand.shape[1]
    S = ld if S is None else S
    cost = np.zeros(S, dtype=np.int64)
    pred = np.zeros((S, n + 1), dtype=np.int32) if want_pred else None
    rc = _L().oracle_split_penalized(n, _p(tour), _p(dist), int(Q), int(lam), _p(demand), ld, int(S), _p(cost),
                                     _p(pred) if pred is not None else None, int(threads))
    if rc:
        raise ValueError("oracle_split_penalized rc=%d" % rc)
    return (cost, pred) if want_pred else cost


def split_values(tour, dist, demand, Q, S: int | None = None, threads: int = 0):
    """f3 (DESIGN R23): prefix / suffix split values, int64 [S][n+1] each (INF = infeasible):
    fwd[s][i] = Split of sigma_1..sigma_i, bwd[s][i] = Split of sigma_{i+1}..sigma_n."""
    tour = np.ascontiguousarray(tour, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=np.int32)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    n = tour.shape[0]
    ld = demand.shape[1]
    S = ld if S is None else S
    fwd = np.zeros((S, n + 1), dtype=np.int64)
    bwd = np.zeros((S, n + 1), dtype=np.int64)
    rc = _L().oracle_split_values(n, _p(tour), _p(dist), int(Q), _p(demand), ld, int(S), _p(fwd), _p(bwd),
                                  int(threads))
    if rc:
        raise ValueError("oracle_split_values rc=%d" % rc)
    return fwd, bwd


def split_limits(tour, dist, demand, Q, Lmax: int = -1, K: int = 0, want_pred: bool = False,
                 S: int | None = None, threads: int = 0):
    """f4 (DESIGN R24): split with route duration t(p,i) <= Lmax (Lmax < 0: none) and at most
    K routes (K <= 0: none).  int64 [S] costs (INF = infeasible), optionally the optimum's
    predecessors [S][n+1] (-1 off the path) and route counts [S]."""
    tour = np.ascontiguousarray(tour, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=np.int32)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    n = tour.shape[0]
    ld = demand.shape[1]
    S = ld if S is None else S
    cost = np.zeros(S, dtype=np.int64)
    pred = np.zeros((S, n + 1), dtype=np.int32) if want_pred else None
    kused = np.zeros(S, dtype=np.int32) if want_pred else None
    rc = _L().oracle_split_limits(n, _p(tour), _p(dist), int(Q), int(Lmax), int(K), _p(demand), ld, int(S),
                                  _p(cost), _p(pred) if want_pred else None, _p(kused) if want_pred else None,
                                  int(threads))
    if rc:
        raise ValueError("oracle_split_limits rc=%d" % rc)
    return (cost, pred, kused) if want_pred else cost


def split_f32(tour, dist, demand, Q, S: int | None = None, threads: int = 0) -> np.ndarray:
    """a5 fp32 mode (DESIGN R25): real-valued costs dist (fp64 [(n+1)^2]); float32 [S] costs
    (+inf = infeasible), each candidate one fp32 add of the route cost rounded once from fp64."""
    tour = np.ascontiguousarray(tour, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=np.float64)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    n = tour.shape[0]
    ld = demand.shape[1]
    S = ld if S is None else S
    cost = np.zeros(S, dtype=np.float32)
    rc = _L().oracle_split_f32(n, _p(tour), _p(dist), int(Q), _p(demand), ld, int(S), _p(cost), int(threads))
    if rc:
        raise ValueError("oracle_split_f32 rc=%d" % rc)
    return cost


def saa_f32(cost) -> dict:
    """SAA of float32 costs: sequential fp64 sums, two-pass variance."""
    cost = np.ascontiguousarray(cost, dtype=np.float32)
    out = np.zeros(7, dtype=np.float64)
    rc = _L().oracle_saa_f32(_p(cost), cost.shape[0], _p(out))
    if rc == 3:
        raise ValueError("all scenarios infeasible (SPEC:287)")
    return {"m": int(out[0]), "infeasible": int(out[1]), "mean": out[2], "var": out[3], "stderr": out[4],
            "ci95_lo": out[5], "ci95_hi": out[6]}


def split_tours(tours, dist, demand, Q, S: int | None = None, threads: int = 0) -> np.ndarray:
    tours = np.ascontiguousarray(tours, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=np.int32)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    T, n = tours.shape
    ld = demand.shape[1]
    S = ld if S is None else S
    cost = np.zeros((T, S), dtype=np.int64)
    rc = _L().oracle_split_batch_tours(n, T, _p(tours), _p(dist), int(Q), _p(demand), ld, int(S),
                                       _p(cost), int(threads))
    if rc:
        raise ValueError("oracle_split_batch_tours rc=%d" % rc)
    return cost


def routes_from_pred(pred_row, tour):
    """Walk predecessors from n back to 0 -> list of routes (customer ids)."""
    n = len(tour)
    out = []
    i = n
    while i > 0:
        p = int(pred_row[i])
        if p < 0 or p >= i:
            raise ValueError("corrupt predecessor chain")
        out.append([int(c) for c in tour[p:i]])
        i = p
    return out[::-1]


def saa(cost) -> dict:
    """SAA statistics over feasible scenarios (exact sums)."""
    cost = np.ascontiguousarray(cost, dtype=np.int64)
    out = np.zeros(7, dtype=np.float64)
    sums = np.zeros(4, dtype=np.uint64)
    rc = _L().oracle_saa(_p(cost), cost.shape[0], _p(out), _p(sums))
    s = int(sums[0]) | (int(sums[1]) << 64)
    if s >= 1 << 127:
        s -= 1 << 128
    sq = int(sums[2]) | (int(sums[3]) << 64)
    res = {"m": int(out[0]), "infeasible": int(out[1]), "sum": s, "sumsq": sq}
    if rc == 0:
        res.update(mean=float(out[2]), var=float(out[3]), stderr=float(out[4]),
                   ci95_lo=float(out[5]), ci95_hi=float(out[6]))
    return res


def irp(H, M, visit, cust, demand, S: int | None = None, threads: int = 0) -> np.ndarray:
    """IRP recourse cost per scenario; explicit (I, x) DP."""
    visit = np.ascontiguousarray(visit, dtype=np.uint8)
    cust = np.ascontiguousarray(cust, dtype=np.int32)
    demand = np.ascontiguousarray(demand, dtype=np.uint16)
    ld = demand.shape[1]
    S = ld if S is None else S
    cost = np.zeros(S, dtype=np.int64)
    rc = _L().oracle_irp(int(H), int(M), _p(visit), _p(cust), _p(demand), ld, int(S), _p(cost),
                         int(threads))
    if rc:
        raise ValueError("oracle_irp rc=%d" % rc)
    return cost
