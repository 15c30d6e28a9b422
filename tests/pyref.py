"""Independent pure-Python pins for the oracle (tests only).

Each routine here is a DIFFERENT algorithm from the one in oracle/oracle.c, so
agreement is evidence, not a retyped formula:

* brute_force_split   -- enumerate all 2^(n-1) contiguous partitions of the tour
                         (SPEC:230-238), cost of each route computed from scratch.
* brute_force_penalized -- the same enumeration with lam * max(0, load - Q) per route.
* deque_split         -- O(n) sliding-window-minimum split on the separable form
                         f(i) = B[i] + min_{p in [mask(i), i-1]} (f(p) + A[p])
                         with a monotone deque (Vidal-style linear split).
* two_pointer_mask    -- Eq. (2) by a two-pointer sweep over prefix sums.
* brute_force_irp     -- enumerate every action sequence of the IRP recourse.
"""
from __future__ import annotations

import itertools
import os
from collections import deque

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_golden(name: str) -> dict:
    out = {}
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, _, rest = line.partition(" ")
            if "|" in rest:
                out[key] = [[int(v) for v in part.split()] for part in rest.split("|")]
            else:
                out[key] = [int(v, 16) if name.startswith("philox") else int(v) for v in rest.split()]
    return out


def route_cost(route, dist):
    c = dist[0][route[0]]
    for a, b in zip(route, route[1:]):
        c += dist[a][b]
    return c + dist[route[-1]][0]


def brute_force_penalized(tour, q_tour, dist, Q, lam):
    """Penalized split by enumeration: min over all contiguous partitions of
    sum(route cost + lam * max(0, route load - Q)) (DESIGN R22)."""
    n = len(tour)
    best = None
    for cuts in itertools.product((0, 1), repeat=n - 1):
        routes, start = [], 0
        for k, cut in enumerate(cuts):
            if cut:
                routes.append(list(range(start, k + 1)))
                start = k + 1
        routes.append(list(range(start, n)))
        cost = sum(route_cost([tour[k] for k in r], dist) + lam * max(0, sum(q_tour[k] for k in r) - Q)
                   for r in routes)
        if best is None or cost < best:
            best = cost
    return best


def brute_force_split(tour, q_tour, dist, Q):
    """Min over all contiguous partitions; returns (cost, routes) or (None, None)."""
    n = len(tour)
    best, best_routes = None, None
    for cuts in itertools.product((0, 1), repeat=n - 1):
        routes, start = [], 0
        for k, cut in enumerate(cuts):
            if cut:
                routes.append(list(range(start, k + 1)))
                start = k + 1
        routes.append(list(range(start, n)))
        if any(sum(q_tour[k] for k in r) > Q for r in routes):
            continue
        cost = sum(route_cost([tour[k] for k in r], dist) for r in routes)
        if best is None or cost < best:
            best, best_routes = cost, [[tour[k] for k in r] for r in routes]
    return best, best_routes


def two_pointer_mask(q_tour, Q):
    """mask(i), i = 1..n, by a monotone two-pointer over prefix sums; -1 if q_i > Q."""
    n = len(q_tour)
    P = [0]
    for v in q_tour:
        P.append(P[-1] + v)
    out, lo = [], 0
    for i in range(1, n + 1):
        if q_tour[i - 1] > Q:
            out.append(-1)
            lo = i
            continue
        while P[i] - P[lo] > Q:
            lo += 1
        out.append(lo)
    return out


def deque_split(tour, q_tour, dist, Q):
    """O(n) split: separable route cost t(p,i) = A[p] + B[i] with
    A[p] = c[0][s_{p+1}] - D[p+1], B[i] = D[i] + c[s_i][0] (SPEC:249 prefix form),
    sliding-window minimum over p in [mask(i), i-1] with a monotone deque."""
    n = len(tour)
    s = [0] + list(tour)
    D = [0, 0] + [0] * (n - 1)
    for i in range(2, n + 1):
        D[i] = D[i - 1] + dist[s[i - 1]][s[i]]
    A = [dist[0][s[p + 1]] - D[p + 1] for p in range(n)]
    B = [0] + [D[i] + dist[s[i]][0] for i in range(1, n + 1)]
    masks = two_pointer_mask(q_tour, Q)
    if any(m < 0 for m in masks):
        return None
    f = [0] * (n + 1)
    dq = deque()  # indices p with increasing g(p) = f(p) + A[p]
    for i in range(1, n + 1):
        p_new = i - 1
        g_new = f[p_new] + A[p_new]
        while dq and f[dq[-1]] + A[dq[-1]] >= g_new:
            dq.pop()
        dq.append(p_new)
        while dq[0] < masks[i - 1]:
            dq.popleft()
        f[i] = B[i] + f[dq[0]] + A[dq[0]]
    return f[n]


def brute_force_irp(H, visit_row, params, d_seq):
    """Min total cost over every action sequence x_0..x_{H-1} for one customer.
    params = (U, X, I0, h, b, c); lost-sales dynamics of SURVEY §8(c6)."""
    U, X, I0, h, b, c = params
    ranges = [range(0, (X if visit_row[t] else 0) + 1) for t in range(H)]
    best = None
    for xs in itertools.product(*ranges):
        I, cost, ok = I0, 0, True
        for t in range(H):
            x = xs[t]
            if I + x > U:
                ok = False
                break
            y = I + x
            d = d_seq[t]
            Ip = max(0, y - d)
            cost += c * x + h * Ip + b * max(0, d - y)
            I = Ip
        if ok and (best is None or cost < best):
            best = cost
    return best
