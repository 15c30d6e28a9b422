"""Randomized GPU parity sweep: many small random instances (n = 1..60, random Q, demands with
zeros, ties, values equal to Q and above it, asymmetric integer costs) through every entry point,
element by element against the CPU oracle."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def spdp():
    import paper_2511_18022_b200 as m
    return m


def to_dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        a = a.view(np.int16)
    return torch.from_numpy(a).cuda()


def as_i32(c):
    c = np.asarray(c)
    return np.where(c == oracle.INF, 2**31 - 1, c).astype(np.int64)


def _instance(rng):
    n = int(rng.integers(1, 61))
    S = int(rng.integers(1, 300))
    Q = int(rng.integers(1, 60))
    dist = rng.integers(0, 200, size=(n + 1, n + 1)).astype(np.int32)
    np.fill_diagonal(dist, 0)
    tour = (rng.permutation(n) + 1).astype(np.int32)
    q = rng.integers(0, max(2, Q // 2), size=(n, S))
    q[rng.random((n, S)) < 0.05] = Q                               # loads that exactly fill a route
    q[:, rng.random(S) < 0.03] = 0                                 # all-zero scenarios
    bad = rng.random(S) < 0.04
    q[rng.integers(0, n), bad] = Q + 1 + rng.integers(0, 5)        # infeasible scenarios
    dem = np.zeros((n, (S + 7) // 8 * 8), dtype=np.uint16)
    dem[:, :S] = np.minimum(q, 65535)
    return n, S, Q, dist, tour, dem


@pytest.mark.parametrize("seed", range(12))
def test_random_instances_every_entry_point(spdp, seed):
    rng = np.random.default_rng(9000 + seed)
    n, S, Q, dist, tour, dem = _instance(rng)
    T, D, dd = to_dev(tour), to_dev(dem), to_dev(dist)
    want = as_i32(oracle.split(tour, dist, dem, Q, S=S))
    for algo in (None, "int", "f32", "deque", "u16"):
        for hint in (0, 8, 20, 32, 64):
            cost, _ = spdp.split_eval(T, dd, D, Q, S=S, window_hint=hint, algo=algo)
            assert np.array_equal(cost.cpu().numpy().astype(np.int64), want), (algo, hint)
    # batched tours and the f3 neighbour evaluation from tour 0's values
    tours = np.ascontiguousarray(np.stack([tour] + [(rng.permutation(n) + 1).astype(np.int32) for _ in range(3)]
                                          + list(synth.perturb_tours(tour, 4, seed)[1:])))
    wt = as_i32(oracle.split_tours(tours, dist, dem, Q, S=S))
    bc, _ = spdp.split_eval_batch(to_dev(tours), dd, D, Q, S=S, window_hint=20)
    assert np.array_equal(bc.cpu().numpy().astype(np.int64), wt)
    fwd, bwd = spdp.split_values(T, dd, D, Q, S=S)
    wf, wb = oracle.split_values(tour, dist, dem, Q, S=S)
    assert np.array_equal(fwd.cpu().numpy().T.astype(np.int64), as_i32(wf))
    assert np.array_equal(bwd.cpu().numpy().T.astype(np.int64), as_i32(wb))
    for smem, io in ((False, False), (False, True), (True, False)):
        nc, _ = spdp.split_eval_neighbours(T, fwd, bwd, to_dev(tours), dd, D, Q, S=S, window_hint=16, smem=smem,
                                           int_only=io)
        assert np.array_equal(nc.cpu().numpy().astype(np.int64), wt), (smem, io)
    # f2 penalized, f4 limits, fp32 mode
    lam = int(rng.integers(0, 30))
    pc, _ = spdp.split_eval_penalized(T, dd, D, Q, lam, S=S)
    assert np.array_equal(pc.cpu().numpy().astype(np.int64), oracle.split_penalized(tour, dist, dem, Q, lam, S=S))
    trip = int(max(dist[0, c] + dist[c, 0] for c in tour))
    for Lmax, K in ((-1, 0), (trip + int(rng.integers(0, 300)), 0), (-1, int(rng.integers(1, n + 1))),
                    (2 * trip, int(rng.integers(1, n + 1)))):
        for g in (False, True):
            lc, _ = spdp.split_eval_limits(T, dd, D, Q, max_duration=Lmax, max_routes=K, S=S, scratch_global=g)
            wl = as_i32(oracle.split_limits(tour, dist, dem, Q, Lmax=Lmax, K=K, S=S))
            assert np.array_equal(lc.cpu().numpy().astype(np.int64), wl), (Lmax, K, g)
    distf = dist.astype(np.float64) + rng.random(dist.shape)
    np.fill_diagonal(distf, 0.0)
    c32 = spdp.split_eval_f32(T, to_dev(distf), D, Q, S=S).cpu().numpy()
    assert np.array_equal(c32.view(np.uint32), oracle.split_f32(tour, distf, dem, Q, S=S).view(np.uint32))
