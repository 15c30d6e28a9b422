"""GPU parity of f4 (DESIGN R24): the split with a route-duration limit and a fleet
limit, vs the CPU oracle, element by element (bit-exact int32 costs, exact SAA sums),
through both scratch placements of the kernel."""
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


def _partial_expect(costs):
    feas = [int(v) for v in costs if v != 2**31 - 1]
    sq = [v * v for v in feas]
    return (len(feas), len(costs) - len(feas), sum(feas), sum(v & 0xffffffff for v in sq), sum(v >> 32 for v in sq))


def _limits(inst, dem, frac_routes):
    """Duration limits around the largest out-and-back trip; fleet limits around the
    capacity bound ceil(sum q / Q) of the nominal demands."""
    d, t = inst["dist"], inst["tour"]
    trip = int(max(d[0, c] + d[c, 0] for c in t))
    kmin = int(np.ceil(inst["nominal"].astype(np.int64).sum() / inst["Q"]))
    # kmin + 6: slack spread over the ring passes' band widths 2 / 4 / 8 / 16; kmin + 20: slack 16..31,
    # the warp-per-scenario kernel; kmin + 40: slack >= 32, the general kernel
    return [(-1, 0), (trip, 0), (int(trip * 1.5), 0), (-1, kmin + frac_routes), (-1, 1),
            (int(trip * 1.5), kmin + 2 * frac_routes), (-1, kmin + 6), (-1, kmin + 20), (int(trip * 1.5), kmin + 20),
            (-1, kmin + 40)]


@pytest.mark.parametrize("name,S,extra_q,glob", [("C1", 100, 0, False), ("C1", 100, 0, True), ("C2", 2_003, 0, False),
                                                 ("C2", 1_001, 30, True), ("C3", 301, 0, False)])
def test_limits_parity(spdp, name, S, extra_q, glob):
    cfg = synth.config_instance(name, S=S)
    inst = cfg["inst"]
    model = dict(cfg["model"])
    model["q_cap"] = int(min(cfg["Q"] + extra_q, 65535))
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    tour, dist, D = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem)
    for Lmax, K in _limits(inst, dem, 1):
        cost, part = spdp.split_eval_limits(tour, dist, D, cfg["Q"], max_duration=Lmax, max_routes=K, S=S,
                                            scratch_global=glob)
        want = as_i32(oracle.split_limits(inst["tour"], inst["dist"], dem, cfg["Q"], Lmax=Lmax, K=K, S=S))
        got = cost.cpu().numpy().astype(np.int64)
        assert np.array_equal(got, want), (Lmax, K)
        assert tuple(int(v) for v in part.cpu().numpy()[:5]) == _partial_expect(want)


def test_limits_without_limits_equal_split(spdp):
    """No limits: the same costs as spdp_split_eval (n = 1000, the workspace-scratch path)."""
    cfg = synth.config_instance("C4", S=517)
    inst, S = cfg["inst"], 517
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    tour, dist, D = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem)
    cost, _ = spdp.split_eval_limits(tour, dist, D, cfg["Q"], S=S)
    ref, _ = spdp.split_eval(tour, dist, D, cfg["Q"], S=S, window_hint=64)
    assert torch.equal(cost, ref)
    kmin = int(np.ceil(inst["nominal"].astype(np.int64).sum() / inst["Q"]))
    cost, _ = spdp.split_eval_limits(tour, dist, D, cfg["Q"], max_routes=kmin + 1, S=S)
    want = as_i32(oracle.split_limits(inst["tour"], inst["dist"], dem, cfg["Q"], K=kmin + 1, S=S))
    assert np.array_equal(cost.cpu().numpy().astype(np.int64), want)


def test_limits_edge_cases(spdp):
    # n = 1; a demand above Q; a duration below every trip
    dist = np.array([[0, 7], [9, 0]], dtype=np.int32)
    dem = synth.explicit_demands([[3], [5], [6]])
    for Lmax, K, want in ((-1, 0, [16, 16, 2**31 - 1]), (15, 0, [2**31 - 1] * 3), (16, 1, [16, 16, 2**31 - 1])):
        cost, part = spdp.split_eval_limits(to_dev(np.array([1], dtype=np.int32)), to_dev(dist), to_dev(dem), 5,
                                            max_duration=Lmax, max_routes=K, S=3)
        assert cost.cpu().tolist() == want


@pytest.mark.parametrize("n,S", [(1, 1), (2, 9), (5, 130), (40, 3)])
def test_limits_tiny(spdp, n, S):
    inst = synth.make_instance(n, seed=55 + n, r=2.0)
    model = synth.demand_model(inst["nominal"], inst["Q"], seed=98)
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    tour, dist, D = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem)
    trip = int(max(inst["dist"][0, c] + inst["dist"][c, 0] for c in inst["tour"]))
    for Lmax, K in ((-1, 0), (trip, 0), (-1, 1), (-1, max(1, n // 2)), (2 * trip, max(1, n // 3))):
        for g in (False, True):
            cost, _ = spdp.split_eval_limits(tour, dist, D, inst["Q"], max_duration=Lmax, max_routes=K, S=S,
                                             scratch_global=g)
            want = as_i32(oracle.split_limits(inst["tour"], inst["dist"], dem, inst["Q"], Lmax=Lmax, K=K, S=S))
            assert np.array_equal(cost.cpu().numpy().astype(np.int64), want), (Lmax, K, g)


def test_limits_large_n_table_in_global_memory(spdp):
    """n above the shared-memory table size (the position table read through L1)."""
    n, S = 2600, 17
    inst = synth.make_instance(n, seed=2600, r=12.0)
    model = synth.demand_model(inst["nominal"], inst["Q"], seed=97)
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    tour, dist, D = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem)
    kmin = int(np.ceil(inst["nominal"].astype(np.int64).sum() / inst["Q"]))
    trip = int(max(inst["dist"][0, c] + inst["dist"][c, 0] for c in inst["tour"]))
    for Lmax, K in ((-1, 0), (2 * trip, 0), (-1, kmin + 2)):
        for g in (False, True):
            cost, _ = spdp.split_eval_limits(tour, dist, D, inst["Q"], max_duration=Lmax, max_routes=K, S=S,
                                             scratch_global=g)
            want = as_i32(oracle.split_limits(inst["tour"], inst["dist"], dem, inst["Q"], Lmax=Lmax, K=K, S=S))
            assert np.array_equal(cost.cpu().numpy().astype(np.int64), want), (Lmax, K, g)
