"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element.

Bar: bit-exact for the generated demands, masks, prefixes and
every per-scenario cost (integers); SAA sums exact, mean identical.
"""
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


def to_dev(a, dtype=None):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        a = a.view(np.int16)
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def dev_u16(t):
    return t.cpu().numpy().view(np.uint16)


def oracle_cost_as_i32(c):
    c = np.asarray(c)
    return np.where(c == oracle.INF, 2**31 - 1, c).astype(np.int64)


# ------------------------------------------------------------------ a1 generator
@pytest.mark.parametrize("kind", [synth.FIXED, synth.UNIFORM, synth.CORRELATED])
def test_gen_demands_bit_exact(spdp, kind):
    inst = synth.make_instance(100, seed=101)
    model = synth.demand_model(inst["nominal"], inst["Q"], kind=kind, seed=0x5EED0001)
    S = 50_003
    d = spdp.gen_demands(model, 0, S)
    want = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    assert np.array_equal(dev_u16(d)[:, :S], want[:, :S])
    # shard invariance: a rank's slice equals the same columns of the single run
    b, e = 12_345, 40_000
    shard = spdp.gen_demands(model, b, e - b)
    assert np.array_equal(dev_u16(shard)[:, :e - b], want[:, b:e])


# ------------------------------------------------------------------ a3 / a4
def test_prefix_and_mask(spdp):
    inst = synth.make_instance(60, seed=5, r=3.0)
    model = synth.demand_model(inst["nominal"], inst["Q"] + 40, seed=17)  # some q > Q -> INFEASIBLE masks
    S = 3001
    dem = oracle.gen_demands(model, 0, S)
    tour = to_dev(inst["tour"])
    D = to_dev(dem)
    P = spdp.demand_prefix(tour, D).cpu().numpy().astype(np.int64)
    assert np.array_equal(P, oracle.demand_prefix(inst["tour"], dem))
    M = spdp.split_mask(tour, D, inst["Q"]).cpu().numpy()
    assert np.array_equal(M, oracle.mask(inst["tour"], dem, inst["Q"]))


# ------------------------------------------------------------------ a5 / a6 single tour
ALGOS = (None, "int", "f32", "deque", "u16")


def _check_split(spdp, inst, dem, S, hints=(0, 8, 16, 32, 64), Q=None, algos=ALGOS):
    Q = inst["Q"] if Q is None else Q
    want = oracle_cost_as_i32(oracle.split(inst["tour"], inst["dist"], dem, Q, S=S))
    want_saa = oracle.saa(oracle.split(inst["tour"], inst["dist"], dem, Q, S=S))
    tour, dist, D = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem)
    for h in hints:
      for algo in algos:
        cost, part = spdp.split_eval(tour, dist, D, Q, S=S, window_hint=h, validate=(h == 0), algo=algo)
        got = cost.cpu().numpy().astype(np.int64)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, "hint %d algo %s: %d mismatches, first s=%d got %d want %d" % (
            h, algo, bad.size, bad[0], got[bad[0]], want[bad[0]])
        p = part.cpu().numpy()
        assert p[0] == want_saa["m"] and p[1] == want_saa["infeasible"]
        assert p[2] == want_saa["sum"] and (int(p[4]) << 32) + int(p[3]) == want_saa["sumsq"]
        if want_saa["m"] > 0:
            est = spdp.saa_mean(part)
            assert est["mean"] == want_saa["mean"]
            assert est["var"] == pytest.approx(want_saa["var"], rel=1e-12, abs=1e-12)
    return want


def test_split_config1_brute_force(spdp):
    cfg = synth.config_instance("C1")
    inst = cfg["inst"]
    dem = oracle.gen_demands(cfg["model"], 0, 100, ld=104)
    want = _check_split(spdp, inst, dem, 100)
    import pyref
    for s in range(100):
        q_tour = [int(dem[c - 1, s]) for c in inst["tour"]]
        bf, _ = pyref.brute_force_split(inst["tour"].tolist(), q_tour, inst["dist"].tolist(), inst["Q"])
        assert want[s] == bf


@pytest.mark.parametrize("name,S", [("C2", 20_011), ("C3", 3_001), ("C4", 1_203)])
def test_split_configs_multi_tile_ragged(spdp, name, S):
    cfg = synth.config_instance(name)
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    _check_split(spdp, cfg["inst"], dem, S)


def test_split_edge_cases(spdp):
    rng = np.random.default_rng(0)
    # n = 1; zero demands (window = whole tour -> general kernel); q == Q; q > Q (infeasible);
    # Q larger than every load.
    for n in (1, 2, 7, 33, 300):
        inst = synth.make_instance(n, seed=n, r=3.0)
        Q = inst["Q"]
        S = 777
        rows = rng.integers(0, Q + 1, size=(S, n))
        rows[0] = 0
        rows[1] = Q
        rows[2, rng.integers(0, n)] = Q + 1
        rows[3:40] = rng.integers(0, 2, size=(37, n))
        dem = synth.explicit_demands(rows.tolist())
        _check_split(spdp, inst, dem, S, hints=(0, 8, 64))
        _check_split(spdp, inst, dem, S, hints=(16,), Q=2**31 - 1)


def test_split_all_infeasible_partial(spdp):
    inst = synth.make_instance(5, seed=1)
    dem = synth.explicit_demands([[inst["Q"] + 1] * 5] * 9)
    cost, part = spdp.split_eval(to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem), inst["Q"], S=9)
    assert (cost.cpu().numpy() == spdp.INFEASIBLE).all()
    assert part.cpu().numpy()[1] == 9
    with pytest.raises(spdp.SpdpError):
        spdp.saa_mean(part)


# ------------------------------------------------------------------ a8 batched tours
def test_split_batch_tours(spdp):
    inst = synth.make_instance(150, seed=9, r=6.0)
    tours = synth.perturb_tours(inst["tour"], 37, 3)
    model = synth.demand_model(inst["nominal"], inst["Q"], seed=5)
    S = 2_500
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    want = oracle.split_tours(tours, inst["dist"], dem, inst["Q"], S=S)
    for h, algo in ((0, None), (16, "int"), (32, "f32"), (16, "deque"), (8, None)):
        cost, part = spdp.split_eval_batch(to_dev(tours), to_dev(inst["dist"]), to_dev(dem), inst["Q"], S=S,
                                           window_hint=h, algo=algo)
        assert np.array_equal(cost.cpu().numpy().astype(np.int64), oracle_cost_as_i32(want))
        p = part.cpu().numpy()
        for t in range(tours.shape[0]):
            w = oracle.saa(want[t])
            assert p[t, 0] == w["m"] and p[t, 2] == w["sum"] and (int(p[t, 4]) << 32) + int(p[t, 3]) == w["sumsq"]


# ------------------------------------------------------------------ validation / errors
def test_validation_errors(spdp):
    inst = synth.make_instance(10, seed=2)
    dem = to_dev(synth.explicit_demands([[1] * 10] * 8))
    bad_tour = inst["tour"].copy()
    bad_tour[0] = bad_tour[1]
    with pytest.raises(spdp.SpdpError) as e:
        spdp.split_eval(to_dev(bad_tour), to_dev(inst["dist"]), dem, inst["Q"], validate=True)
    assert e.value.status == spdp.SPDP_E_DATA
    with pytest.raises(spdp.SpdpError) as e:
        spdp.split_eval(to_dev(inst["tour"]), to_dev(inst["dist"]), dem, 0)
    assert e.value.status == spdp.SPDP_E_USAGE
    neg = inst["dist"].copy()
    neg[0, inst["tour"][0]] = -1
    with pytest.raises(spdp.SpdpError):
        spdp.split_eval(to_dev(inst["tour"]), to_dev(neg), dem, inst["Q"], validate=True)


# ------------------------------------------------------------------ e2e host path
def test_host_entry_matches_device(spdp):
    cfg = synth.config_instance("C2")
    inst = cfg["inst"]
    S = 10_007
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=S + 5)  # ragged host ld
    want = oracle.split(inst["tour"], inst["dist"], dem, inst["Q"], S=S)
    cost_h = np.zeros(S, dtype=np.int32)
    est = spdp.split_eval_host(inst["tour"], inst["dist"], dem, inst["Q"], S=S, cost_h=cost_h, window_hint=16)
    assert np.array_equal(cost_h.astype(np.int64), oracle_cost_as_i32(want))
    assert est["mean"] == oracle.saa(want)["mean"]


# ------------------------------------------------------------------ a9 / a10 IRP
def test_irp_parity(spdp):
    cfg = synth.irp_config(S=301)
    irp = cfg["irp"]
    H, M = irp["H"], irp["M"]
    dem = oracle.gen_demands(cfg["model"], 0, 301, ld=304)
    want = oracle.irp(H, M, irp["visit"], irp["cust"], dem, S=301)
    cost, part = spdp.irp_dp(irp["visit"], irp["cust"], to_dev(dem), H, M, S=301)
    assert np.array_equal(cost.cpu().numpy(), want)
    assert part.cpu().numpy()[2] == int(want.sum())


def test_irp_state_parallel_kernel(spdp):
    """SPDP_F_IRP_STATES (lanes = inventory states, the "3-D" layout): C5's model on a small S, and
    random prefix-band and general-band customers, against the oracle."""
    cfg = synth.irp_config(S=301)
    irp = cfg["irp"]
    H, M = irp["H"], irp["M"]
    dem = oracle.gen_demands(cfg["model"], 0, 301, ld=304)
    want = oracle.irp(H, M, irp["visit"], irp["cust"], dem, S=301)
    cost, part = spdp.irp_dp(irp["visit"], irp["cust"], to_dev(dem), H, M, S=301, states=True)
    assert np.array_equal(cost.cpu().numpy(), want)
    assert part.cpu().numpy()[2] == int(want.sum())
    rng = np.random.default_rng(31)
    for trial in range(8):
        H, M = int(rng.integers(1, 12)), int(rng.integers(1, 4))
        visit = rng.integers(0, 2, size=(M, H)).astype(np.uint8)
        cust = []
        for _ in range(M):
            U = int(rng.integers(0, 150))
            X = int(rng.integers(0, U + 5)) if trial % 2 else int(rng.integers(U, U + 5))
            cust.append([U, X, int(rng.integers(0, U + 1)), int(rng.integers(0, 4)), int(rng.integers(0, 30)),
                         int(rng.integers(0, 4))])
        cust = np.array(cust, dtype=np.int32)
        dem = rng.integers(0, 60, size=(H * M, 72)).astype(np.uint16)
        want = oracle.irp(H, M, visit, cust, dem, S=67)
        cost, _ = spdp.irp_dp(visit, cust, to_dev(dem), H, M, S=67, states=True, want_partial=False)
        assert np.array_equal(cost.cpu().numpy(), want), "trial %d" % trial


def test_irp_random_small(spdp):
    rng = np.random.default_rng(4)
    for trial in range(12):
        H, M = int(rng.integers(1, 9)), int(rng.integers(1, 4))
        visit = rng.integers(0, 2, size=(M, H)).astype(np.uint8)
        cust = []
        for _ in range(M):
            U = int(rng.integers(0, 200 if trial % 2 else 40))
            X = int(rng.integers(0, U + 5))
            cust.append([U, X, int(rng.integers(0, U + 1)), int(rng.integers(0, 4)), int(rng.integers(0, 30)),
                         int(rng.integers(0, 4))])
        cust = np.array(cust, dtype=np.int32)
        S = 67
        dem = rng.integers(0, 60, size=(H * M, 72)).astype(np.uint16)
        want = oracle.irp(H, M, visit, cust, dem, S=S)
        cost, _ = spdp.irp_dp(visit, cust, to_dev(dem), H, M, S=S)
        assert np.array_equal(cost.cpu().numpy(), want), "trial %d" % trial


# ------------------------------------------------------------------ f1 route recovery
@pytest.mark.parametrize("name,S", [("C1", 100), ("C2", 5_003), ("C3", 777)])
def test_split_routes_pred_exact(spdp, name, S):
    """pred (last split point of every prefix) equals the oracle's, ties -> largest p; the routes
    of the optimal split partition the tour, every route load <= Q, and the route costs add up
    to f(n) (the route cost of Eq. (1) evaluated on the recovered routes)."""
    cfg = synth.config_instance(name)
    inst = cfg["inst"]
    tour = cfg["tours"][0]
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    rng = np.random.default_rng(7)
    scen = np.unique(np.concatenate([rng.integers(0, S, size=64), [0, S - 1]])).astype(np.int64)
    want_cost, want_pred = oracle.split(tour, inst["dist"], dem, inst["Q"], want_pred=True, S=S)
    cost, pred, nr, ml = spdp.split_routes(to_dev(tour), to_dev(inst["dist"]), to_dev(dem), inst["Q"],
                                           torch.from_numpy(scen).cuda(), S=S)
    pred, cost, nr, ml = pred.cpu().numpy(), cost.cpu().numpy(), nr.cpu().numpy(), ml.cpu().numpy()
    assert np.array_equal(cost.astype(np.int64), oracle_cost_as_i32(want_cost[scen]))
    assert np.array_equal(pred, want_pred[scen])
    dist = inst["dist"]
    for k, s in enumerate(scen):
        routes = oracle.routes_from_pred(pred[k], tour)
        assert [c for r in routes for c in r] == [int(c) for c in tour]          # a partition, in tour order
        loads = [sum(int(dem[c - 1, s]) for c in r) for r in routes]
        assert max(loads) <= inst["Q"] and max(loads) == ml[k] and len(routes) == nr[k]
        rc = sum(int(dist[0, r[0]]) + sum(int(dist[a, b]) for a, b in zip(r, r[1:])) + int(dist[r[-1], 0])
                 for r in routes)
        assert rc == cost[k]


def test_split_routes_wide_windows(spdp):
    """The warp route kernel with windows far wider than a warp (Q above the whole tour's load: every
    split point is a candidate of every layer, up to n = 300), plus a collinear instance (many equal
    values: the tie rule -- the largest p -- decides pred)."""
    for n, seed, coll in ((300, 91, False), (150, 92, True)):
        inst = synth.make_instance(n, seed, r=4.0)
        if coll:  # all customers on a line through the depot: many ties among split points
            d = np.abs(np.subtract.outer(np.arange(n + 1), np.arange(n + 1))).astype(np.int32)
            inst = dict(inst, dist=d)
        Q = int(inst["nominal"].astype(np.int64).sum() * 3)
        model = synth.demand_model(inst["nominal"], min(Q, 65535), seed=0x5EED00BB + seed)
        S = 64
        dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
        scen = np.array([0, 7, 31, 63], dtype=np.int64)
        want_cost, want_pred = oracle.split(inst["tour"], inst["dist"], dem, Q, want_pred=True, S=S)
        cost, pred, nr, ml = spdp.split_routes(to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem), Q,
                                               torch.from_numpy(scen).cuda(), S=S)
        assert np.array_equal(cost.cpu().numpy().astype(np.int64), oracle_cost_as_i32(want_cost[scen])), (n, coll)
        assert np.array_equal(pred.cpu().numpy(), want_pred[scen]), (n, coll)


def test_split_routes_large_n_thread_kernel(spdp):
    """n above the warp kernel's shared-memory limit (1024): the thread-per-scenario route kernel;
    pred bit-exact against the oracle (ties -> largest p), route count and max load consistent."""
    inst = synth.make_instance(1100, 77, r=6.0)
    model = synth.demand_model(inst["nominal"], inst["Q"], seed=0x5EED00AA)
    S = 96
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    scen = np.array([0, 5, 17, 42, 95], dtype=np.int64)
    want_cost, want_pred = oracle.split(inst["tour"], inst["dist"], dem, inst["Q"], want_pred=True, S=S)
    cost, pred, nr, ml = spdp.split_routes(to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem), inst["Q"],
                                           torch.from_numpy(scen).cuda(), S=S)
    assert np.array_equal(cost.cpu().numpy().astype(np.int64), oracle_cost_as_i32(want_cost[scen]))
    assert np.array_equal(pred.cpu().numpy(), want_pred[scen])
    for k, s_ in enumerate(scen):
        routes = oracle.routes_from_pred(pred.cpu().numpy()[k], inst["tour"])
        assert len(routes) == int(nr[k].item())
        assert max(sum(int(dem[c - 1, s_]) for c in r) for r in routes) == int(ml[k].item())


def test_split_routes_infeasible(spdp):
    inst = synth.make_instance(6, seed=3)
    Q = inst["Q"]
    rows = [[1] * 6, [Q + 1] + [1] * 5, [1] * 5 + [Q + 1]]
    dem = synth.explicit_demands(rows)
    want_cost, want_pred = oracle.split(inst["tour"], inst["dist"], dem, Q, want_pred=True, S=3)
    cost, pred, nr, _ = spdp.split_routes(to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem), Q,
                                          torch.arange(3, dtype=torch.int64).cuda(), S=3)
    assert np.array_equal(cost.cpu().numpy().astype(np.int64), oracle_cost_as_i32(want_cost))
    assert np.array_equal(pred.cpu().numpy(), want_pred)
    assert list(nr.cpu().numpy()[1:]) == [0, 0]


def test_irp_lazy_shift_prefix_band(spdp):
    """The lazy-shift lane kernel (every customer has X == 0 or X >= U): random parameters,
    demands above U (shift past the whole state space), long horizons without delivery."""
    rng = np.random.default_rng(11)
    for trial in range(10):
        H, M = int(rng.integers(1, 40)), int(rng.integers(1, 4))
        visit = (rng.random((M, H)) < rng.random()).astype(np.uint8)
        cust = []
        for _ in range(M):
            U = int(rng.integers(0, 128))
            X = 0 if rng.random() < 0.15 else int(rng.integers(U, U + 50))
            cust.append([U, X, int(rng.integers(0, U + 1)), int(rng.integers(0, 5)), int(rng.integers(0, 40)),
                         int(rng.integers(0, 5))])
        cust = np.array(cust, dtype=np.int32)
        S = 333
        dem = rng.integers(0, 2 * 128 if trial % 3 == 0 else 40, size=(H * M, 336)).astype(np.uint16)
        want = oracle.irp(H, M, visit, cust, dem, S=S)
        cost, part = spdp.irp_dp(visit, cust, to_dev(dem), H, M, S=S)
        assert np.array_equal(cost.cpu().numpy(), want), "trial %d" % trial
        assert part.cpu().numpy()[2] == int(want.sum())


def test_irp_affine_tail_stress(spdp):
    """The affine-tail representation of the lazy kernel (DESIGN §6 IRP): the explicit region
    shrinks by every period's demand and deliveries extend W affinely above it, so cover slow
    collapse (demands 0..3: deliveries on a nearly full explicit region), fast collapse (demands
    around U), zero costs (c = 0, h = 0 or b = 0), c above b, tiny U, I0 at both ends, and dense
    and sparse visit patterns -- all against the eager oracle DP."""
    rng = np.random.default_rng(23)
    for trial in range(40):
        H, M = int(rng.integers(1, 31)), int(rng.integers(1, 4))
        visit = (rng.random((M, H)) < [0.1, 0.5, 0.9][trial % 3]).astype(np.uint8)
        cust = []
        for _ in range(M):
            U = int(rng.integers(0, 6)) if trial % 5 == 0 else int(rng.integers(1, 120))
            X = 0 if rng.random() < 0.1 else int(rng.integers(U, U + 20))
            I0 = [0, U, int(rng.integers(0, U + 1))][trial % 3]
            c = 0 if trial % 7 == 0 else int(rng.integers(0, 40))
            h = 0 if trial % 4 == 1 else int(rng.integers(0, 6))
            b = 0 if trial % 6 == 2 else int(rng.integers(0, 50))
            cust.append([U, X, I0, h, b, c])
        cust = np.array(cust, dtype=np.int32)
        S = 129
        hi = [4, 40, 130][trial % 3]
        dem = rng.integers(0, hi, size=(H * M, 136)).astype(np.uint16)
        want = oracle.irp(H, M, visit, cust, dem, S=S)
        cost, _ = spdp.irp_dp(visit, cust, to_dev(dem), H, M, S=S, want_partial=False)
        assert np.array_equal(cost.cpu().numpy(), want), "trial %d" % trial


def test_irp_long_horizon(spdp):
    """H above 64 periods: the affine-tail kernel's visit pattern beyond its 64-bit ballot mask (read
    per period), long collapsed phases, and deliveries late in the horizon -- against the oracle."""
    rng = np.random.default_rng(37)
    for trial in range(3):
        H, M = [70, 96, 65][trial], 2
        visit = (rng.random((M, H)) < [0.3, 0.6, 0.9][trial]).astype(np.uint8)
        visit[:, -3:] = 1  # deliveries beyond t = 64
        cust = np.array([[int(rng.integers(1, 60)), 0, 0, 1, 7, 2] for _ in range(M)], dtype=np.int32)
        for m in range(M):
            cust[m, 1] = cust[m, 0] + int(rng.integers(0, 5))  # X >= U: the prefix band
            cust[m, 2] = int(rng.integers(0, cust[m, 0] + 1))
        S = 97
        dem = rng.integers(0, 12, size=(H * M, 104)).astype(np.uint16)
        want = oracle.irp(H, M, visit, cust, dem, S=S)
        cost, _ = spdp.irp_dp(visit, cust, to_dev(dem), H, M, S=S, want_partial=False)
        assert np.array_equal(cost.cpu().numpy(), want), "trial %d" % trial


# ------------------------------------------------------------------ f2 penalized split
@pytest.mark.parametrize("name,S,lam", [("C1", 100, 5), ("C2", 20_011, 10), ("C2", 3_001, 0), ("C3", 2_003, 50),
                                        ("C2", 2_003, 10 ** 6)])
def test_split_penalized_parity(spdp, name, S, lam):
    cfg = synth.config_instance(name)
    inst = cfg["inst"]
    tour = cfg["tours"][0]
    Q = inst["Q"] - inst["Q"] // 4  # tighter than the demand model's clamp: overloaded routes are common
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    want = oracle.split_penalized(tour, inst["dist"], dem, Q, lam, S=S)
    for h in (0, 16, 24):
        cost, part = spdp.split_eval_penalized(to_dev(tour), to_dev(inst["dist"]), to_dev(dem), Q, lam, S=S,
                                               window_hint=h)
        got = cost.cpu().numpy().astype(np.int64)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, "hint %d: %d mismatches, first s=%d got %d want %d" % (
            h, bad.size, bad[0], got[bad[0]], want[bad[0]])
        p = part.cpu().numpy()
        w = oracle.saa(want)
        assert p[0] == S and p[1] == 0 and p[2] == w["sum"] and (int(p[4]) << 32) + int(p[3]) == w["sumsq"]


def test_split_penalized_edge_cases(spdp):
    """Demands above Q (overloaded single customers), zero demands (window = whole tour:
    deferred lanes), lambda large enough to push lanes to the int64 path."""
    rng = np.random.default_rng(3)
    for n in (1, 5, 40, 150):
        inst = synth.make_instance(n, seed=40 + n, r=3.0)
        Q = inst["Q"]
        rows = rng.integers(0, Q + 1, size=(300, n))
        rows[0] = 0
        rows[1] = Q + 5
        rows[2:40] = rng.integers(0, 3, size=(38, n))
        rows[40:60] = rng.integers(Q // 2, 2 * Q, size=(20, n))
        dem = synth.explicit_demands(rows.tolist())
        for lam in (0, 7, 3000):
            want = oracle.split_penalized(inst["tour"], inst["dist"], dem, Q, lam, S=300)
            cost, _ = spdp.split_eval_penalized(to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem), Q, lam, S=300,
                                                window_hint=16)
            assert np.array_equal(cost.cpu().numpy().astype(np.int64), want), (n, lam)


def test_split_f2_large_loads_ring_reset(spdp):
    """Large Q and demands: the packed-fp32 sweep's tile-to-tile prefix restart runs into its exact
    range every few tiles and must clear the ring (p_limit path); costs stay bit-exact."""
    inst = synth.make_instance(60, seed=77, Q=20_000)
    rng = np.random.default_rng(8)
    S = 1_200_003  # ~10 tiles per warp: several restarts and resets per warp
    dem = np.zeros((60, spdp.padded_ld(S)), dtype=np.uint16)
    dem[:, :S] = rng.integers(0, 20_001, size=(60, S), dtype=np.uint16)
    want = oracle_cost_as_i32(oracle.split(inst["tour"], inst["dist"], dem, inst["Q"], S=S))
    for algo, h in ((None, 20), ("f32", 16), ("int", 20)):
        cost, _ = spdp.split_eval(to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem), inst["Q"], S=S,
                                  window_hint=h, algo=algo)
        assert np.array_equal(cost.cpu().numpy().astype(np.int64), want), algo


@pytest.mark.parametrize("hint", [8, 16, 20, 24, 32])
def test_split_wide_first_group_variants(spdp, hint):
    """The mean-window hint (spdp.h SPDP_F_MEAN_WINDOW) selects the sweep variants with a wide
    unconditional candidate group; results are identical for every hint pair."""
    cfg = synth.config_instance("C3")
    inst = cfg["inst"]
    S = 4_099
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    tours = cfg["tours"][:5]
    want = oracle.split_tours(tours, inst["dist"], dem, inst["Q"], S=S)
    for mean in (0, 3, 8, 30):
        cost, _ = spdp.split_eval_batch(to_dev(tours), to_dev(inst["dist"]), to_dev(dem), inst["Q"], S=S,
                                        window_hint=hint, mean_window=mean)
        assert np.array_equal(cost.cpu().numpy().astype(np.int64), oracle_cost_as_i32(want)), (hint, mean)
