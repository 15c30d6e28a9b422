"""GPU parity of f3 (DESIGN R23): prefix / suffix split values and the neighbourhood
evaluation of candidate tours from a parent's values, vs the CPU oracle, element by
element (bit-exact int32 costs, exact SAA sums)."""
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
    feas = costs[costs != 2**31 - 1].astype(object)
    sq = [int(v) * int(v) for v in feas]
    return (len(feas), int((costs == 2**31 - 1).sum()), int(sum(feas)),
            sum(v & 0xffffffff for v in sq), sum(v >> 32 for v in sq))


@pytest.mark.parametrize("name,S,extra_q", [("C1", 100, 0), ("C2", 2_003, 0), ("C2", 1_001, 40), ("C3", 301, 0)])
def test_split_values_parity(spdp, name, S, extra_q):
    cfg = synth.config_instance(name, S=S)
    inst = cfg["inst"]
    model = dict(cfg["model"])
    model["q_cap"] = int(min(cfg["Q"] + extra_q, 65535))  # extra_q > 0: some scenarios infeasible
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    fwd, bwd = spdp.split_values(to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem), cfg["Q"], S=S)
    wf, wb = oracle.split_values(inst["tour"], inst["dist"], dem, cfg["Q"], S=S)
    assert np.array_equal(fwd.cpu().numpy().T.astype(np.int64), as_i32(wf))
    assert np.array_equal(bwd.cpu().numpy().T.astype(np.int64), as_i32(wb))


def _candidates(tour, T, seed):
    """perturbed tours + the edge cases: the parent itself, a change at the first / last
    position only, the full reversal (prefix 0, suffix 0) and a random permutation."""
    n = len(tour)
    out = list(synth.perturb_tours(tour, max(T - 5, 1), seed))
    rng = np.random.default_rng(seed)
    out.append(tour.copy())
    if n >= 2:
        x = tour.copy()
        x[0], x[1] = x[1], x[0]
        out.append(x)
        y = tour.copy()
        y[-1], y[-2] = y[-2], y[-1]
        out.append(y)
    out.append(tour[::-1].copy())
    out.append((rng.permutation(n) + 1).astype(np.int32))
    return np.ascontiguousarray(np.stack(out), dtype=np.int32)


@pytest.mark.parametrize("smem,int_only", [(False, False), (False, True), (True, False)])
@pytest.mark.parametrize("name,S,T,hint,extra_q", [
    ("C1", 100, 24, 0, 0), ("C2", 3_001, 40, 16, 0), ("C2", 2_003, 30, 24, 30), ("C3", 1_001, 40, 32, 0),
    ("C3", 777, 20, 16, 0), ("C4", 203, 12, 16, 0), ("C4", 203, 12, 32, 0), ("C4", 203, 12, 64, 0)])
def test_neighbours_parity(spdp, name, S, T, hint, extra_q, smem, int_only):
    """Bit-exact vs the oracle's split of every candidate (C4 with a 16-entry ring sends most
    lanes through the overflow path)."""
    cfg = synth.config_instance(name, S=S)
    inst = cfg["inst"]
    model = dict(cfg["model"])
    model["q_cap"] = int(min(cfg["Q"] + extra_q, 65535))
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    tours = _candidates(inst["tour"], T, 300 + T)
    parent, dist, D = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem)
    fwd, bwd = spdp.split_values(parent, dist, D, cfg["Q"], S=S)
    cost, part = spdp.split_eval_neighbours(parent, fwd, bwd, to_dev(tours), dist, D, cfg["Q"], S=S,
                                            window_hint=hint, validate=True, smem=smem, int_only=int_only)
    want = as_i32(oracle.split_tours(tours, inst["dist"], dem, cfg["Q"], S=S))
    got = cost.cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want)
    p = part.cpu().numpy()
    for t in range(tours.shape[0]):
        assert tuple(int(v) for v in p[t, :5]) == _partial_expect(want[t])


def test_neighbours_match_batch_at_full_C3(spdp):
    """At BASELINE configs[2] (256 tours x 10^5 scenarios, n = 200): identical to the batched
    sweep for every (tour, scenario), and to the oracle on a sample of scenarios."""
    cfg = synth.config_instance("C3")
    inst, S = cfg["inst"], cfg["S"]
    D = spdp.gen_demands(cfg["model"], 0, S)
    tours = to_dev(cfg["tours"])
    parent, dist = to_dev(inst["tour"]), to_dev(inst["dist"])
    fwd, bwd = spdp.split_values(parent, dist, D, cfg["Q"], S=S)
    cost, part = spdp.split_eval_neighbours(parent, fwd, bwd, tours, dist, D, cfg["Q"], S=S, window_hint=20)
    bcost, bpart = spdp.split_eval_batch(tours, dist, D, cfg["Q"], S=S, window_hint=24)
    assert torch.equal(cost, bcost)
    assert torch.equal(part, bpart)
    icost, ipart = spdp.split_eval_neighbours(parent, fwd, bwd, tours, dist, D, cfg["Q"], S=S, window_hint=20,
                                              int_only=True)
    assert torch.equal(icost, bcost) and torch.equal(ipart, bpart)
    # SPDP_F_NBR_AUTO: the C3 population's long spans switch the call to the batched sweep (same results)
    acost, apart = spdp.split_eval_neighbours(parent, fwd, bwd, tours, dist, D, cfg["Q"], S=S, window_hint=20,
                                              auto=True)
    assert torch.equal(acost, bcost) and torch.equal(apart, bpart)
    assert spdp.last_kernel().startswith("split_sweep")
    gt = to_dev(synth.local_move_tours(inst["tour"], 64, 5))
    gcost, gpart = spdp.split_eval_neighbours(parent, fwd, bwd, gt, dist, D, cfg["Q"], S=S, window_hint=20, auto=True)
    assert spdp.last_kernel().startswith("split_nbr")
    g2, gp2 = spdp.split_eval_batch(gt, dist, D, cfg["Q"], S=S, window_hint=20)
    assert torch.equal(gcost, g2) and torch.equal(gpart, gp2)
    cols = np.random.default_rng(5).choice(S, size=64, replace=False)
    dem = D.cpu().numpy().view(np.uint16)[:, cols]
    dem = np.ascontiguousarray(np.pad(dem, ((0, 0), (0, (-dem.shape[1]) % 8))))
    want = as_i32(oracle.split_tours(cfg["tours"], inst["dist"], dem, cfg["Q"], S=64))
    assert np.array_equal(cost.cpu().numpy()[:, cols].astype(np.int64), want)


def test_neighbours_usage_errors(spdp):
    cfg = synth.config_instance("C1")
    inst = cfg["inst"]
    S = 100
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    parent, dist, D = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem)
    fwd, bwd = spdp.split_values(parent, dist, D, cfg["Q"], S=S)
    bad = to_dev(np.stack([inst["tour"], np.ones_like(inst["tour"])]))
    with pytest.raises(spdp.SpdpError) as ei:
        spdp.split_eval_neighbours(parent, fwd, bwd, bad, dist, D, cfg["Q"], S=S, validate=True)
    assert ei.value.status == spdp.SPDP_E_DATA


@pytest.mark.parametrize("n,S", [(1, 1), (2, 9), (3, 130), (40, 1)])
def test_neighbours_tiny(spdp, n, S):
    """n = 1 (the only candidate is the parent), n = 2 (every candidate a swap), a partial
    128-scenario CTA and a single scenario; values and costs vs the oracle."""
    rng = np.random.default_rng(n * 1000 + S)
    inst = synth.make_instance(n, seed=77 + n, r=2.0)
    model = synth.demand_model(inst["nominal"], inst["Q"], seed=99)
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    parent = inst["tour"]
    tours = np.ascontiguousarray(np.stack([parent] + [(rng.permutation(n) + 1).astype(np.int32) for _ in range(5)]))
    P, dist, D = to_dev(parent), to_dev(inst["dist"]), to_dev(dem)
    fwd, bwd = spdp.split_values(P, dist, D, inst["Q"], S=S)
    wf, wb = oracle.split_values(parent, inst["dist"], dem, inst["Q"], S=S)
    assert np.array_equal(fwd.cpu().numpy().T.astype(np.int64), as_i32(wf))
    assert np.array_equal(bwd.cpu().numpy().T.astype(np.int64), as_i32(wb))
    want = as_i32(oracle.split_tours(tours, inst["dist"], dem, inst["Q"], S=S))
    for smem in (False, True):
        cost, _ = spdp.split_eval_neighbours(P, fwd, bwd, to_dev(tours), dist, D, inst["Q"], S=S, window_hint=16,
                                             smem=smem)
        assert np.array_equal(cost.cpu().numpy().astype(np.int64), want)


def test_neighbours_large_n_table_in_global_memory(spdp):
    """n above the shared-memory table size of the neighbour kernel (4095)."""
    n, S = 4300, 9
    inst = synth.make_instance(n, seed=4300, r=6.0)
    model = synth.demand_model(inst["nominal"], inst["Q"], seed=96)
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    tours = np.ascontiguousarray(synth.perturb_tours(inst["tour"], 4, 11))
    P, dist, D = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(dem)
    fwd, bwd = spdp.split_values(P, dist, D, inst["Q"], S=S)
    want = as_i32(oracle.split_tours(tours, inst["dist"], dem, inst["Q"], S=S))
    assert np.array_equal(fwd.cpu().numpy()[-1].astype(np.int64), want[0])
    for smem in (False, True):
        cost, _ = spdp.split_eval_neighbours(P, fwd, bwd, to_dev(tours), dist, D, inst["Q"], S=S, window_hint=16,
                                             smem=smem)
        assert np.array_equal(cost.cpu().numpy().astype(np.int64), want)


def test_neighbours_more_scenario_tiles_than_one_grid(spdp):
    """S above 65535 x 128 scenarios: the candidate kernels run as several launches; identical to
    the batched sweep everywhere and to the oracle on sampled columns."""
    cfg = synth.config_instance("C1", S=8_400_000)
    inst, S = cfg["inst"], 65535 * 128 + 1_001
    D = spdp.gen_demands(cfg["model"], 0, S)
    tours = np.ascontiguousarray(synth.perturb_tours(inst["tour"], 6, 13))
    P, dist, Tt = to_dev(inst["tour"]), to_dev(inst["dist"]), to_dev(tours)
    fwd, bwd = spdp.split_values(P, dist, D, cfg["Q"], S=S)
    cost, part = spdp.split_eval_neighbours(P, fwd, bwd, Tt, dist, D, cfg["Q"], S=S, window_hint=16)
    bcost, bpart = spdp.split_eval_batch(Tt, dist, D, cfg["Q"], S=S, window_hint=16)
    assert torch.equal(cost, bcost) and torch.equal(part, bpart)
    cols = np.concatenate([np.arange(0, 40), np.arange(S - 40, S)])
    dem = D.cpu().numpy().view(np.uint16)[:, cols]
    want = as_i32(oracle.split_tours(tours, inst["dist"], np.ascontiguousarray(dem), cfg["Q"], S=cols.size))
    assert np.array_equal(cost.cpu().numpy()[:, cols].astype(np.int64), want)


def test_neighbours_several_parents(spdp):
    """P = 3 parents (random tours) with their candidates interleaved: = the oracle's split of
    every candidate and = three single-parent calls."""
    cfg = synth.config_instance("C3", S=1_003)
    inst, S = cfg["inst"], 1_003
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    D, dist = to_dev(dem), to_dev(inst["dist"])
    rng = np.random.default_rng(21)
    parents = np.ascontiguousarray(np.stack([inst["tour"]] + [(rng.permutation(inst["n"]) + 1).astype(np.int32)
                                                             for _ in range(2)]))
    kids, pof = [], []
    for k in range(3):
        for c in synth.local_move_tours(parents[k], 6, 30 + k):
            kids.append(c)
            pof.append(k)
    order = rng.permutation(len(kids))
    tours = np.ascontiguousarray(np.stack([kids[i] for i in order]))
    pof = np.ascontiguousarray(np.array([pof[i] for i in order], dtype=np.int32))
    vals = [spdp.split_values(to_dev(parents[k]), dist, D, cfg["Q"], S=S) for k in range(3)]
    fwd = torch.stack([v[0] for v in vals]).contiguous()
    bwd = torch.stack([v[1] for v in vals]).contiguous()
    cost, part = spdp.split_eval_neighbours_multi(to_dev(parents), to_dev(pof), fwd, bwd, to_dev(tours), dist, D,
                                                  cfg["Q"], S=S, window_hint=16)
    want = as_i32(oracle.split_tours(tours, inst["dist"], dem, cfg["Q"], S=S))
    assert np.array_equal(cost.cpu().numpy().astype(np.int64), want)
    p = part.cpu().numpy()
    for t in range(tours.shape[0]):
        assert tuple(int(v) for v in p[t, :5]) == _partial_expect(want[t])
