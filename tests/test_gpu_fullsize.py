"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The oracle cannot evaluate every output of C3/C4 in seconds, so those are
checked on sampled outputs the oracle computes one by one (plus the fused SAA
partial against a separate reduction of the per-scenario costs); C2 is checked
completely (all 10^6 costs and the SAA estimate).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import bench_config  # noqa: E402  (repo root, same launch configuration as bench.py)


@pytest.fixture(scope="module")
def spdp():
    import paper_2511_18022_b200 as m
    return m


def _sample_cols(model, idx):
    cols = [oracle.gen_demands(model, int(s), 1) for s in idx]
    return np.concatenate(cols, axis=1)


def test_c2_full_all_costs_and_saa(spdp):
    cfg = synth.config_instance("C2")
    inst, S = cfg["inst"], cfg["S"]
    d = spdp.gen_demands(cfg["model"], 0, S)
    tour, dist = torch.from_numpy(inst["tour"]).cuda(), torch.from_numpy(inst["dist"]).cuda()
    dem = oracle.gen_demands(cfg["model"], 0, S)
    assert np.array_equal(d.cpu().numpy().view(np.uint16)[:, :S], dem)
    want = oracle.split(inst["tour"], inst["dist"], dem, inst["Q"])
    w = oracle.saa(want)
    for algo in (None, "f32", "deque", "u16"):  # None = the launch configuration bench.py times
        cost, part = spdp.split_eval(tour, dist, d, inst["Q"], S=S, window_hint=bench_config.HINT["C2"], algo=algo)
        got = cost.cpu().numpy().astype(np.int64)
        assert np.array_equal(got, want), algo
        est = spdp.saa_mean(part)
        assert est["m"] == S and est["mean"] == w["mean"]
        assert abs(est["var"] - w["var"]) <= 1e-12 * w["var"]
    # bench.py's default step: the set ordered by total demand, the ordered launch configuration
    dO, perm = spdp.order_scenarios(d, S=S)
    p = perm.cpu().numpy()
    assert np.array_equal(np.sort(p), np.arange(S))
    cost, part = spdp.split_eval(tour, dist, dO, inst["Q"], S=S, window_hint=bench_config.HINT["C2"],
                                 mean_window=bench_config.MEAN_ORDERED["C2"])
    assert np.array_equal(cost.cpu().numpy().astype(np.int64), np.asarray(want)[p])
    est = spdp.saa_mean(part)
    assert est["m"] == S and est["mean"] == w["mean"]


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_sampled(spdp, name):
    cfg = synth.config_instance(name)
    inst, S, T = cfg["inst"], cfg["S"], cfg["T"]
    d = spdp.gen_demands(cfg["model"], 0, S)
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).cuda()
    dist = torch.from_numpy(inst["dist"]).cuda()
    cost, part = spdp.split_eval_batch(tours, dist, d, inst["Q"], S=S, window_hint=bench_config.HINT[name],
                                       mean_window=bench_config.MEAN[name])
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([rng.integers(0, S, size=150), [0, 1, S - 2, S - 1]]))
    dem = _sample_cols(cfg["model"], idx)
    got = cost.cpu().numpy()
    for t in sorted(set([0, T - 1] + list(rng.integers(0, T, size=3)))):
        want = oracle.split(cfg["tours"][t], inst["dist"], dem, inst["Q"])
        assert np.array_equal(got[t, idx].astype(np.int64), want), "tour %d" % t
    # the fused SAA partial equals an independent reduction of the device's per-scenario costs
    for t in (0, T - 1):
        ref = spdp.saa_reduce(cost[t].contiguous())
        assert torch.equal(ref.cpu(), part[t].cpu())


def test_c2_full_next_rows_sampled(spdp):
    """The NEXT rows and the fp32 mode at C2's full size (10^6 scenarios), in the bench's
    launch configuration, on sampled scenarios the oracle evaluates one by one."""
    cfg = synth.config_instance("C2")
    inst, S = cfg["inst"], cfg["S"]
    d = spdp.gen_demands(cfg["model"], 0, S)
    tour, dist = torch.from_numpy(inst["tour"]).cuda(), torch.from_numpy(inst["dist"]).cuda()
    rng = np.random.default_rng(1)
    idx = np.unique(np.concatenate([rng.integers(0, S, size=120), [0, S - 1]]))
    dem = _sample_cols(cfg["model"], idx)
    Q = inst["Q"]
    # f2 penalized (lambda = 10)
    pc, _ = spdp.split_eval_penalized(tour, dist, d, Q, 10, S=S, window_hint=bench_config.HINT["C2"])
    assert np.array_equal(pc.cpu().numpy()[idx].astype(np.int64), oracle.split_penalized(inst["tour"], inst["dist"],
                                                                                        dem, Q, 10))
    # f4 duration and fleet limits (the bench row's limits)
    trip = int(max(inst["dist"][0, c] + inst["dist"][c, 0] for c in inst["tour"]))
    kmin = int(np.ceil(inst["nominal"].astype(np.int64).sum() / Q))
    for L, K in ((int(trip * 1.5), 0), (-1, kmin + 2)):
        lc, _ = spdp.split_eval_limits(tour, dist, d, Q, max_duration=L, max_routes=K, S=S)
        want = oracle.split_limits(inst["tour"], inst["dist"], dem, Q, Lmax=L, K=K)
        want = np.where(want == oracle.INF, 2**31 - 1, want)
        assert np.array_equal(lc.cpu().numpy()[idx].astype(np.int64), want), (L, K)
    # f3 values of the tour
    fwd, bwd = spdp.split_values(tour, dist, d, Q, S=S)
    wf, wb = oracle.split_values(inst["tour"], inst["dist"], dem, Q)
    assert np.array_equal(fwd.cpu().numpy()[:, idx].T.astype(np.int64), wf)
    assert np.array_equal(bwd.cpu().numpy()[:, idx].T.astype(np.int64), wb)
    # fp32 mode with unrounded Euclidean costs
    xy = np.asarray(inst["coords"], dtype=np.float64)
    distf = np.ascontiguousarray(np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)))
    c32 = spdp.split_eval_f32(tour, torch.from_numpy(distf).cuda(), d, Q, S=S).cpu().numpy()
    assert np.array_equal(c32[idx].view(np.uint32), oracle.split_f32(inst["tour"], distf, dem, Q).view(np.uint32))


def test_c5_irp_full_sampled(spdp):
    """The IRP row at C5's full size (10^5 scenarios, the bench's launch) on sampled scenarios."""
    cfg = synth.irp_config()
    irp, S = cfg["irp"], cfg["S"]
    H, M = irp["H"], irp["M"]
    d = spdp.gen_demands(cfg["model"], 0, S)
    cost, part = spdp.irp_dp(irp["visit"], irp["cust"], d, H, M, S=S)
    rng = np.random.default_rng(2)
    idx = np.unique(np.concatenate([rng.integers(0, S, size=40), [0, S - 1]]))
    dem = _sample_cols(cfg["model"], idx)
    want = oracle.irp(H, M, irp["visit"], irp["cust"], dem)
    assert np.array_equal(cost.cpu().numpy()[idx], want)
    assert int(part.cpu().numpy()[2]) == int(cost.sum().item())
