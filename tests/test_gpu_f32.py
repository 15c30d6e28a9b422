"""GPU parity of the fp32 mode (DESIGN R25): real-valued costs, float32 costs bit-identical to
the oracle's fp32 split; the SAA estimate within 1e-9 relative of the oracle's sequential fp64."""
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


def real_dist(inst):
    xy = np.asarray(inst["coords"], dtype=np.float64)
    return np.ascontiguousarray(np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)))


@pytest.mark.parametrize("name,S,extra_q", [("C1", 100, 0), ("C2", 20_011, 0), ("C2", 3_001, 40), ("C3", 2_003, 0),
                                            ("C4", 301, 0)])
def test_split_f32_parity(spdp, name, S, extra_q):
    cfg = synth.config_instance(name, S=S)
    inst = cfg["inst"]
    model = dict(cfg["model"])
    model["q_cap"] = int(min(cfg["Q"] + extra_q, 65535))
    dem = oracle.gen_demands(model, 0, S, ld=spdp.padded_ld(S))
    dist = real_dist(inst)
    got = spdp.split_eval_f32(to_dev(inst["tour"]), to_dev(dist), to_dev(dem), cfg["Q"], S=S).cpu().numpy()
    want = oracle.split_f32(inst["tour"], dist, dem, cfg["Q"], S=S)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))  # bit for bit (incl. +inf)
    est = spdp.saa_estimate_f32(torch.from_numpy(got).cuda())
    ref = oracle.saa_f32(want)
    assert est["m"] == ref["m"] and est["infeasible"] == ref["infeasible"]
    assert abs(est["mean"] - ref["mean"]) <= 1e-9 * abs(ref["mean"])
    assert abs(est["var"] - ref["var"]) <= 1e-9 * abs(ref["var"]) + 1e-12


def test_split_f32_integer_costs_equal_integer_mode(spdp):
    cfg = synth.config_instance("C2", S=4_099)
    inst, S = cfg["inst"], 4_099
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    D = to_dev(dem)
    tour = to_dev(inst["tour"])
    c32 = spdp.split_eval_f32(tour, to_dev(inst["dist"].astype(np.float64)), D, cfg["Q"], S=S)
    ci, _ = spdp.split_eval(tour, to_dev(inst["dist"]), D, cfg["Q"], S=S, window_hint=20)
    assert torch.equal(c32.to(torch.float64), ci.to(torch.float64))


def test_split_f32_edge_cases(spdp):
    dist = np.array([[0.0, 7.25], [9.5, 0.0]])
    dem = synth.explicit_demands([[3], [5], [6]])
    got = spdp.split_eval_f32(to_dev(np.array([1], dtype=np.int32)), to_dev(dist), to_dev(dem), 5, S=3).cpu().numpy()
    assert got[0] == np.float32(16.75) and got[1] == np.float32(16.75) and np.isinf(got[2])
    allinf = torch.full((5,), float("inf"), device="cuda")
    with pytest.raises(spdp.SpdpError) as ei:
        spdp.saa_estimate_f32(allinf)
    assert ei.value.status == spdp.SPDP_E_DATA


def test_saa_f32_moments_and_dist_helper(spdp):
    """The moments kernel behind the multi-rank fp32 SAA: single process, the dist helper's two
    passes equal spdp_saa_estimate_f32."""
    from paper_2511_18022_b200 import dist as pdist
    rng = np.random.default_rng(3)
    c = rng.uniform(5e4, 9e4, size=100_003).astype(np.float32)
    c[::101] = np.inf
    ct = torch.from_numpy(c).cuda()
    m = spdp.saa_f32_moments(ct, 0.0).cpu().numpy()
    fin = c[np.isfinite(c)].astype(np.float64)
    assert m[0] == fin.size and m[3] == c.size - fin.size
    assert abs(m[1] - fin.sum()) <= 1e-12 * fin.sum()
    a = pdist.saa_estimate_f32(ct)
    b = spdp.saa_estimate_f32(ct)
    assert a["m"] == b["m"] and a["infeasible"] == b["infeasible"]
    assert abs(a["mean"] - b["mean"]) <= 1e-13 * b["mean"] and abs(a["var"] - b["var"]) <= 1e-12 * b["var"]


def test_split_batch_f32_parity(spdp):
    cfg = synth.config_instance("C3", S=701)
    inst, S = cfg["inst"], 701
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    tours = np.ascontiguousarray(cfg["tours"][:9])
    dist = real_dist(inst)
    got = spdp.split_eval_batch_f32(to_dev(tours), to_dev(dist), to_dev(dem), cfg["Q"], S=S).cpu().numpy()
    for t in range(tours.shape[0]):
        want = oracle.split_f32(tours[t], dist, dem, cfg["Q"], S=S)
        assert np.array_equal(got[t].view(np.uint32), want.view(np.uint32)), t
