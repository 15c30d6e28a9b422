"""Scenario ordering (spdp_order_scenarios, DESIGN §"scenario order"): the permutation is the
stable counting sort of the bucketed total demand (numpy restatement of its definition), the
ordered matrix is the permuted columns, and every evaluation on it is the permuted evaluation
(per-scenario costs) with identical SAA partials."""
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


def want_perm(dem, S):
    key = dem[:, :S].astype(np.int64).sum(0)
    bucket = (key * 1024) // (int(key.max()) + 1)
    seg = np.arange(S) // 65536  # segments of 65536 scenarios stay in place
    return np.lexsort((np.arange(S), bucket, seg)).astype(np.int32)


@pytest.mark.parametrize("name,S", [("C1", 1), ("C1", 100), ("C2", 4_097), ("C2", 20_011), ("C3", 9_001),
                                    ("C2", 150_001)])
def test_order_permutation_and_columns(spdp, name, S):
    cfg = synth.config_instance(name, S=S)
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    out, perm = spdp.order_scenarios(to_dev(dem), S=S)
    p = perm.cpu().numpy()
    assert np.array_equal(p, want_perm(dem, S))
    assert np.array_equal(np.sort(p), np.arange(S))
    o = out.cpu().numpy().view(np.uint16)
    assert np.array_equal(o[:, :S], dem[:, :S][:, p])


def test_order_evaluations_are_permuted(spdp):
    cfg = synth.config_instance("C3", S=5_003)
    inst, S = cfg["inst"], cfg["S"]
    dem = oracle.gen_demands(cfg["model"], 0, S, ld=spdp.padded_ld(S))
    D = to_dev(dem)
    out, perm = spdp.order_scenarios(D, S=S)
    p = perm.cpu().numpy()
    tours, dist = to_dev(cfg["tours"][:8]), to_dev(inst["dist"])
    c0, p0 = spdp.split_eval_batch(tours, dist, D, cfg["Q"], S=S, want_cost=True)
    c1, p1 = spdp.split_eval_batch(tours, dist, out, cfg["Q"], S=S, want_cost=True)
    assert np.array_equal(c1.cpu().numpy(), c0.cpu().numpy()[:, p])
    assert np.array_equal(p1.cpu().numpy(), p0.cpu().numpy())
    want = oracle.split(cfg["tours"][0], inst["dist"], dem, cfg["Q"], S=S)
    assert np.array_equal(c1.cpu().numpy()[0], np.asarray(want)[p])
