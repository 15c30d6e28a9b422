"""GPU parity of the cross-GPU combine: partials made by the CUDA path on
scenario shards, summed (simulated ranks) or all-reduced across processes (gloo, the CPU transport
of the same torch.distributed call that NCCL serves on a multi-GPU box), against the single-call
partial over all scenarios and the oracle's sums (scenarios are independent)."""
import os
import socket

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


def _oracle_partial(cost):
    """(m, infeasible, sum, sum of squares) of the oracle's costs, as Python ints."""
    r = oracle.saa(cost)
    return (int(r["m"]), int(r["infeasible"]), int(r["sum"]), int(r["sumsq"]))


def _key(part):
    """The same four numbers of an int64 [6] partial: its sum of squares is sumsq_lo + 2^32 sumsq_hi
    (the halves are per-cost splits summed, spdp.h -- their split differs, their value does not)."""
    p = [int(v) for v in np.asarray(part).reshape(6)]
    return (p[0], p[1], p[2], p[3] + (p[4] << 32))


def _instance(S, q_extra=0):
    cfg = synth.config_instance("C2", S=S)
    inst = cfg["inst"]
    model = dict(cfg["model"])
    if q_extra:
        model["q_cap"] = inst["Q"] + q_extra  # some scenarios infeasible
    return inst, model


@pytest.mark.parametrize("algo", [None, "f32", "deque"])
def test_simulated_ranks_partials_sum_to_the_full_partial(spdp, algo):
    S = 200_003
    inst, model = _instance(S, q_extra=30)
    tour = torch.from_numpy(inst["tour"]).cuda()
    dist = torch.from_numpy(inst["dist"]).cuda()
    full_d = spdp.gen_demands(model, 0, S)
    _, full = spdp.split_eval(tour, dist, full_d, inst["Q"], S=S, window_hint=20, algo=algo)
    full = full.cpu().numpy()
    want = _oracle_partial(oracle.split(inst["tour"], inst["dist"], oracle.gen_demands(model, 0, S), inst["Q"]))
    assert _key(full) == want
    assert want[1] > 0  # infeasible scenarios are part of the combine
    from paper_2511_18022_b200 import dist as pdist
    for R in (2, 3, 8):
        acc = np.zeros(6, dtype=np.int64)
        for r in range(R):
            b, e = pdist.shard_range(S, r, R)
            d = spdp.gen_demands(model, b, e - b)
            _, part = spdp.split_eval(tour, dist, d, inst["Q"], S=e - b, window_hint=20, algo=algo)
            acc += part.cpu().numpy()
        assert np.array_equal(acc, full), (R, acc, full)  # (field by field: every field is a plain sum)
        est = spdp.saa_mean(acc)
        assert est["mean"] == spdp.saa_mean(full)["mean"] and est["m"] == want[0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_18022_b200 as spdp
        from paper_2511_18022_b200 import dist as pdist
        inst, model = _instance(S, q_extra=30)
        b, e = pdist.shard_range(S, rank, world)
        d = spdp.gen_demands(model, b, e - b, device="cuda:0")
        tour = torch.from_numpy(inst["tour"]).cuda()
        dist_m = torch.from_numpy(inst["dist"]).cuda()
        _, part = spdp.split_eval(tour, dist_m, d, inst["Q"], S=e - b, window_hint=20)
        part = part.cpu()  # (gloo reduces host tensors; NCCL would take the device tensor as is)
        pdist.allreduce_partials(part)
        est = spdp.saa_mean(part)
        q.put((rank, part.numpy().tolist(), est["mean"], est["var"]))
    finally:
        dist.destroy_process_group()


def test_two_processes_allreduce_cuda_partials():
    """Two processes on cuda:0, each the CUDA sweep of its shard, one all-reduce(SUM) of the int64
    partials (gloo): bit-identical to the single-process partial and to the oracle."""
    import torch.multiprocessing as mp
    S = 100_001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, S, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inst, model = _instance(S, q_extra=30)
    want = _oracle_partial(oracle.split(inst["tour"], inst["dist"], oracle.gen_demands(model, 0, S), inst["Q"]))
    for rank, part, mean, var in res:
        assert _key(part) == want
    assert res[0][2] == res[1][2] and res[0][3] == res[1][3]


def test_saa_finalize_f32_two_shards_match_single_call(spdp):
    """fp32-mode multi-rank estimate through spdp_saa_finalize_f32 (the C finalize; the binding only
    moves the moments): shards' device moments summed == the single-call spdp_saa_estimate_f32."""
    S = 50_001
    inst, model = _instance(S, q_extra=20)
    xy = np.asarray(inst["coords"], dtype=np.float64)
    distf = torch.from_numpy(np.ascontiguousarray(np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)))).cuda()
    tour = torch.from_numpy(inst["tour"]).cuda()
    d = spdp.gen_demands(model, 0, S)
    cost = spdp.split_eval_f32(tour, distf, d, inst["Q"], S=S)
    single = spdp.saa_estimate_f32(cost)
    halves = [cost[: S // 2], cost[S // 2:]]
    m1 = sum(spdp.saa_f32_moments(c, 0.0).cpu() for c in halves)
    center = spdp.saa_finalize_f32(m1)["mean"]
    m2 = sum(spdp.saa_f32_moments(c, center).cpu() for c in halves)
    est = spdp.saa_finalize_f32(m1, m2)
    assert est["m"] == single["m"] and est["infeasible"] == single["infeasible"] > 0
    assert abs(est["mean"] - single["mean"]) <= 1e-12 * single["mean"]
    assert abs(est["var"] - single["var"]) <= 1e-9 * single["var"]
