"""World-size-2 gloo run of the multi-GPU host logic (sharding + one all-reduce of
the int64 SAA partials + host finalize), on CPU.  The per-rank partials come from
the oracle (test infrastructure); the product's dist helpers and spdp_saa_mean
combine them, and the result must equal the single-process oracle SAA exactly."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial_from_oracle(cost):
    r = oracle.saa(cost)
    sq = r["sumsq"]
    return torch.tensor([r["m"], r["infeasible"], r["sum"], sq & 0xffffffff, sq >> 32, 0], dtype=torch.int64)


def _worker(rank, world, port, S, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_18022_b200 import dist as pdist
        import paper_2511_18022_b200 as spdp
        cfg = synth.config_instance("C2", S=S)
        inst = cfg["inst"]
        b, e = pdist.shard_range(S, rank, world)
        dem = oracle.gen_demands(cfg["model"], b, e - b)
        cost = oracle.split(inst["tour"], inst["dist"], dem, inst["Q"])
        part = _partial_from_oracle(cost)
        pdist.allreduce_partials(part)
        est = spdp.saa_mean(part)
        tmax = pdist.max_over_ranks(float(rank + 1))
        q.put((rank, est["mean"], est["var"], int(part[0]), tmax))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_saa_equals_single_process():
    S = 4001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, S, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.config_instance("C2", S=S)
    inst = cfg["inst"]
    dem = oracle.gen_demands(cfg["model"], 0, S)
    w = oracle.saa(oracle.split(inst["tour"], inst["dist"], dem, inst["Q"]))
    for rank, mean, var, m, tmax in res:
        assert m == S and mean == w["mean"]
        assert abs(var - w["var"]) <= 1e-12 * w["var"]
        assert tmax == 2.0


def test_shard_ranges_cover_exactly():
    from paper_2511_18022_b200 import dist as pdist
    for S in (1, 7, 1000, 10**6 + 3):
        for R in (1, 2, 3, 4, 8):
            rs = [pdist.shard_range(S, r, R) for r in range(R)]
            assert rs[0][0] == 0 and rs[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def _np_moments(cost, center):
    """Host stand-in for spdp_saa_f32_moments (no GPU in this container): {m, sum, ssdev, inf}."""
    c = np.asarray(cost, dtype=np.float32)
    fin = c[np.isfinite(c)].astype(np.float64)
    return torch.tensor([float(fin.size), float(fin.sum()), float(((fin - center) ** 2).sum()),
                         float(c.size - fin.size)], dtype=torch.float64)


def _worker_f32(rank, world, port, S, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_18022_b200 import dist as pdist
        cfg = synth.config_instance("C2", S=S)
        inst = cfg["inst"]
        xy = np.asarray(inst["coords"], dtype=np.float64)
        distf = np.ascontiguousarray(np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)))
        b, e = pdist.shard_range(S, rank, world)
        model = dict(cfg["model"])
        model["q_cap"] = inst["Q"] + 20  # some infeasible scenarios
        dem = oracle.gen_demands(model, b, e - b)
        cost = oracle.split_f32(inst["tour"], distf, dem, inst["Q"])
        est = pdist.saa_estimate_f32(cost, moments_fn=_np_moments)
        q.put((rank, est["m"], est["infeasible"], est["mean"], est["var"]))
    finally:
        dist.destroy_process_group()


def test_two_rank_fp32_saa_equals_single_process():
    """The fp32-mode SAA over 2 ranks (two passes, one all-reduce each) agrees with the
    single-process sequential-fp64 oracle within 1e-9 relative."""
    S = 3001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_f32, args=(r, 2, port, S, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.config_instance("C2", S=S)
    inst = cfg["inst"]
    xy = np.asarray(inst["coords"], dtype=np.float64)
    distf = np.ascontiguousarray(np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)))
    model = dict(cfg["model"])
    model["q_cap"] = inst["Q"] + 20
    w = oracle.saa_f32(oracle.split_f32(inst["tour"], distf, oracle.gen_demands(model, 0, S), inst["Q"]))
    assert w["infeasible"] > 0
    for rank, m, ninf, mean, var in res:
        assert m == w["m"] and ninf == w["infeasible"]
        assert abs(mean - w["mean"]) <= 1e-9 * w["mean"]
        assert abs(var - w["var"]) <= 1e-9 * w["var"]
