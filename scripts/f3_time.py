"""f3 timing on the ordered C3 set: the C3 population and the granular one, u16 path (default) vs the
int32 ring (int_only) vs the batched sweep; partials checked equal to the batch."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, bench_config, paper_2511_18022_b200 as spdp
dev = torch.device("cuda")
cfg = synth.config_instance("C3"); inst = cfg["inst"]
d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
d, _ = spdp.order_scenarios(d, S=cfg["S"])
dist = torch.from_numpy(inst["dist"]).to(dev)
tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
parent = tours[0].contiguous()
fwd = torch.empty((cfg["n"] + 1, cfg["S"]), dtype=torch.int32, device=dev); bwd = torch.empty_like(fwd)
spdp.split_values(parent, dist, d, inst["Q"], S=cfg["S"], fwd=fwd, bwd=bwd)
h = bench_config.HINT["C3"]; mw = bench_config.MEAN_ORDERED["C3"]
def t(fn, it=5):
    for _ in range(2): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(it):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)
for name, tt in (("population", tours), ("granular", torch.from_numpy(synth.local_move_tours(inst["tour"], cfg["T"], 400)).to(dev))):
    cb, pb = spdp.split_eval_batch(tt, dist, d, inst["Q"], S=cfg["S"], want_cost=True, window_hint=h, mean_window=mw)
    cu, pu = spdp.split_eval_neighbours(parent, fwd, bwd, tt, dist, d, inst["Q"], S=cfg["S"], window_hint=h, mean_window=mw)
    k_u = spdp.last_kernel()
    ci, pi = spdp.split_eval_neighbours(parent, fwd, bwd, tt, dist, d, inst["Q"], S=cfg["S"], window_hint=h, int_only=True)
    k_i = spdp.last_kernel()
    print(name, "costs equal batch: u16 %s int %s; partials %s %s" % (bool(torch.equal(cu, cb)), bool(torch.equal(ci, cb)),
          bool(torch.equal(pu, pb)), bool(torch.equal(pi, pb))), flush=True)
    tb = t(lambda: spdp.split_eval_batch(tt, dist, d, inst["Q"], S=cfg["S"], want_cost=False, window_hint=h, mean_window=mw))
    tu = t(lambda: spdp.split_eval_neighbours(parent, fwd, bwd, tt, dist, d, inst["Q"], S=cfg["S"], want_cost=False,
                                              window_hint=h, mean_window=mw))
    ti = t(lambda: spdp.split_eval_neighbours(parent, fwd, bwd, tt, dist, d, inst["Q"], S=cfg["S"], want_cost=False,
                                              window_hint=h, int_only=True))
    print(name, "batch %.3f ms | f3 u16 (%s) %.3f ms | f3 int32 ring (%s) %.3f ms" % (tb, k_u, tu, k_i, ti), flush=True)
