"""C3 batch on three layouts of the scenario set: as generated, ordered by total demand
(spdp_order_scenarios), and ordered (globally, stable) by tour 0's Eq. (3) window sum -- a probe of
whether a window-based key groups warps better than total demand."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, bench_config, paper_2511_18022_b200 as spdp
dev = torch.device("cuda")
cfg = synth.config_instance("C3"); inst = cfg["inst"]; S = cfg["S"]; n = cfg["n"]
d = spdp.gen_demands(cfg["model"], 0, S, device=dev)
tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev); dist = torch.from_numpy(inst["dist"]).to(dev)
dO, _ = spdp.order_scenarios(d, S=S)
m = spdp.split_mask(tours[0].contiguous(), d, inst["Q"], S=S).to(torch.int64)
idx = torch.arange(1, n + 1, device=dev, dtype=torch.int64).unsqueeze(1)
key = ((idx - m) * (m >= 0)).sum(0)  # window sum per scenario (tour 0)
perm = torch.sort(key, stable=True, descending=True).indices  # longest windows first
dW = spdp.empty_demand(n, S, dev)
dW[:, :S] = d[:, :S].index_select(1, perm)
tot = d[:, :S].to(torch.int64).sum(0)
permT = torch.sort(tot, stable=True).indices
dT = spdp.empty_demand(n, S, dev)
dT[:, :S] = d[:, :S].index_select(1, permT)
def t(dd, mw):
    fn = lambda: spdp.split_eval_batch(tours, dist, dd, inst["Q"], S=S, want_cost=False, window_hint=20, mean_window=mw)
    for _ in range(2): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts), spdp.last_kernel()
for name, dd in (("natural", d), ("total demand, 64K segments", dO), ("total demand, global", dT), ("window sum (tour 0), global", dW)):
    for mw in (4, 6):
        print("%-30s mw=%d %.3f ms %s" % (name, mw, *t(dd, mw)), flush=True)
