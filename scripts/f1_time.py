import os, sys, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, paper_2511_18022_b200 as spdp
dev = torch.device("cuda")
cfg2 = synth.config_instance("C2"); inst2 = cfg2["inst"]
d = spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev)
tour2, dist2 = torch.from_numpy(inst2["tour"]).to(dev), torch.from_numpy(inst2["dist"]).to(dev)
K = 4096
scen = torch.arange(0, cfg2["S"], cfg2["S"] // K, dtype=torch.int64, device=dev)[:K].contiguous()
fn = lambda: spdp.split_routes(tour2, dist2, d, inst2["Q"], scen, S=cfg2["S"])
for _ in range(3): fn()
torch.cuda.synchronize(); ts=[]
for _ in range(10):
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("f1 routes 4096 scenarios: call %.4f ms" % statistics.median(ts))
ev=[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
for a,b in ev: a.record(); b.record()
for a,b in ev:
    spdp.set_profile_events(a,b); fn()
spdp.set_profile_events(); torch.cuda.synchronize()
print("f1 route kernel %s: %.4f ms" % (spdp.last_kernel(), statistics.median(a.elapsed_time(b) for a,b in ev)))
