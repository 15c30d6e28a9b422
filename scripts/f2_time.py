import os, sys, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, bench_config, paper_2511_18022_b200 as spdp
dev = torch.device("cuda")
cfg2 = synth.config_instance("C2"); inst2 = cfg2["inst"]
d = spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev)
tour2, dist2 = torch.from_numpy(inst2["tour"]).to(dev), torch.from_numpy(inst2["dist"]).to(dev)
costp = torch.empty(cfg2["S"], dtype=torch.int32, device=dev); partp = torch.zeros(6, dtype=torch.int64, device=dev)
fn = lambda: spdp.split_eval_penalized(tour2, dist2, d, inst2["Q"], 10, S=cfg2["S"], cost=costp, partial=partp, window_hint=20)
for _ in range(3): fn()
torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): fn()
b.record(); torch.cuda.synchronize(); print("f2 penalized %.4f ms" % (a.elapsed_time(b)/10))
