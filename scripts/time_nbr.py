"""Device time of spdp_split_eval_neighbours at C3 (the C3 and the granular populations) per ring width."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_18022_b200 as spdp
import synth

dev = torch.device("cuda")
cfg = synth.config_instance("C3")
inst = cfg["inst"]
d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
dist = torch.from_numpy(inst["dist"]).to(dev)
parent = torch.from_numpy(inst["tour"]).to(dev)
fwd, bwd = spdp.split_values(parent, dist, d, inst["Q"], S=cfg["S"])
pops = {"C3": cfg["tours"], "granular": synth.local_move_tours(inst["tour"], cfg["T"], 400)}
for name, tt in pops.items():
    tours = torch.from_numpy(np.ascontiguousarray(tt)).to(dev)
    for h, smem, io in [(20, False, False), (20, False, True), (20, True, False)]:
        fn = lambda: spdp.split_eval_neighbours(parent, fwd, bwd, tours, dist, d, inst["Q"], S=cfg["S"],
                                                want_cost=False, window_hint=h, smem=smem, int_only=io)
        for _ in range(2):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        print("%-9s hint=%2d int_only=%d %-26s %.3f ms" % (name, h, io, spdp.last_kernel(), a.elapsed_time(b) / 5))
