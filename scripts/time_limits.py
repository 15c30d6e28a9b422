"""Device time of spdp_split_eval_limits at C2 for a few (duration, fleet) limits (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_18022_b200 as spdp
import synth

dev = torch.device("cuda")
cfg = synth.config_instance("C2")
inst = cfg["inst"]
d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
tour, dist = torch.from_numpy(inst["tour"]).to(dev), torch.from_numpy(inst["dist"]).to(dev)
trip = int(max(inst["dist"][0, c] + inst["dist"][c, 0] for c in inst["tour"]))
kmin = int(np.ceil(inst["nominal"].astype(np.int64).sum() / inst["Q"]))
for L, K, g in ((int(trip * 1.5), 0, False), (-1, kmin + 2, False), (int(trip * 1.5), kmin + 2, False),
                (-1, kmin + 6, False), (-1, kmin + 2, True)):
    for _ in range(2):
        c, p = spdp.split_eval_limits(tour, dist, d, inst["Q"], max_duration=L, max_routes=K, scratch_global=g)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        c, p = spdp.split_eval_limits(tour, dist, d, inst["Q"], max_duration=L, max_routes=K, scratch_global=g)
    b.record()
    torch.cuda.synchronize()
    print("Lmax=%d K=%d general_only=%d: %.3f ms  (feasible, infeasible) = %s" % (
        L, K, g, a.elapsed_time(b) / 3, p.cpu().tolist()[:2]))
