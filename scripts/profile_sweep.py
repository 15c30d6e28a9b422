"""Short driver for ncu: a few C2 steps (or --config C3/C4, --irp) through the C-ABI."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import bench_config
import paper_2511_18022_b200 as spdp
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--hint", type=int, default=None)
ap.add_argument("--irp", action="store_true")
ap.add_argument("--nbr", action="store_true", help="f3: values of tour 0 + neighbour evaluation of the population")
ap.add_argument("--granular", action="store_true", help="f3 with the granular one-move population")
ap.add_argument("--limits", action="store_true", help="f4: duration 1.5 x max trip + fleet ceil(sum mu / Q) + 2")
ap.add_argument("--f32", action="store_true", help="fp32 mode with unrounded Euclidean costs")
ap.add_argument("--ordered", action="store_true", help="scenario set ordered by total demand (as bench.py)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
if a.irp:
    c5 = synth.irp_config()
    irp = c5["irp"]
    d = spdp.gen_demands(c5["model"], 0, c5["S"], device=dev)
    for _ in range(a.iters):
        spdp.irp_dp(irp["visit"], irp["cust"], d, irp["H"], irp["M"], S=c5["S"])
else:
    cfg = synth.config_instance(a.config)
    inst = cfg["inst"]
    d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
    if a.ordered:
        d, _ = spdp.order_scenarios(d, S=cfg["S"])
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
    dist = torch.from_numpy(inst["dist"]).to(dev)
    h = a.hint if a.hint is not None else bench_config.HINT[a.config]
    if a.granular:
        tours = torch.from_numpy(synth.local_move_tours(inst["tour"], cfg["T"], 400)).to(dev)
    if a.limits:
        trip = int(max(inst["dist"][0, c] + inst["dist"][c, 0] for c in inst["tour"]))
        kmin = int(np.ceil(inst["nominal"].astype(np.int64).sum() / inst["Q"]))
    if a.nbr:
        parent = tours[0].contiguous()
        fwd, bwd = spdp.split_values(parent, dist, d, inst["Q"], S=cfg["S"])
    for _ in range(a.iters):
        if a.f32:
            xy = np.asarray(inst["coords"], dtype=np.float64)
            distf = torch.from_numpy(np.ascontiguousarray(np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)))).to(dev)
            spdp.split_eval_f32(tours[0].contiguous(), distf, d, inst["Q"], S=cfg["S"])
        elif a.limits:
            spdp.split_eval_limits(tours[0].contiguous(), dist, d, inst["Q"], max_duration=int(trip * 1.5),
                                   max_routes=kmin + 2, S=cfg["S"])
        elif a.nbr:
            spdp.split_eval_neighbours(parent, fwd, bwd, tours, dist, d, inst["Q"], S=cfg["S"], want_cost=False,
                                       window_hint=h)
        elif cfg["T"] == 1:
            spdp.split_eval(tours[0].contiguous(), dist, d, inst["Q"], S=cfg["S"], window_hint=h,
                            mean_window=(bench_config.MEAN_ORDERED if a.ordered else bench_config.MEAN)[a.config])
        else:
            spdp.split_eval_batch(tours, dist, d, inst["Q"], S=cfg["S"], want_cost=False, window_hint=h,
                                  mean_window=(bench_config.MEAN_ORDERED if a.ordered else bench_config.MEAN)[a.config])
torch.cuda.synchronize()
print("done")
