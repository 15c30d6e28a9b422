"""Time the sweep kernel alone (profile-event hook) for several window hints / configs."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench_config
import paper_2511_18022_b200 as spdp
import synth

dev = torch.device("cuda", 0)
configs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2"]
hints = [int(h) for h in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 16, 32]
for name in configs:
    cfg = synth.config_instance(name)
    inst = cfg["inst"]
    d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
    dist = torch.from_numpy(inst["dist"]).to(dev)
    for h in hints:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        tot = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for a, b in evs:
            a.record(); b.record()
        for it in range(13):
            if it >= 3:
                spdp.set_profile_events(*evs[it - 3])
                tot[it - 3][0].record()
            spdp.split_eval_batch(tours, dist, d, inst["Q"], S=cfg["S"], window_hint=h, want_cost=cfg["T"] == 1,
                                  mean_window=int(os.environ.get("SPDP_MEANW", bench_config.MEAN[name])))
            if it >= 3:
                tot[it - 3][1].record()
        spdp.set_profile_events()
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in evs)
        ms_tot = statistics.median(a.elapsed_time(b) for a, b in tot)
        print("%s VE=%s hint=%d sweep_ms=%.4f total_ms=%.4f evals/s=%.3e" % (
            name, os.environ.get("SPDP_VOTE_EVERY", "4"), h, ms, ms_tot, cfg["S"] * cfg["T"] / ms_tot * 1e3), flush=True)
