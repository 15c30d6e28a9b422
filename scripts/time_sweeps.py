"""Time the sweep kernel alone (profile-event hook) per config x algorithm x window hint, and
check that every algorithm returns the same per-scenario costs (on the GPU, against the first).

    python scripts/time_sweeps.py C2,C3 auto,u16,f32 [hints]
"""
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
algos = [None if a == "auto" else a for a in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto"])]
hints_arg = [int(h) for h in sys.argv[3].split(",")] if len(sys.argv) > 3 and sys.argv[3] else None
mws_arg = [int(m) for m in sys.argv[4].split(",")] if len(sys.argv) > 4 and sys.argv[4] else None
q_arg = int(sys.argv[5]) if len(sys.argv) > 5 else None
for name in configs:
    cfg = synth.config_instance(name)
    inst = cfg["inst"]
    d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
    dist = torch.from_numpy(inst["dist"]).to(dev)
    hints = hints_arg or [bench_config.HINT[name]]
    ref = None
    for algo, h, mw in [(a, h, m) for a in algos for h in hints for m in (mws_arg or [bench_config.MEAN[name]])]:
        if True:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            tot = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for a, b in evs:
                a.record()
                b.record()
            cost = None
            for it in range(13):
                if it >= 3:
                    spdp.set_profile_events(*evs[it - 3])
                    tot[it - 3][0].record()
                cost, part = spdp.split_eval_batch(tours, dist, d, q_arg or inst["Q"], S=cfg["S"], window_hint=h, want_cost=True,
                                                   mean_window=mw, algo=algo)
                if it >= 3:
                    tot[it - 3][1].record()
            spdp.set_profile_events()
            torch.cuda.synchronize()
            ms = statistics.median(a.elapsed_time(b) for a, b in evs)
            ms_tot = statistics.median(a.elapsed_time(b) for a, b in tot)
            same = "ref"
            if ref is None:
                ref = cost.clone()
            else:
                same = "same" if torch.equal(ref, cost) else "DIFF(%d)" % int((ref != cost).sum().item())
            print("%s algo=%s hint=%d mw=%d kernel=%s sweep_ms=%.4f total_ms=%.4f evals/s=%.3e %s" % (
                name, algo or "auto", h, mw, spdp.last_kernel(), ms, ms_tot, cfg["S"] * cfg["T"] / ms_tot * 1e3, same),
                flush=True)
