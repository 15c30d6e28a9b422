"""Overflow-list size of the sweep (scenarios deferred to the finish kernel) per config/hint/algorithm."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2511_18022_b200 as spdp, synth
dev = torch.device("cuda", 0)
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3", "C4"]
hints = [int(h) for h in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 20, 32]
algos = sys.argv[3].split(",") if len(sys.argv) > 3 else ["int", "f32"]
for name in cfgs:
    cfg = synth.config_instance(name)
    inst = cfg["inst"]
    d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
    dist = torch.from_numpy(inst["dist"]).to(dev)
    for h in hints:
        for algo in algos:
            spdp.split_eval_batch(tours, dist, d, inst["Q"], S=cfg["S"], window_hint=h, want_cost=False, algo=algo)
            torch.cuda.synchronize()
            ws = [v for k, v in spdp._WS.items() if k[-1] == "split"][0]
            hdr = ws[:16].cpu().numpy().view(np.uint32)
            print(name, "hint", h, algo, "ovf_count", hdr[0], "of", cfg["S"] * cfg["T"], flush=True)
