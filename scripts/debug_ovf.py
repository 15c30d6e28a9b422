import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2511_18022_b200 as spdp, synth
dev = torch.device("cuda", 0)
for name in ["C2", "C3", "C4"]:
    cfg = synth.config_instance(name)
    inst = cfg["inst"]
    d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
    dist = torch.from_numpy(inst["dist"]).to(dev)
    for h in (16, 32, 64):
        spdp.split_eval_batch(tours, dist, d, inst["Q"], S=cfg["S"], window_hint=h, want_cost=False)
        torch.cuda.synchronize()
        ws = [v for k, v in spdp._WS.items() if k[1] == "split"][0]
        hdr = ws[:16].cpu().numpy().view(np.uint32)
        print(name, "hint", h, "ovf_count", hdr[0], "of", cfg["S"] * cfg["T"], flush=True)
