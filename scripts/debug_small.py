import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2511_18022_b200 as spdp, synth
cfg = synth.config_instance("C2", S=5000)
inst = cfg["inst"]
d = spdp.gen_demands(cfg["model"], 0, 5000)
c, p = spdp.split_eval(torch.from_numpy(inst["tour"]).cuda(), torch.from_numpy(inst["dist"]).cuda(), d, inst["Q"], S=5000, window_hint=20)
torch.cuda.synchronize()
print("ok", c[:5].tolist())
