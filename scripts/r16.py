"""C2 sensitivity row: r = 16 customers per route (Q 4x larger, windows ~4x)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2511_18022_b200 as spdp, synth
dev = torch.device("cuda", 0)
inst = synth.make_instance(100, 101, r=16.0)
model = synth.demand_model(inst["nominal"], inst["Q"], seed=0x5EED0001)
S = 1_000_000
d = spdp.gen_demands(model, 0, S, device=dev)
tour, dist = torch.from_numpy(inst["tour"]).to(dev), torch.from_numpy(inst["dist"]).to(dev)
m = spdp.split_mask(tour, d, inst["Q"], S=S)
idx = torch.arange(1, 101, device=dev, dtype=torch.int64).unsqueeze(1)
w = (idx - m.to(torch.int64))
print("Q", inst["Q"], "mean window", float(w.float().mean()), "max", int(w.max()))
for algo, h, mw in ((None, 0, 0), ("f32", 32, 16), ("deque", 64, 0), (None, 32, 16), ("int", 64, 0)):
    fn = lambda: spdp.split_eval(tour, dist, d, inst["Q"], S=S, window_hint=h, mean_window=mw, algo=algo)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): fn()
    b.record(); torch.cuda.synchronize()
    print(algo, h, mw, "ms %.4f" % (a.elapsed_time(b) / 10), spdp.last_kernel(), flush=True)
