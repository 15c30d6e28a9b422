"""C4 (n = 1000, 10^6 scenarios) sweep time on the natural and the ordered scenario set."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, bench_config, paper_2511_18022_b200 as spdp
dev = torch.device("cuda")
cfg = synth.config_instance("C4", S=int(sys.argv[1]) if len(sys.argv) > 1 else None); inst = cfg["inst"]
d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
tour = torch.from_numpy(inst["tour"]).to(dev); dist = torch.from_numpy(inst["dist"]).to(dev)
part = torch.zeros(6, dtype=torch.int64, device=dev)
res = {}
for name in ("natural", "ordered"):
    if name == "ordered":
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); d2, _ = spdp.order_scenarios(d, S=cfg["S"]); b.record(); torch.cuda.synchronize()
        print("order_ms %.3f" % a.elapsed_time(b)); d = d2
    fn = lambda: spdp.split_eval(tour, dist, d, inst["Q"], S=cfg["S"], want_cost=False, partial=part,
                                 window_hint=bench_config.HINT["C4"], mean_window=bench_config.MEAN["C4"])
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    res[name] = part.clone()
    print(name, spdp.last_kernel(), "call med %.4f ms" % statistics.median(ts), flush=True)
print("partials equal:", bool(torch.equal(res["natural"], res["ordered"])), res["natural"].tolist())
