import os, sys, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, paper_2511_18022_b200 as spdp
dev = torch.device("cuda")
cfg2 = synth.config_instance("C2"); inst2 = cfg2["inst"]
d0 = spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev)
dO, _ = spdp.order_scenarios(d0, S=cfg2["S"])
xy = np.asarray(inst2["coords"], dtype=np.float64)
distf = torch.from_numpy(np.ascontiguousarray(np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)))).to(dev)
tour2 = torch.from_numpy(inst2["tour"]).to(dev)
costf = torch.empty(cfg2["S"], dtype=torch.float32, device=dev)
for name, d in (("natural", d0), ("ordered", dO)):
    fn = lambda: spdp.split_eval_f32(tour2, distf, d, inst2["Q"], S=cfg2["S"], cost=costf)
    for _ in range(3): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in ev: a.record(); b.record()
    ts = []
    for a, b in ev:
        spdp.set_profile_events(a, b); fn()
    spdp.set_profile_events(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): fn()
    b.record(); torch.cuda.synchronize()
    print(os.environ.get("TAG",""), name, spdp.last_kernel(), "sweep %.4f call %.4f ms" % (statistics.median(x.elapsed_time(y) for x, y in ev), a.elapsed_time(b) / 20))
