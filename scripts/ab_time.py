"""A/B timing of the ordered C2 step and the ordered C3 batch (full call: prep + sweep + finish),
median of 7 repetitions of 20 calls each, plus the sweep alone (profile events)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, bench_config, paper_2511_18022_b200 as spdp
dev = torch.device("cuda")
out = []
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3"]):
    cfg = synth.config_instance(name); inst = cfg["inst"]
    d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
    d, _ = spdp.order_scenarios(d, S=cfg["S"])
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev); dist = torch.from_numpy(inst["dist"]).to(dev)
    h = int(os.environ.get("AB_HINT_" + name, bench_config.HINT[name])); mw = int(os.environ.get("AB_MW_" + name, bench_config.MEAN_ORDERED[name]))
    part = torch.zeros(cfg["T"], 6, dtype=torch.int64, device=dev)
    fn = lambda: spdp.split_eval_batch(tours, dist, d, inst["Q"], S=cfg["S"], want_cost=False, window_hint=h,
                                       mean_window=mw, partial=part)
    for _ in range(3): fn()
    ts = []
    for r in range(7):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): fn()
        b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 20)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev: a.record(); b.record()
    for a, b in ev:
        spdp.set_profile_events(a, b); fn()
    spdp.set_profile_events(); torch.cuda.synchronize()
    sw = statistics.median(a.elapsed_time(b) for a, b in ev)
    out.append("%s %s call med %.4f min %.4f ms, sweep med %.4f ms" % (name, spdp.last_kernel(), statistics.median(ts), min(ts), sw))
print(os.environ.get("AB_TAG", ""), " | ".join(out), flush=True)
