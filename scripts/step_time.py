"""Step time of spdp.split_eval on C2 with and without the profile-event hook (PDL overlap check)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2511_18022_b200 as spdp, synth
dev = torch.device("cuda", 0)
cfg = synth.config_instance(sys.argv[1] if len(sys.argv) > 1 else "C2")
hint = int(sys.argv[2]) if len(sys.argv) > 2 else 20
inst = cfg["inst"]
S = cfg["S"]
d = spdp.gen_demands(cfg["model"], 0, S, device=dev)
tour = torch.from_numpy(inst["tour"]).to(dev)
dist = torch.from_numpy(inst["dist"]).to(dev)
cost = torch.empty(S, dtype=torch.int32, device=dev)
part = torch.zeros(6, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream(dev)
step = lambda: spdp.split_eval(tour, dist, d, inst["Q"], S=S, window_hint=hint, cost=cost, partial=part)
for _ in range(10):
    step()
torch.cuda.synchronize()
K = 200
for mode in ("plain", "prof", "plain"):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for x, y in evs:
        x.record(st); y.record(st)
    torch.cuda.synchronize()
    a.record(st)
    for k in range(K):
        if mode == "prof":
            spdp.set_profile_events(*evs[k])
        step()
    b.record(st)
    torch.cuda.synchronize()
    spdp.set_profile_events()
    ms = a.elapsed_time(b) / K
    sw = statistics.mean(x.elapsed_time(y) for x, y in evs) if mode == "prof" else float("nan")
    print("%s hint=%d step_ms=%.4f sweep_ms=%.4f evals/s=%.3e" % (mode, hint, ms, sw, S / ms * 1e3), flush=True)
