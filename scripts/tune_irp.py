import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2511_18022_b200 as spdp, synth
dev = torch.device("cuda", 0)
c5 = synth.irp_config()
irp = c5["irp"]
d = spdp.gen_demands(c5["model"], 0, c5["S"], device=dev)
cost = torch.empty(c5["S"], dtype=torch.int64, device=dev)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
for i in range(7):
    if i >= 2: evs[i - 2][0].record()
    spdp.irp_dp(irp["visit"], irp["cust"], d, irp["H"], irp["M"], S=c5["S"], cost=cost)
    if i >= 2: evs[i - 2][1].record()
torch.cuda.synchronize()
print("irp C5 ms %.4f" % statistics.median(a.elapsed_time(b) for a, b in evs))
