import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, bench_config, paper_2511_18022_b200 as spdp
dev=torch.device("cuda")
for name in ("C2","C3"):
    cfg=synth.config_instance(name); inst=cfg["inst"]
    d=spdp.gen_demands(cfg["model"],0,cfg["S"],device=dev)
    tours=torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev); dist=torch.from_numpy(inst["dist"]).to(dev)
    h=bench_config.HINT[name]; mw=bench_config.MEAN[name]
    fn=lambda: spdp.split_eval_batch(tours,dist,d,inst["Q"],S=cfg["S"],want_cost=False,window_hint=h,mean_window=mw)
    for _ in range(3): fn()
    ts=[]
    for r in range(5):
        a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): fn()
        b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b)/10)
    print(name, spdp.last_kernel(), "min %.4f med %.4f ms" % (min(ts), sorted(ts)[2]))
