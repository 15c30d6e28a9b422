"""Anatomy of one C2 sweep launch (packed-u16 kernel) from the debug timeline (spdp_debug_timeline):
per-warp tile records -> launch-to-first-tile latency, steady tile time, end spread per SM, idle
SM-time in the tail.  Also times the sweep alone (profile events) at several S.

    python scripts/tail_probe.py [S,...] [natural|ordered]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench_config
import paper_2511_18022_b200 as spdp
import synth

dev = torch.device("cuda", 0)
Ss = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1000000]
order = sys.argv[2] if len(sys.argv) > 2 else "ordered"
# event overhead of a trivial kernel (the floor of any event-timed launch)
_x = torch.zeros(1, device=dev)
_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
for a, b in _ev:
    a.record()
    _x.add_(1)
    b.record()
torch.cuda.synchronize()
print("trivial kernel, event-timed: median %.2f us" % (1e3 * statistics.median(a.elapsed_time(b) for a, b in _ev)))
for S in Ss:
    cfg = synth.config_instance("C2", S=S)
    inst = cfg["inst"]
    d = spdp.gen_demands(cfg["model"], 0, S, device=dev)
    mean = bench_config.MEAN["C2"]
    if order == "ordered":
        d, _ = spdp.order_scenarios(d, S=S)
        mean = bench_config.MEAN_ORDERED["C2"]
    tour = torch.from_numpy(inst["tour"]).to(dev)
    dist = torch.from_numpy(inst["dist"]).to(dev)
    cost = torch.empty(S, dtype=torch.int32, device=dev)
    part = torch.zeros(4, dtype=torch.int64, device=dev)

    def run():
        spdp.split_eval(tour, dist, d, inst["Q"], S=S, window_hint=bench_config.HINT["C2"], mean_window=mean,
                        cost=cost, partial=part)

    for _ in range(5):
        run()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in evs:
        a.record()
        b.record()
    for a, b in evs:
        spdp.set_profile_events(a, b)
        run()
    spdp.set_profile_events()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    print("S=%d order=%s kernel=%s sweep_us median=%.2f mean=%.2f min=%.2f" % (
        S, order, spdp.last_kernel(), 1e3 * statistics.median(ms), 1e3 * statistics.mean(ms), 1e3 * min(ms)), flush=True)
    ntiles = (S + 255) // 256
    buf = torch.zeros(2 + 4 * (ntiles * 4 + 8 * 600), dtype=torch.int64, device=dev)
    spdp.debug_timeline(buf)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    en.record()
    spdp.set_profile_events(st, en)
    run()
    spdp.set_profile_events()
    torch.cuda.synchronize()
    spdp.debug_timeline()
    run()
    torch.cuda.synchronize()
    nrec = int(buf[0].item())
    r = buf[2:2 + 4 * nrec].view(nrec, 4).cpu().numpy().astype(np.int64)
    kind = r[:, 1] & 0xffffffff
    cta_start = r[kind == 0xfffffff0, 2]
    warp_done = r[kind == 0xfffffff1, 2]
    r = r[kind < 0xfffffff0]
    nrec = len(r)
    base = r[:, 2].min()
    print("  CTA start rel. first tile: min %.2f max %.2f us; warp done after flush: max %.2f us" % (
        (cta_start.min() - base) / 1e3, (cta_start.max() - base) / 1e3, (warp_done.max() - base) / 1e3))
    # gaps between consecutive tiles of a warp
    slot_ = r[:, 0] & 0xffff
    gaps = []
    for s_ in np.unique(slot_):
        rr = r[slot_ == s_]
        rr = rr[np.argsort(rr[:, 2])]
        gaps.extend((rr[1:, 2] - rr[:-1, 3]).tolist())
    gaps = np.array(gaps if gaps else [0])
    print("  tile-switch gap: median %.2f p90 %.2f us, total %.1f%% of warp time" % (
        np.median(gaps) / 1e3, np.percentile(gaps, 90) / 1e3, 100.0 * gaps.sum() / (r[:, 3] - r[:, 2]).sum()))
    sm = r[:, 0] >> 16
    slot = r[:, 0] & 0xffff
    t0 = r[:, 2] - r[:, 2].min()
    t1 = r[:, 3] - r[:, 2].min()
    dur = t1 - t0
    T = t1.max()
    print("  timeline: %d warp-tiles, launch (event) %.2f us, first tile start..last end %.2f us" % (
        nrec, 1e3 * st.elapsed_time(en), T / 1e3))
    print("  first starts: min %.2f med %.2f max %.2f us (relative to the first)" % (
        0, np.median(np.sort(t0)[:4 * 592]) / 1e3, np.sort(t0)[min(len(t0), 4 * 592) - 1] / 1e3))
    print("  warp-tile duration: median %.2f p10 %.2f p90 %.2f max %.2f us" % tuple(
        x / 1e3 for x in (np.median(dur), np.percentile(dur, 10), np.percentile(dur, 90), dur.max())))
    # per-warp slot end, per-SM end
    ends = {}
    for s_, e_ in zip(slot, t1):
        ends[s_] = max(ends.get(s_, 0), e_)
    we = np.array(sorted(ends.values()))
    print("  warp end: p10 %.2f median %.2f p90 %.2f max %.2f us" % tuple(
        x / 1e3 for x in (np.percentile(we, 10), np.median(we), np.percentile(we, 90), we.max())))
    sme = {}
    for s_, e_ in zip(sm, t1):
        sme[s_] = max(sme.get(s_, 0), e_)
    se = np.array(sorted(sme.values()))
    print("  SM end: min %.2f median %.2f max %.2f us; busy warp-time / (warps x span) = %.3f" % (
        se.min() / 1e3, np.median(se) / 1e3, se.max() / 1e3, dur.sum() / (len(ends) * T)))
    # active warps over time (histogram in 2 us bins)
    bins = np.arange(0, T + 2000, 2000)
    act = [int(((t0 < b + 1000) & (t1 > b + 1000)).sum()) for b in bins]
    print("  active warps per 2us:", " ".join(str(a) for a in act))
    # tile time vs slot-in-SM (warp slot % 16 within the SM's CTAs)
    by = {}
    for s_, du in zip(slot % 4, dur):
        by.setdefault(int(s_), []).append(du)
    print("  duration by warp-in-CTA:", {k: round(float(np.median(v)) / 1e3, 2) for k, v in sorted(by.items())})
    cta = slot // 4
    byc = {}
    for c_, du in zip(cta % 4, dur):
        byc.setdefault(int(c_), []).append(du)
    print("  duration by CTA % 4:", {k: round(float(np.median(v)) / 1e3, 2) for k, v in sorted(byc.items())})
    cnt = np.bincount(slot)
    print("  tiles per warp: min %d median %d max %d" % (cnt[cnt > 0].min(), np.median(cnt[cnt > 0]), cnt.max()))
