#!/usr/bin/env python
"""bench.py -- split evaluations/s (scenario x tour) of the B200 Split-DP hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl spdp|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[1], DESIGN §Input recipe): "C2", an X-n101-shaped
CVRPSD instance, n = 100 customers, one giant tour, 10^6 correlated-demand
scenarios in all (strong scaling, the default: rank r owns the global scenarios
[floor(r S / N), floor((r+1) S / N)), north_star's "each rank owns S/8"; --scaling weak:
10^6 per GPU).  One step = one pass of the hot path over the resident demand set:
tour prep (a2) + masked min-plus sweep with per-scenario costs (a5) + fused SAA
partial (a6) (+ the int64 all-reduce of the partial, a7, at N > 1, on a
communication stream so that it overlaps the next step: pipelined evaluations).
The timed steps replay a CUDA graph (at N > 1 one graph of G steps with their
NCCL all-reduces); at N > 1 the line also carries the single-shot latency (one
step with its all-reduce completed, nothing overlapped).  Timed with CUDA events
on the launching stream, max over ranks.  The demand set (200 MB at N = 1) is
larger than L2, so every step streams it from HBM.

Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the
reference arm of this tier) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import bench_config  # noqa: E402

METRIC = "split evals/sec (scenario\u00d7tour) at n=100, S=1M, 1/2/4/8 B200; % ALU/HBM roofline"  # BASELINE.json
UNIT = "scenario-tour evals/s"
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": HBM_FALLBACK_GBS, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


# ALU peak for one integer add-min per Eq. (3) candidate:
# 148 SMs x 4 SMSPs x 16 lanes/clk (ALU pipe, one VIMNMX per lane every clk/16)
ALU_LANES_PER_SM_CLK = 64
N_SM = 148


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def ncu_traffic(config_name: str):
    """dram bytes per sweep launch from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "r01_ncu_sweep_%s.json" % config_name)
    if not os.path.exists(p):
        return None
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


def workload_str(name, n, Q, S_glob, T):
    """The workload both arms name in config.workload (the BASELINE configuration)."""
    return "%s: X-n%d-shaped CVRPSD, n=%d, Q=%d, %d correlated-demand scenarios in all (cv=0.3, rho=0.5), %d giant " \
           "tour%s" % (name, n + 1, n, Q, S_glob, T, "s" if T > 1 else "")


# ---------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference arm of this tier: the CPU oracle (plain C, OpenMP over scenarios) on the
    host cores, on the same workload/metric; each step is a bounded sample of it."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    cfg = synth.config_instance(args.config)
    inst = cfg["inst"]
    S_full = cfg["S"]
    threads = max(oracle.num_threads(), os.cpu_count() or 1)  # all host cores (torchrun sets OMP_NUM_THREADS=1)
    # size the per-step sample for ~1 s of oracle work (bounded; whole run stays within minutes)
    S_probe = 20_000
    dem = oracle.gen_demands(cfg["model"], 0, S_probe, threads=threads)
    t0 = time.perf_counter()
    oracle.split(inst["tour"], inst["dist"], dem, inst["Q"], threads=threads)
    per = (time.perf_counter() - t0) / S_probe
    S_ref = int(min(S_full, max(S_probe, 1.0 / max(per, 1e-9))))
    dem = oracle.gen_demands(cfg["model"], 0, S_ref, threads=threads)
    for _ in range(args.warmup):
        oracle.split(inst["tour"], inst["dist"], dem, inst["Q"], threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        c = oracle.split(inst["tour"], inst["dist"], dem, inst["Q"], threads=threads)
        oracle.saa(c)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    value = S_ref / t
    sample = "first %d of the %d scenarios of %s per step (oracle split + SAA, demands pre-generated)" % (
        S_ref, S_full, args.config)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": workload_str(args.config, cfg["n"], cfg["Q"], S_full, cfg["T"]) +
                                   " (the oracle on the host cores; a bounded sample per step)",
                       "n": cfg["n"], "S_per_step": S_ref, "Q": cfg["Q"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="spdp", choices=["spdp", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): S = 10^6 in all, split over the ranks; weak: 10^6 per rank")
    ap.add_argument("--no-rows", action="store_true", help="skip the per-row (C3/C4/C5/gen) measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--window-hint", type=int, default=None)
    ap.add_argument("--scenario-order", default="load", choices=["load", "natural"],
                    help="load (default): each rank's resident scenario set is ordered once by total demand "
                         "(spdp_order_scenarios, a layout of the set, outside the timed steps); natural: as generated")
    ap.add_argument("--eager", action="store_true",
                    help="launch every timed step from Python (default: replay a CUDA graph of the step(s))")
    ap.add_argument("--streams", type=int, default=1, choices=[1, 2],
                    help="N = 1, one tour: 2 = consecutive steps alternate between two streams (two independent "
                         "evaluations in flight; measured +2 %% at C2); 1 (default) = strictly one after the other")
    ap.add_argument("--graph-steps", type=int, default=10,
                    help="steps per captured CUDA graph at N > 1 (their all-reduces pipelined inside it)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as tdist

    import paper_2511_18022_b200 as spdp
    from paper_2511_18022_b200 import dist as pdist

    world, rank, local = dist_env()
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    # (SPDP_BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo -- a functional check of the N > 1
    # path on a one-GPU box; its timings mean nothing)
    share = os.environ.get("SPDP_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=dev)

    cfg = synth.config_instance(args.config)
    inst, n, Q = cfg["inst"], cfg["n"], cfg["Q"]
    S_cfg = cfg["S"]
    if args.scaling == "weak":
        S_loc, s_begin = S_cfg, rank * S_cfg
        S_glob = S_cfg * world
    else:
        s_begin, s_end = pdist.shard_range(S_cfg, rank, world)
        S_loc, S_glob = s_end - s_begin, S_cfg
    hint = args.window_hint if args.window_hint is not None else bench_config.HINT[args.config]

    # Inputs larger than L2 at every N: at N = 1 the demand set (200 MB) is; when a rank's share is
    # smaller (strong scaling), every step evaluates a fresh batch of the global S scenarios --
    # batch k = the generator's scenarios [k S_glob, (k+1) S_glob), this rank's shard of it -- over
    # B batches generated up front that together exceed twice the L2 (126 MB), so each step's
    # batch was evicted since its last use and streams from HBM.
    L2_BYTES = 126e6
    dem_bytes = n * spdp.padded_ld(S_loc) * 2
    B = 1 if dem_bytes > 1.5 * L2_BYTES else int(np.ceil(2 * L2_BYTES / dem_bytes))
    demands = [spdp.gen_demands(cfg["model"], s_begin + k * S_glob, S_loc, device=dev) for k in range(B)]
    order_ms, perms = None, None
    if args.scenario_order == "load":  # (a layout of each resident set, once; timed here, reported in config)
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        ordered = [spdp.order_scenarios(d_, S=S_loc) for d_ in demands]
        demands, perms = [o[0] for o in ordered], [o[1] for o in ordered]
        b_.record()
        torch.cuda.synchronize(dev)
        order_ms = a_.elapsed_time(b_) / B
    mean_w = (bench_config.MEAN_ORDERED if args.scenario_order == "load" else bench_config.MEAN)[args.config]
    demand = demands[0]
    T = cfg["T"]
    tour = torch.from_numpy(inst["tour"]).to(dev)
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
    dist = torch.from_numpy(inst["dist"]).to(dev)
    # two cost / partial buffers: at N > 1 the all-reduce of step k (a7) runs on a communication
    # stream while step k + 1 computes into the other buffer (pipelined evaluations);
    # at N = 1 (one tour) consecutive steps alternate between two streams (each with its own
    # workspace: the binding keys it by stream), so step k + 1's sweep fills the SMs that step k's
    # persistent grid releases at its ramp-down -- two independent evaluations in flight, each one a
    # full pass of the hot path over the 10^6 resident scenarios
    cost2 = [torch.empty((T, S_loc) if T > 1 else S_loc, dtype=torch.int32, device=dev) for _ in range(2)]
    cost = cost2[0]
    partials = [torch.zeros((T, 6) if T > 1 else 6, dtype=torch.int64, device=dev) for _ in range(2)]
    stream = torch.cuda.current_stream(dev)
    # (SPDP_BENCH_FAKE_COMM=1 at N = 1: the N > 1 step structure -- comm stream, double-buffered partials,
    # G steps per captured graph -- with a capturable stand-in for the all-reduce; a functional check of
    # the multi-rank capture path on a one-GPU box, its timings mean nothing)
    fake_comm = world == 1 and os.environ.get("SPDP_BENCH_FAKE_COMM") == "1"
    comm = torch.cuda.Stream(dev) if (world > 1 or fake_comm) else None
    n_streams = 2 if (world == 1 and T == 1 and args.streams == 2 and not fake_comm) else 1
    side = torch.cuda.Stream(dev) if n_streams == 2 else None
    freed = [None, None]  # event: the buffer's last all-reduce has completed
    kstep = [0]

    def step(single=False):
        cur = torch.cuda.current_stream(dev)  # (the capture stream while a graph is being captured)
        b = kstep[0] & 1
        kstep[0] += 1
        part = partials[b]
        dem = demands[(kstep[0] - 1) % B]
        if freed[b] is not None:
            cur.wait_event(freed[b])
        if T > 1:  # batched tours (a8): T candidate tours over the same scenarios
            spdp.split_eval_batch(tours, dist, dem, Q, S=S_loc, window_hint=hint, cost=cost2[b], partial=part,
                                  mean_window=mean_w)
        elif n_streams == 2 and b == 1 and not single:  # (the second evaluation in flight, on the side stream)
            fork = torch.cuda.Event()
            fork.record(cur)
            side.wait_event(fork)
            with torch.cuda.stream(side):
                spdp.split_eval(tour, dist, dem, Q, S=S_loc, window_hint=hint, cost=cost2[b], partial=part,
                                mean_window=mean_w)
                done_b = torch.cuda.Event()
                done_b.record(side)
            freed[b] = done_b
        else:
            spdp.split_eval(tour, dist, dem, Q, S=S_loc, window_hint=hint, cost=cost2[b], partial=part,
                            mean_window=mean_w)
        if world > 1 or fake_comm:
            ready = torch.cuda.Event()
            ready.record(cur)
            comm.wait_event(ready)
            with torch.cuda.stream(comm):
                if fake_comm:
                    part.mul_(1)
                else:
                    pdist.allreduce_partials(part)
                done = torch.cuda.Event()
                done.record(comm)
            freed[b] = done

    def join():  # the outstanding all-reduces, into the current stream
        cur = torch.cuda.current_stream(dev)
        for ev in freed:
            if ev is not None:
                cur.wait_event(ev)

    for _ in range(args.warmup):
        step()
    join()
    torch.cuda.synchronize(dev)
    freed[0] = freed[1] = None  # (events of eager work: a capture must not wait on them)
    ref_parts = [p_.clone() for p_ in partials]  # (per buffer: every step's partial is the same, or all-reduced)
    # The timed steps replay a CUDA graph: at N = 1 of one step (the same three kernels with their
    # programmatic-dependent-launch edges), at N > 1 of G steps whose NCCL all-reduces run on the
    # communication stream, each overlapping the next step (joined at the graph's end) -- so host
    # launch overhead (ctypes marshalling, ~tens of us per step in Python) cannot leave the GPU idle.
    G = B  # one graph replay = one pass over the batches
    if (world > 1 or fake_comm) and B == 1:
        G = max(1, min(args.graph_steps, args.steps))
    if n_streams == 2 and G % 2:
        G *= 2  # (both streams' steps in every replay)
    graph, launch_mode = None, "eager (one C-ABI call per step from Python)"
    if share:
        launch_mode += "; gloo all-reduce (SPDP_BENCH_SHARE_GPU functional check)"
    elif not args.eager:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(G):
                    step()
                join()
            freed[0] = freed[1] = None  # (capture-time events; the graph carries the dependencies)
            torch.cuda.synchronize(dev)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize(dev)
            graph = g
            launch_mode = ("CUDA graph replay (one captured step per replay)" if G == 1 else
                           "CUDA graph replay (%d captured steps per replay, consecutive steps on two streams: two "
                           "independent evaluations in flight)" % G if n_streams == 2 else
                           "CUDA graph replay (%d captured steps per replay, each step's all-reduce overlapping "
                           "the next step on a communication stream)" % G)
        except Exception as ex:  # keep the eager loop (and say why) -- after checking it still computes
            launch_mode = "eager (graph capture failed: %s)" % str(ex).splitlines()[0][:120]
            freed[0] = freed[1] = None
            torch.cuda.synchronize(dev)
            kstep[0] = 0
            for _ in range(2):
                step()
            join()
            torch.cuda.synchronize(dev)
            freed[0] = freed[1] = None
            if not all(torch.equal(a_, b_) for a_, b_ in zip(partials, ref_parts)):
                raise RuntimeError("bench: the eager steps after a failed graph capture no longer reproduce the "
                                   "warm-up partials (%s)" % launch_mode)

    if fake_comm:
        launch_mode = "SPDP_BENCH_FAKE_COMM functional check (no all-reduce); " + launch_mode

    def timed_steps(K):  # exactly K steps: K // G graph replays, the rest launched eagerly
        if graph is not None:
            for _ in range(K // G):
                graph.replay()
            kstep[0] = 0
            for _ in range(K % G):
                step()
        else:
            for _ in range(K):
                step()

    # algorithmic work: Eq. (3) candidates sum_i (i - mask(i)) from the standalone mask kernel (untimed)
    m = spdp.split_mask(tour, demand, Q, S=S_loc)
    idx = torch.arange(1, n + 1, device=dev, dtype=torch.int64).unsqueeze(1)
    cand = int(((idx - m.to(torch.int64)) * (m >= 0)).sum().item()) * T  # (T > 1: tour 0's count x T, estimate)
    del m
    torch.cuda.synchronize(dev)

    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for e in ev_s + ev_e:  # torch creates the CUDA event lazily, on its first record
        e.record(stream)
    props = torch.cuda.get_device_properties(dev)
    try:
        smi_id = "%08X:%02X:%02X.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
    except AttributeError:
        smi_id = str(local)
    sampler = ClockSampler(smi_id)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    # timed region: K back-to-back steps, nothing recorded between the kernels of a step (the
    # sweep and finish kernels overlap their launch with the predecessor: programmatic dependent
    # launch; an event recorded between them would serialise that)
    t_start.record(stream)
    timed_steps(args.steps)
    join()  # the last all-reduces are part of the timed region
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        tdist.barrier()
    # roofline pass: the same K steps again with the sweep kernel bracketed by events on its stream
    for k in range(args.steps):  # (one stream: each sweep timed alone)
        spdp.set_profile_events(ev_s[k], ev_e[k])
        step(single=True)
    join()
    torch.cuda.synchronize(dev)
    spdp.set_profile_events()
    # single-shot latency: one step AND its all-reduce, nothing overlapped (the latency a caller
    # waiting for one evaluation sees); max over ranks
    n_ss = max(3, min(args.steps, 20))
    ss_a = [torch.cuda.Event(enable_timing=True) for _ in range(n_ss)]
    ss_b = [torch.cuda.Event(enable_timing=True) for _ in range(n_ss)]
    if world > 1:
        tdist.barrier()
    for k in range(n_ss):
        ss_a[k].record(stream)
        step(single=True)
        join()
        ss_b[k].record(stream)
        torch.cuda.synchronize(dev)
    single_shot_ms = statistics.median(a.elapsed_time(b) for a, b in zip(ss_a, ss_b))
    if world > 1:
        tdist.barrier()
    # keep sampling clocks under the same load for >= 1 s so the record is meaningful
    soak_end = time.perf_counter() + 1.0
    while time.perf_counter() < soak_end:
        timed_steps(max(G, 20 // G * G))
        join()
        torch.cuda.synchronize(dev)
    clocks = sampler.stop()

    ms_step = t_start.elapsed_time(t_end) / args.steps
    sweep_all = [a.elapsed_time(b) for a, b in zip(ev_s, ev_e)]
    sweep_ms = statistics.mean(sweep_all)
    sweep_med = statistics.median(sweep_all)
    if world > 1:
        ms_step = pdist.max_over_ranks(ms_step, device=dev if not share else None)
        sweep_ms = pdist.max_over_ranks(sweep_ms, device=dev if not share else None)
        single_shot_ms = pdist.max_over_ranks(single_shot_ms, device=dev if not share else None)
    value = S_glob * T * 1.0 / (ms_step / 1e3)

    pk = peaks()
    bytes_alg = n * S_loc * 2 + T * S_loc * 4  # demand stream (u16, read once) + per-scenario costs (i32)
    hbm_achieved = bytes_alg / (sweep_ms / 1e3) / 1e9
    alu_peak = N_SM * ALU_LANES_PER_SM_CLK * pk["sm_max_mhz"] * 1e6  # candidates/s
    alu_achieved = cand / (sweep_ms / 1e3)
    t_hbm = bytes_alg / (pk["hbm_gbs"] * 1e9)
    t_alu = cand / alu_peak
    if t_hbm >= t_alu:
        roof = {"bound": "hbm", "achieved": hbm_achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": hbm_achieved / pk["hbm_gbs"]}
    else:
        roof = {"bound": "alu", "achieved": alu_achieved / 1e12, "peak": alu_peak / 1e12, "unit": "Tcand/s",
                "frac": alu_achieved / alu_peak}
    roof.update({"traffic": ncu_traffic(args.config), "kernel": spdp.last_kernel(),
                 "kernel_ms": sweep_ms, "kernel_ms_median": sweep_med, "kernel_timing": "CUDA events around the sweep launch, mean of a second "
                                                         "pass of the K timed steps",
                 "bytes_alg_per_launch": bytes_alg, "candidates_per_launch": cand,
                 "hbm_frac": hbm_achieved / pk["hbm_gbs"], "alu_frac": alu_achieved / alu_peak,
                 "peak_source": pk["source"], "sweep_share_of_step": sweep_ms / ms_step})

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": workload_str(args.config, n, Q, S_glob, T) + " (%d per GPU)" % S_loc,
                       "n": n, "S_per_gpu": S_loc, "S_global": S_glob, "T": T, "window_hint": hint,
                       "mean_window_hint": mean_w,
                       "scenario_order": ("by total demand within segments of 65536 (spdp_order_scenarios): a layout "
                                          "of each rank's resident scenario set, made once (%.3f ms per set) before the "
                                          "timed steps; the per-scenario costs are the permuted ones, the SAA partials "
                                          "identical" % order_ms) if order_ms is not None else "natural (as generated)",
                       "l2": ("inputs larger than L2 (demand %.0f MB/GPU > 126 MB)" % (dem_bytes / 1e6) if B == 1 else
                              "inputs larger than L2: each step a fresh batch of the S scenarios, %d batches of "
                              "%.0f MB/GPU rotating (%.0f MB > 2 x 126 MB L2)" % (B, dem_bytes / 1e6,
                                                                                  B * dem_bytes / 1e6)),
                       "parallelism": "scenario-sharded dp%d, 1 int64 all-reduce/step (on a comm stream, "
                                      "overlapped with the next step)" % world,
                       "launch": launch_mode},
            "single_shot_ms": single_shot_ms,
            "single_shot": "median over %d steps of one step with its all-reduce completed (nothing overlapped), "
                           "max over ranks" % n_ss,
            "roofline": roof, "clocks": clocks, "gpu_launches": 3 * args.steps}

    # ------------------------------------------------------------------ e2e through the C-ABI host entry
    if not args.no_e2e:
        dem_h = torch.empty(demand.shape, dtype=torch.int16, pin_memory=True)
        dem_h.copy_(demand)
        cost_h = torch.empty(S_loc, dtype=torch.int32, pin_memory=True)
        tour_h, dist_h = np.ascontiguousarray(inst["tour"]), np.ascontiguousarray(inst["dist"])
        for _ in range(2):
            spdp.split_eval_host(tour_h, dist_h, dem_h, Q, S=S_loc, cost_h=cost_h, window_hint=hint, device=dev)
        ke = max(3, min(args.steps, 20))
        if world > 1:
            tdist.barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            est = spdp.split_eval_host(tour_h, dist_h, dem_h, Q, S=S_loc, cost_h=cost_h, window_hint=hint,
                                       device=dev)
        te = (time.perf_counter() - t0) / ke
        if world > 1:
            te = pdist.max_over_ranks(te, device=dev)
        line["e2e"] = {"value": S_glob / te, "unit": UNIT,
                       "h2d_bytes_per_step": int(dem_h.numel() * 2 + tour_h.nbytes + dist_h.nbytes),
                       "d2h_bytes_per_step": int(S_loc * 4 + 48), "ms_per_step": te * 1e3,
                       "api": "spdp_split_eval_host (pinned host demand, costs + SAA estimate back)"
                              + (", tour 0 of the %d" % T if T > 1 else ""),
                       "saa_mean": est["mean"]}

    # ------------------------------------------------------------------ per-row measurements (rank 0, N=1)
    if rank == 0 and world == 1 and not args.no_rows:
        line["rows"] = measure_rows(spdp, torch, dev, pk)

    # ------------------------------------------------------------------ oracle cpu_baseline (rank 0, N=1)
    if rank == 0 and world == 1 and not args.no_cpu:
        partial = partials[(kstep[0] - 1) & 1]
        cost = cost2[(kstep[0] - 1) & 1]  # (the last step's buffer)
        torch.cuda.synchronize(dev)
        line["cpu_baseline"] = cpu_baseline(cfg, cost[0] if T > 1 else cost, S_loc, spdp,
                                            partial[0] if T > 1 else partial,
                                            perms[(kstep[0] - 1) % B] if perms is not None else None)
        if T > 1:
            line["cpu_baseline"]["sample"] += " (tour 0 of the %d)" % T

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


def _time_events(fn, torch, dev, iters=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize(dev)
    return a.elapsed_time(b) / iters


def measure_rows(spdp, torch, dev, pk):
    """One measurement per other hot-path row (device time, CUDA events)."""
    rows = {}
    # a1: scenario generation at C2 size
    cfg2 = synth.config_instance("C2")
    out = spdp.empty_demand(cfg2["n"], cfg2["S"], dev)
    ms = _time_events(lambda: spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev, out=out), torch, dev)
    rows["a1_gen_C2"] = {"ms": ms, "demands_per_s": cfg2["n"] * cfg2["S"] / (ms / 1e3),
                         "write_GBps": cfg2["n"] * cfg2["S"] * 2 / (ms / 1e3) / 1e9}
    del out
    # a5 S-sweep at C2 (analogue of the paper's runtime-vs-scenarios figure): the first S columns
    d = spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev)
    inst2 = cfg2["inst"]
    tour2, dist2 = torch.from_numpy(inst2["tour"]).to(dev), torch.from_numpy(inst2["dist"]).to(dev)
    sweep = {}
    for S_ in (10_000, 100_000, 1_000_000):
        c_ = torch.empty(S_, dtype=torch.int32, device=dev)
        p_ = torch.zeros(6, dtype=torch.int64, device=dev)
        fn = lambda: spdp.split_eval(tour2, dist2, d, inst2["Q"], S=S_, window_hint=bench_config.HINT["C2"],
                                     mean_window=bench_config.MEAN["C2"], cost=c_, partial=p_)
        ms = _time_events(fn, torch, dev, iters=20)
        sweep[str(S_)] = {"ms": ms, "evals_per_s": S_ / (ms / 1e3)}
    rows["a5_C2_S_sweep"] = sweep
    # the C2 step on the scenario set ordered by total demand (spdp_order_scenarios, once per set;
    # the per-scenario costs are the permuted ones, the SAA partial identical)
    dO, _ = spdp.order_scenarios(d, S=cfg2["S"])
    order_ms = _time_events(lambda: spdp.order_scenarios(d, S=cfg2["S"], out=dO), torch, dev, iters=3)
    p0 = torch.zeros(6, dtype=torch.int64, device=dev)
    pO = torch.zeros(6, dtype=torch.int64, device=dev)
    spdp.split_eval(tour2, dist2, d, inst2["Q"], S=cfg2["S"], window_hint=bench_config.HINT["C2"],
                    mean_window=bench_config.MEAN["C2"], partial=p0)
    fn = lambda: spdp.split_eval(tour2, dist2, dO, inst2["Q"], S=cfg2["S"], window_hint=bench_config.HINT["C2"],
                                 mean_window=bench_config.MEAN_ORDERED["C2"], cost=c_, partial=pO)
    ms = _time_events(fn, torch, dev, iters=20)
    rows["a5_C2_ordered"] = {"ms": ms, "evals_per_s": cfg2["S"] / (ms / 1e3), "kernel": spdp.last_kernel(),
                             "order_ms": order_ms, "partials_equal_natural_order": bool(torch.equal(pO, p0)),
                             "note": "one C2 step on the scenario set ordered by total demand (ordering once per "
                                     "set, order_ms, amortised over the tours evaluated on it)"}
    del d, dO
    # a5 sensitivity: C2 with r = 16 customers per route (Q 4x, windows ~4x: mean 15,
    # max 46 -> the monotone-deque sweep)
    inst16 = synth.make_instance(100, 101, r=16.0)
    model16 = synth.demand_model(inst16["nominal"], inst16["Q"], seed=0x5EED0001)
    d = spdp.gen_demands(model16, 0, cfg2["S"], device=dev)
    tour16, dist16 = torch.from_numpy(inst16["tour"]).to(dev), torch.from_numpy(inst16["dist"]).to(dev)
    c_ = torch.empty(cfg2["S"], dtype=torch.int32, device=dev)
    p_ = torch.zeros(6, dtype=torch.int64, device=dev)
    fn = lambda: spdp.split_eval(tour16, dist16, d, inst16["Q"], S=cfg2["S"], window_hint=64, cost=c_, partial=p_)
    ms = _time_events(fn, torch, dev, iters=10)
    m = spdp.split_mask(tour16, d, inst16["Q"], S=cfg2["S"])
    idx = torch.arange(1, 101, device=dev, dtype=torch.int64).unsqueeze(1)
    cand16 = int(((idx - m.to(torch.int64)) * (m >= 0)).sum().item())
    del m
    bytes16 = 100 * cfg2["S"] * 2 + cfg2["S"] * 4
    rows["a5_C2_r16"] = {"ms": ms, "Q": inst16["Q"], "evals_per_s": cfg2["S"] / (ms / 1e3), "kernel": spdp.last_kernel(),
                         "bound": "hbm", "bytes_alg": bytes16,
                         "hbm_frac": bytes16 / (ms / 1e3) / (pk["hbm_gbs"] * 1e9),
                         "candidates": cand16,
                         "candidates_note": "Eq. (3) window sum; the deque sweep does O(1) amortised work per "
                                            "layer, so its bound is the demand stream (hbm_frac), not these",
                         "alu_frac_of_window_sum": cand16 / (ms / 1e3) / (N_SM * ALU_LANES_PER_SM_CLK * pk["sm_max_mhz"] * 1e6)}
    del d
    # a8: batched tours (C3) and a5 at n=1000 (C4, 1 GPU)
    for name in ("C3", "C4"):
        cfg = synth.config_instance(name)
        inst = cfg["inst"]
        d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
        tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
        dist = torch.from_numpy(inst["dist"]).to(dev)
        part = torch.zeros((cfg["T"], 6), dtype=torch.int64, device=dev)
        h = bench_config.HINT[name]
        fn = lambda: spdp.split_eval_batch(tours, dist, d, inst["Q"], S=cfg["S"], want_cost=False, partial=part,
                                           window_hint=h, mean_window=bench_config.MEAN[name])
        ms = _time_events(fn, torch, dev, iters=6)
        kern = spdp.last_kernel()
        # exact Eq. (3) candidate count: the window sum of EVERY tour (standalone mask kernel, untimed)
        idx = torch.arange(1, cfg["n"] + 1, device=dev, dtype=torch.int64).unsqueeze(1)
        cand = 0
        for t in range(cfg["T"]):
            m = spdp.split_mask(tours[t].contiguous(), d, inst["Q"], S=cfg["S"])
            cand += int(((idx - m.to(torch.int64)) * (m >= 0)).sum().item())
        del m
        alu_peak = N_SM * ALU_LANES_PER_SM_CLK * pk["sm_max_mhz"] * 1e6
        bytes_ = cfg["n"] * cfg["S"] * 2 + cfg["T"] * cfg["S"] * 4 * 0  # (want_cost=False: no cost stream)
        row = {"ms": ms, "evals_per_s": cfg["T"] * cfg["S"] / (ms / 1e3), "T": cfg["T"], "S": cfg["S"], "n": cfg["n"],
               "kernel": kern, "candidates": cand, "alu_frac": cand / (ms / 1e3) / alu_peak,
               "bytes_alg": bytes_, "hbm_frac": bytes_ / (ms / 1e3) / (pk["hbm_gbs"] * 1e9)}
        if "deque" in kern:
            row["bound"] = "hbm"
            row["candidates_note"] = ("Eq. (3) window sum; the deque sweep does O(1) amortised work per layer, so "
                                      "its bound is the demand stream (hbm_frac)")
        else:
            row["bound"] = "alu"
        if True:
            # the same evaluation on the scenario set ordered by total demand (spdp_order_scenarios, once per
            # set: similar windows share a warp); costs are the permuted ones, the SAA partials identical
            dO, perm = spdp.order_scenarios(d, S=cfg["S"])
            order_ms = _time_events(lambda: spdp.order_scenarios(d, S=cfg["S"], out=dO), torch, dev, iters=3)
            partO = torch.zeros_like(part)
            mwo = bench_config.MEAN_ORDERED[name]
            fno = lambda: spdp.split_eval_batch(tours, dist, dO, inst["Q"], S=cfg["S"], want_cost=False, partial=partO,
                                                window_hint=h, mean_window=mwo)
            mso = _time_events(fno, torch, dev, iters=6)
            row["natural_order"] = {k: row[k] for k in ("ms", "evals_per_s", "kernel", "alu_frac", "hbm_frac")}
            row.update({"ms": mso, "evals_per_s": cfg["T"] * cfg["S"] / (mso / 1e3), "kernel": spdp.last_kernel(),
                        "alu_frac": cand / (mso / 1e3) / alu_peak,
                        "hbm_frac": bytes_ / (mso / 1e3) / (pk["hbm_gbs"] * 1e9),
                        "scenario_order": "by total demand (spdp_order_scenarios, %.3f ms once per scenario set; "
                                          "alu_frac_incl_order adds it to this one batch of %d tours)" % (order_ms, cfg["T"]),
                        "order_ms": order_ms, "alu_frac_incl_order": cand / ((mso + order_ms) / 1e3) / alu_peak,
                        "partials_equal_natural_order": bool(torch.equal(partO, part))})
            del dO, perm
        rows["a8_batch_%s" % name if cfg["T"] > 1 else "a5_%s" % name] = row
        del d
    # f3: the C3 population evaluated from tour 0's prefix / suffix values (spdp_split_values once,
    # then spdp_split_eval_neighbours over the 256 candidates): same costs as a8, fewer layers
    cfg = synth.config_instance("C3")
    inst = cfg["inst"]
    d = spdp.gen_demands(cfg["model"], 0, cfg["S"], device=dev)
    d, _ = spdp.order_scenarios(d, S=cfg["S"])  # (the scenario set's layout, as in the a8 row: every leg below on it)
    mw3 = bench_config.MEAN_ORDERED["C3"]
    tours = torch.from_numpy(np.ascontiguousarray(cfg["tours"])).to(dev)
    parent = tours[0].contiguous()
    dist = torch.from_numpy(inst["dist"]).to(dev)
    part = torch.zeros((cfg["T"], 6), dtype=torch.int64, device=dev)
    fwd = torch.empty((cfg["n"] + 1, cfg["S"]), dtype=torch.int32, device=dev)
    bwd = torch.empty_like(fwd)
    h = bench_config.HINT["C3"]
    ms_v = _time_events(lambda: spdp.split_values(parent, dist, d, inst["Q"], S=cfg["S"], fwd=fwd, bwd=bwd),
                        torch, dev, iters=6)
    ms_n = _time_events(lambda: spdp.split_eval_neighbours(parent, fwd, bwd, tours, dist, d, inst["Q"], S=cfg["S"],
                                                           want_cost=False, partial=part, window_hint=h),
                        torch, dev, iters=6)
    _, bpart = spdp.split_eval_batch(tours, dist, d, inst["Q"], S=cfg["S"], want_cost=False, window_hint=h)
    equal_c3 = bool(torch.equal(part, bpart))
    def span(tt):
        return float(np.mean([0 if (tt[k] == tt[0]).all() else
                              int(np.nonzero(tt[k] != tt[0])[0][-1] - np.nonzero(tt[k] != tt[0])[0][0] + 1)
                              for k in range(len(tt))]))
    # the same 256 x 10^5 evaluation for a granular population (one move of radius <= 10 per candidate)
    lt = synth.local_move_tours(inst["tour"], cfg["T"], 400)
    ltours = torch.from_numpy(lt).to(dev)
    ms_nl = _time_events(lambda: spdp.split_eval_neighbours(parent, fwd, bwd, ltours, dist, d, inst["Q"], S=cfg["S"],
                                                            want_cost=False, partial=part, window_hint=h),
                         torch, dev, iters=6)
    kern = spdp.last_kernel()
    ms_bl = _time_events(lambda: spdp.split_eval_batch(ltours, dist, d, inst["Q"], S=cfg["S"], want_cost=False,
                                                       window_hint=h, mean_window=mw3),
                         torch, dev, iters=6)
    _, lpart = spdp.split_eval_batch(ltours, dist, d, inst["Q"], S=cfg["S"], want_cost=False, window_hint=h)
    # SPDP_F_NBR_AUTO (reads the spans back, one sync): the batched sweep for the C3 population
    ms_auto_c3 = _time_events(lambda: spdp.split_eval_neighbours(parent, fwd, bwd, tours, dist, d, inst["Q"],
                                                                 S=cfg["S"], want_cost=False, partial=part,
                                                                 window_hint=h, auto=True,
                                                                 mean_window=mw3), torch, dev, iters=4)
    ms_auto_gr = _time_events(lambda: spdp.split_eval_neighbours(parent, fwd, bwd, ltours, dist, d, inst["Q"],
                                                                 S=cfg["S"], want_cost=False, partial=part,
                                                                 window_hint=h, auto=True,
                                                                 mean_window=mw3), torch, dev, iters=4)
    rows["f3_neighbours_C3"] = {
        "ms": ms_v + ms_n, "values_ms": ms_v, "neighbours_ms": ms_n, "T": cfg["T"], "S": cfg["S"], "n": cfg["n"],
        "evals_per_s": cfg["T"] * cfg["S"] / ((ms_v + ms_n) / 1e3), "mean_changed_span": span(cfg["tours"]),
        "partials_equal_batch": equal_c3, "kernel": kern, "auto_neighbours_ms": ms_auto_c3,
        "scenario_order": "by total demand (as the a8 row; values, neighbours and batch all on it)",
        "granular": {"neighbours_ms": ms_nl, "ms": ms_v + ms_nl, "batch_ms": ms_bl, "mean_changed_span": span(lt),
                     "evals_per_s": cfg["T"] * cfg["S"] / ((ms_v + ms_nl) / 1e3), "auto_neighbours_ms": ms_auto_gr,
                     "partials_equal_batch": bool(torch.equal(part, lpart))}}
    del d, fwd, bwd
    # f4: C2 with a route-duration limit (1.5 x the largest out-and-back trip) and a fleet limit
    # (capacity bound ceil(sum mu / Q) + 2 routes), each alone and together
    cfg2 = synth.config_instance("C2")
    inst2 = cfg2["inst"]
    d = spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev)
    tour2, dist2 = torch.from_numpy(inst2["tour"]).to(dev), torch.from_numpy(inst2["dist"]).to(dev)
    trip = int(max(inst2["dist"][0, c] + inst2["dist"][c, 0] for c in inst2["tour"]))
    kmin = int(np.ceil(inst2["nominal"].astype(np.int64).sum() / inst2["Q"]))
    costl = torch.empty(cfg2["S"], dtype=torch.int32, device=dev)
    partl = torch.zeros(6, dtype=torch.int64, device=dev)
    f4 = {"Lmax": int(trip * 1.5), "K": kmin + 2}
    for tag, L, K in (("duration", int(trip * 1.5), 0), ("fleet", -1, kmin + 2), ("both", int(trip * 1.5), kmin + 2)):
        fn = lambda: spdp.split_eval_limits(tour2, dist2, d, inst2["Q"], max_duration=L, max_routes=K, S=cfg2["S"],
                                            cost=costl, partial=partl)
        ms = _time_events(fn, torch, dev, iters=3, warm=1)
        f4[tag] = {"ms": ms, "evals_per_s": cfg2["S"] / (ms / 1e3),
                   "infeasible": int(partl[1].item()), "kernel": spdp.last_kernel()}
    # the same on the scenario set ordered by total demand (the headline's layout): similar vehicle
    # counts and windows share a warp
    dO, _ = spdp.order_scenarios(d, S=cfg2["S"])
    for tag, L, K in (("duration", int(trip * 1.5), 0), ("fleet", -1, kmin + 2), ("both", int(trip * 1.5), kmin + 2)):
        fn = lambda: spdp.split_eval_limits(tour2, dist2, dO, inst2["Q"], max_duration=L, max_routes=K, S=cfg2["S"],
                                            cost=costl, partial=partl)
        f4[tag]["ordered_ms"] = _time_events(fn, torch, dev, iters=3, warm=1)
    rows["f4_limits_C2"] = f4
    del d, dO
    # a5 fp32 mode at C2: real-valued (unrounded Euclidean, fp64) costs, float32 DP (DESIGN R25)
    cfg2 = synth.config_instance("C2")
    inst2 = cfg2["inst"]
    d = spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev)
    d, _ = spdp.order_scenarios(d, S=cfg2["S"])  # (the headline's layout of the resident set)
    xy = np.asarray(inst2["coords"], dtype=np.float64)
    distf = torch.from_numpy(np.ascontiguousarray(np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)))).to(dev)
    tour2 = torch.from_numpy(inst2["tour"]).to(dev)
    costf = torch.empty(cfg2["S"], dtype=torch.float32, device=dev)
    ms = _time_events(lambda: spdp.split_eval_f32(tour2, distf, d, inst2["Q"], S=cfg2["S"], cost=costf), torch, dev,
                      iters=5)
    est = spdp.saa_estimate_f32(costf)
    rows["a5_f32_C2"] = {"ms": ms, "evals_per_s": cfg2["S"] / (ms / 1e3), "kernel": spdp.last_kernel(),
                         "saa_mean": est["mean"], "scenario_order": "by total demand (as the headline)"}
    del d
    # f2: penalized split at C2 (lambda = 10 cost units per unit of overload, Q of C2)
    cfg2 = synth.config_instance("C2")
    inst2 = cfg2["inst"]
    d = spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev)
    tour2, dist2 = torch.from_numpy(inst2["tour"]).to(dev), torch.from_numpy(inst2["dist"]).to(dev)
    costp = torch.empty(cfg2["S"], dtype=torch.int32, device=dev)
    partp = torch.zeros(6, dtype=torch.int64, device=dev)
    fn = lambda: spdp.split_eval_penalized(tour2, dist2, d, inst2["Q"], 10, S=cfg2["S"], cost=costp, partial=partp,
                                           window_hint=bench_config.HINT["C2"])
    ms = _time_events(fn, torch, dev, iters=5)
    kern_f2 = spdp.last_kernel()
    dO, _ = spdp.order_scenarios(d, S=cfg2["S"])
    ms_o = _time_events(lambda: spdp.split_eval_penalized(tour2, dist2, dO, inst2["Q"], 10, S=cfg2["S"], cost=costp,
                                                          partial=partp, window_hint=bench_config.HINT["C2"]),
                        torch, dev, iters=5)
    rows["f2_penalized_C2"] = {"ms": ms, "lambda": 10, "evals_per_s": cfg2["S"] / (ms / 1e3),
                               "kernel": kern_f2, "ordered_ms": ms_o}
    del d, dO
    # f1: route recovery (spdp_split_routes) for 4096 scenarios of C2 (one thread per scenario)
    cfg2 = synth.config_instance("C2")
    inst2 = cfg2["inst"]
    d = spdp.gen_demands(cfg2["model"], 0, cfg2["S"], device=dev)
    tour2, dist2 = torch.from_numpy(inst2["tour"]).to(dev), torch.from_numpy(inst2["dist"]).to(dev)
    K = 4096
    scen = torch.arange(0, cfg2["S"], cfg2["S"] // K, dtype=torch.int64, device=dev)[:K].contiguous()
    fn = lambda: spdp.split_routes(tour2, dist2, d, inst2["Q"], scen, S=cfg2["S"])
    ms = _time_events(fn, torch, dev, iters=5)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    for a_, b_ in ev:
        a_.record()
        b_.record()
    for a_, b_ in ev:  # the route kernel alone (profile events on its stream): the call above is host-bound
        spdp.set_profile_events(a_, b_)
        fn()
    spdp.set_profile_events()
    torch.cuda.synchronize(dev)
    kms_f1 = statistics.median(a_.elapsed_time(b_) for a_, b_ in ev)
    kern_f1 = spdp.last_kernel()
    _, _, _, ml = spdp.split_routes(tour2, dist2, d, inst2["Q"], scen, S=cfg2["S"])
    rows["f1_routes_C2"] = {"ms": ms, "kernel_ms": kms_f1, "kernel": kern_f1, "scenarios": K,
                            "scenarios_per_s": K / (ms / 1e3),
                            "max_route_load_le_Q": bool((ml <= inst2["Q"]).all().item())}
    del d
    # a9/a10: IRP (C5)
    c5 = synth.irp_config()
    irp = c5["irp"]
    d = spdp.gen_demands(c5["model"], 0, c5["S"], device=dev)
    costb = torch.empty(c5["S"], dtype=torch.int64, device=dev)
    fn = lambda: spdp.irp_dp(irp["visit"], irp["cust"], d, irp["H"], irp["M"], S=c5["S"], cost=costb)
    ms = _time_events(fn, torch, dev, iters=3)
    kern_irp = spdp.last_kernel()
    # the same DP with the other layouts (same results): eager-shift lanes, and state-parallel lanes
    # (scenario x customer -> warps, inventory state -> lanes: the "3-D" layout)
    ms_eager = _time_events(lambda: spdp.irp_dp(irp["visit"], irp["cust"], d, irp["H"], irp["M"], S=c5["S"],
                                                cost=costb, eager=True), torch, dev, iters=3)
    ms_states = _time_events(lambda: spdp.irp_dp(irp["visit"], irp["cust"], d, irp["H"], irp["M"], S=c5["S"],
                                                 cost=costb, states=True), torch, dev, iters=3)
    # roofline: the demand stream (H M u16 per scenario) + the int64 cost.  The affine-tail kernel's
    # work per (scenario, customer) is O(I0 + H) (DESIGN §6 IRP), not the eager DP's (U + 1) H state
    # updates (states_per_s: the eager-equivalent rate); it is issue-bound (ncu: IPC 2.7 of 4,
    # profiles/r02_ncu_irp_C5.json), and hbm_frac shows how far the data stream is from limiting it
    bytes_irp = irp["H"] * irp["M"] * c5["S"] * 2 + c5["S"] * 8
    U = int(irp["cust"][0, 0])
    rows["a9_a10_irp_C5"] = {"ms": ms, "scenarios_per_s": c5["S"] / (ms / 1e3), "kernel": kern_irp,
                             "stages_per_s": c5["S"] * irp["M"] * irp["H"] / (ms / 1e3),
                             "states_per_s_eager_equivalent": c5["S"] * irp["M"] * irp["H"] * (U + 1) / (ms / 1e3),
                             "bytes_alg": bytes_irp, "hbm_frac": bytes_irp / (ms / 1e3) / (pk["hbm_gbs"] * 1e9),
                             "eager_lane_ms": ms_eager, "state_parallel_ms": ms_states,
                             # the eager DP's candidates (band [0, y] on visited periods,
                             # the demand step's J = 0 minimum), counted exactly from the model, at one
                             # candidate per ALU lane per clock -- the floor of any eager-DP kernel
                             "eager_candidates": irp_eager_candidates(irp, c5),
                             "eager_alu_floor_ms": irp_eager_candidates(irp, c5) / (N_SM * ALU_LANES_PER_SM_CLK *
                                                                                   pk["sm_max_mhz"] * 1e6) * 1e3,
                             "bound": "issue (ALU): O(I0 + H) integer steps per (scenario, customer) after the "
                                      "affine-tail reformulation; hbm_frac = the demand stream's share"}
    return rows


def irp_eager_candidates(irp, c5):
    """Candidates of the eager IRP DP (SURVEY §8(a9/a10)) over the whole C5 sample, with every state
    reachable (an upper bound of any state-by-state kernel's work): per (scenario, customer, period),
    a visited period's band step sum_{y=0..U} (min(y, X) + 1), and the J = 0 step's min(d, U) + 1 --
    taken at the nominal demand (mu_m) per customer and period (a count of work, not a cost)."""
    U = int(irp["cust"][0, 0])
    X = int(irp["cust"][0, 1])
    band = sum(min(y, X) + 1 for y in range(U + 1))
    per_sm = 0
    for m in range(irp["M"]):
        for t in range(irp["H"]):
            per_sm += (band if irp["visit"][m, t] else 0) + min(int(irp["mu"][m]), U) + 1
    return per_sm * c5["S"]


def cpu_baseline(cfg, cost_dev, S, spdp, partial_dev, perm_dev=None):
    import oracle
    inst = cfg["inst"]
    threads = max(oracle.num_threads(), os.cpu_count() or 1)  # all host cores (torchrun sets OMP_NUM_THREADS=1)
    dem = oracle.gen_demands(cfg["model"], 0, S, threads=threads)
    t0 = time.perf_counter()
    want = oracle.split(inst["tour"], inst["dist"], dem, inst["Q"], threads=threads)
    w = oracle.saa(want)
    t = time.perf_counter() - t0
    got = cost_dev.cpu().numpy().astype(np.int64)
    if perm_dev is not None:  # (an ordered scenario set: column j holds scenario perm[j])
        want_cols = np.asarray(want)[perm_dev.cpu().numpy()]
    else:
        want_cols = np.asarray(want)
    parity = bool(np.array_equal(got, want_cols))
    est = spdp.saa_mean(partial_dev)
    # the paper's 1-thread baseline: one host thread on a 10^5-scenario prefix
    S1 = min(S, 100_000)
    t0 = time.perf_counter()
    oracle.split(inst["tour"], inst["dist"], dem, inst["Q"], S=S1, threads=1)
    t1 = time.perf_counter() - t0
    cpu_model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            cpu_model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), "")
    except OSError:
        pass
    return {"value": S / t, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": "all %d scenarios of the timed workload, once (oracle split + SAA; demands pre-generated "
                      "by the oracle's own generator)" % S,
            "seconds": t, "parity_all_costs_bit_exact": parity, "saa_mean_equal": est["mean"] == w["mean"],
            "cpu_model": cpu_model,
            "single_thread": {"value": S1 / t1, "unit": UNIT, "cores": 1,
                              "sample": "first %d scenarios, oracle split only" % S1}}


if __name__ == "__main__":
    sys.exit(main())
