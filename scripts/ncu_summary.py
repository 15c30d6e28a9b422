"""Summarise an ncu --set full report into a small JSON (committed under profiles/).

    python scripts/ncu_summary.py <report.ncu-rep> <out.json> [--units N]

--units: algorithmic units per launch (e.g. scenario-layers) to normalise the
instruction mix."""
import csv
import io
import json
import subprocess
import sys
from collections import Counter


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, out = sys.argv[1], sys.argv[2]
    units = None
    if "--units" in sys.argv:
        units = float(sys.argv[sys.argv.index("--units") + 1])
    raw = ncu_csv(rep, "--page", "raw")
    d = dict(zip(raw[0], raw[2]))
    unit = dict(zip(raw[0], raw[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
             "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}

    def f(k):
        try:
            v = float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return None
        return v * scale.get(unit.get(k, ""), 1.0)

    res = {
        "kernel": d.get("Kernel Name", "")[:160],
        "duration_us": f("gpu__time_duration.sum"),
        "dram_bytes_read": f("dram__bytes_read.sum"),
        "dram_bytes_write": f("dram__bytes_write.sum"),
        "sm_clock_hz": f("smsp__cycles_elapsed.avg.per_second"),
        "ipc_per_sm": f("sm__inst_executed.avg.per_cycle_active"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": f("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "warps_active_per_sm": f("sm__warps_active.avg.per_cycle_active"),
        "registers": f("launch__registers_per_thread"),
        "smem_per_block": f("launch__shared_mem_per_block_dynamic"),
        "grid": d.get("launch__grid_size"),
        "block": d.get("launch__block_size"),
        "stalls_per_issue": {},
    }
    for k, v in d.items():
        if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                val = float(v)
            except ValueError:
                continue
            if val >= 0.05:
                res["stalls_per_issue"][k.split("stalled_")[1].split("_per")[0]] = round(val, 3)
    if res["dram_bytes_read"] is not None:
        res["dram_bytes_per_launch"] = (res["dram_bytes_read"] or 0) + (res["dram_bytes_write"] or 0)
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    if len(src) > 2:
        hdr = src[1]
        i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
        c = Counter()
        for r in src[2:]:
            toks = r[i_src].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") else toks[0]
            try:
                c[op.split(".")[0]] += int(r[i_ex])
            except ValueError:
                pass
        tot = sum(c.values())
        res["warp_instructions"] = tot
        if units:
            res["units"] = units
            res["instr_per_unit"] = round(tot / units, 2)
            res["mix_per_unit"] = {k: round(v / units, 2) for k, v in c.most_common(16)}
        else:
            res["mix"] = dict(c.most_common(16))
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps({k: res[k] for k in ("kernel", "duration_us", "dram_bytes_per_launch", "ipc_per_sm",
                                          "alu_pipe_pct", "fma_pipe_pct") if k in res}))


if __name__ == "__main__":
    main()
