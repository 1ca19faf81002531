#!/usr/bin/env python
"""Summarise an ncu report (full set) of the fused kernel into profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <out-name> [--config large]
Writes profiles/<out-name>.json (selected raw metrics, stall breakdown, top
SASS opcodes) and, with --config, records the per-launch DRAM traffic in
profiles/ncu_traffic.json for bench.py's roofline.traffic field.
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
    "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__inst_executed_pipe_fp64.sum", "smsp__inst_executed_pipe_xu.sum",
    "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_alu.sum",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("name")
    ap.add_argument("--config", default=None)
    a = ap.parse_args()
    raw = ncu("-i", a.report, "--page", "raw", "--csv")
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    metrics = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            metrics[m] = {"value": vals[i], "unit": units[i]}
    src = ncu("-i", a.report, "--page", "source", "--csv", "--print-source", "sass")
    srows = list(csv.reader(io.StringIO(src)))
    shdr = srows[1]
    data = srows[2:]
    ix = {h: j for j, h in enumerate(shdr)}

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    ops, stalls = Counter(), Counter()
    for r in data:
        toks = r[ix["Source"]].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        ops[op.split(".")[0]] += f(r[ix["Instructions Executed"]])
        for h in shdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                stalls[h[6:]] += f(r[ix[h]])
    tot_ops = sum(ops.values()) or 1.0
    tot_st = sum(stalls.values()) or 1.0
    out = {
        "report": os.path.basename(a.report),
        "kernel": rows[2][hdr.index("Kernel Name")] if "Kernel Name" in hdr else None,
        "metrics": metrics,
        "stall_pct": {k: round(v / tot_st * 100, 1) for k, v in stalls.most_common(12)},
        "top_opcodes_pct": {k: round(v / tot_ops * 100, 2) for k, v in ops.most_common(20)},
        "warp_instructions": tot_ops,
    }
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", a.name + ".json"), "w") as fh:
        json.dump(out, fh, indent=1)
    if a.config:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = {}
        if os.path.exists(path):
            d = json.load(open(path))
        rd = float(metrics["dram__bytes_read.sum"]["value"].replace(",", ""))
        wr = float(metrics["dram__bytes_write.sum"]["value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(metrics["dram__bytes_read.sum"]["unit"], 1)
        wr *= scale.get(metrics["dram__bytes_write.sum"]["unit"], 1)
        d[a.config] = rd + wr
        d[a.config + "_source"] = a.name
        json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
