"""Kernel-only timing of vtrace_loss_and_grad (dev tool): CUDA-graph loop of N calls
over R rotated input sets (R x working set > 4 x L2 where it fits), CUDA events,
median of 5 repeats.  Prints µs per call and the fraction of the measured HBM peak
(SURVEY 8(d) algorithmic bytes: 3 A s + 20 per step, + 4 B + 64).

usage: python tools/kernel_time.py [config[:B=..,T=..]] ... [--kernel 1|2] [--pdl]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_01561_b200 as pkg  # noqa: E402
from paper_1802_01561_b200 import workload as wl  # noqa: E402

if os.environ.get("KT_LIB"):  # A/B variant library (tools/ab_build.py)
    pkg.vtrace.load_library(os.environ["KT_LIB"])

PEAK = 6552.3
try:
    PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    pass


def time_config(spec, kernel=0, pdl=False, n=200):
    name, _, kv = spec.partition(":")
    kw = {k: int(v) for k, v in (x.split("=") for x in kv.split(",") if x)}
    inp = wl.make_inputs(name, **kw)
    T, B, A = inp["T"], inp["B"], inp["A"]
    s = 2 if inp["dtype"] == wl.DTYPE_BF16 else 4
    algo = T * B * (3 * A * s + 20) + 4 * B + 64
    ws_bytes = T * B * (3 * A * s + 20)
    R = max(1, min(8, (4 * 126 * 2**20) // ws_bytes + 1))
    base = pkg.tensors_from_workload(inp, "cuda")
    sets = [{k: v.clone() for k, v in base.items()} for _ in range(R)]
    outs = [{"grad_target_logits": torch.empty_like(base["target_logits"]),
             "grad_values": torch.empty(T, B, device="cuda"),
             "partials": torch.empty(8, dtype=torch.float64, device="cuda")} for _ in range(R)]
    wsp = pkg.Workspace(T, B, A, inp["dtype"])
    rm = inp["reward_mode"]

    def call(i):
        d = sets[i % R]
        pkg.loss_and_grad(*[d[k] for k in pkg.vtrace.INPUT_NAMES], reward_mode=rm, workspace=wsp,
                          out=outs[i % R], kernel=kernel, overlap_previous=pdl)

    for i in range(10):
        call(i)
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(n):
                call(i)
    torch.cuda.current_stream().wait_stream(st)
    res = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1e3 / n)
    res.sort()
    us = res[2]
    gbs = algo / us / 1e3
    print(json.dumps({"config": spec, "kernel": pkg.kernel_for(T, B, A, inp["dtype"]),
                      "forced": kernel, "pdl": pdl, "us_per_call": round(us, 3),
                      "all": [round(x, 2) for x in res], "GBps": round(gbs, 1),
                      "frac": round(gbs / PEAK, 4), "rotated_sets": R}), flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    kernel = 0
    if "--kernel" in sys.argv:
        kernel = int(sys.argv[sys.argv.index("--kernel") + 1])
        args = [a for a in args if a != str(kernel)]
    pdl = "--pdl" in sys.argv
    for spec in args or ["large"]:
        time_config(spec, kernel=kernel, pdl=pdl)
