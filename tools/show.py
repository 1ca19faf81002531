"""Summarise gpurun_out results for a tag: test tails, bench lines, parity margins."""
import glob
import json
import sys

tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{tag}_gpu*.txt")):
    lines = open(f).read().strip().splitlines()
    print(f, "|", " ".join(lines[-2:]))
for f in sorted(glob.glob(f"gpurun_out/{tag}_bench*.txt")):
    ok = False
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            ok = True
            r = d.get("roofline") or {}
            print(f"{f:44s} {d['config']['workload']:7s} ms {d['ms_per_step']:.4f} frac {r.get('frac', 0):.3f} "
                  f"GB/s {r.get('achieved', 0):.0f} e2e {(d.get('e2e') or {}).get('ms_per_step')}")
    if not ok:
        print(f, open(f).read()[-300:])
for f in sorted(glob.glob(f"gpurun_out/{tag}_margin*.jsonl")):
    worst = {}
    for l in open(f):
        d = json.loads(l)
        k = d["output"]
        if d["max_err_over_tol"] > worst.get(k, (0, ""))[0]:
            worst[k] = (d["max_err_over_tol"], d["test"])
    print(f, " ".join(f"{k}={v[0]:.3f}" for k, v in sorted(worst.items())))
