"""Eager calls of vtrace_loss_and_grad on one config, for ncu captures (dev tool).
usage: python tools/ncu_target.py [config[:B=..,T=..]] [calls] [kernel]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_01561_b200 as pkg  # noqa: E402
from paper_1802_01561_b200 import workload as wl  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "large"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kernel = int(sys.argv[3]) if len(sys.argv) > 3 else 0
name, _, kv = spec.partition(":")
kw = {k: int(v) for k, v in (x.split("=") for x in kv.split(",") if x)}
inp = wl.make_inputs(name, **kw)
d = pkg.tensors_from_workload(inp, "cuda")
ws = pkg.Workspace(inp["T"], inp["B"], inp["A"], inp["dtype"])
args = [d[k] for k in pkg.vtrace.INPUT_NAMES]
out = pkg.loss_and_grad(*args, workspace=ws, reward_mode=inp["reward_mode"], kernel=kernel)
for _ in range(calls - 1):
    pkg.loss_and_grad(*args, workspace=ws, reward_mode=inp["reward_mode"], out=out, kernel=kernel)
torch.cuda.synchronize()
print("ok", pkg.kernel_for(inp["T"], inp["B"], inp["A"], inp["dtype"]), out["partials"].tolist())
