"""Small repro: one fused call on a named config (for compute-sanitizer runs)."""
import sys
import torch
import paper_1802_01561_b200 as pkg
from paper_1802_01561_b200 import workload as wl

name = sys.argv[1] if len(sys.argv) > 1 else "dmlab"
which = sys.argv[2] if len(sys.argv) > 2 else "loss"
inp = wl.make_inputs(name, B=int(sys.argv[3]) if len(sys.argv) > 3 else None)
dev = pkg.tensors_from_workload(inp, "cuda")
args = [dev[k] for k in pkg.vtrace.INPUT_NAMES]
if which == "loss":
    out = pkg.loss_and_grad(*args, reward_mode=inp["reward_mode"])
else:
    out = pkg.from_logits(*args, reward_mode=inp["reward_mode"])
torch.cuda.synchronize()
print("ok", name, which, {k: float(v.float().abs().sum()) for k, v in out.items()})
