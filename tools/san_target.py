"""Small launches of every kernel of libvtrace.so, for compute-sanitizer (dev tool):
the column-block kernel (nts = 1 and nts > 1, loss and from_logits, fp32 and bf16,
programmatic dependent chain), the look-back kernel (TMA and plain loads), the
learner update (single and multi-gradient) and the tcgen05 output layer.  Each call
is checked against the previous identical call (bitwise) so a race that changes the
results also fails here.  usage: python tools/san_target.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_01561_b200 as pkg  # noqa: E402
from paper_1802_01561_b200 import vtrace as vt  # noqa: E402
from paper_1802_01561_b200 import workload as wl  # noqa: E402


def run(inp, kernel=0, pdl=False, reps=2):
    d = pkg.tensors_from_workload(inp, "cuda")
    args = [d[k] for k in vt.INPUT_NAMES]
    ws = pkg.Workspace(inp["T"], inp["B"], inp["A"], inp["dtype"])
    outs = []
    for _ in range(reps):
        o = pkg.loss_and_grad(*args, workspace=ws, reward_mode=inp["reward_mode"], kernel=kernel,
                              overlap_previous=pdl)
        f = pkg.from_logits(*args, workspace=ws, reward_mode=inp["reward_mode"], kernel=kernel,
                            overlap_previous=pdl)
        torch.cuda.synchronize()
        outs.append({**{k: v.clone() for k, v in o.items()}, **{"f_" + k: v.clone() for k, v in f.items()}})
    for k in outs[0]:
        assert torch.equal(outs[0][k], outs[1][k]), ("non-deterministic", k)
    assert pkg.read_device_status(ws) == (0, -1)
    print("ok", inp["T"], inp["B"], inp["A"], kernel, pdl, flush=True)


run(wl.make_inputs("large", T=20, B=8192))                         # cb, nts = 1, 147 CTAs
run(wl.make_inputs("large", T=20, B=8192), pdl=True)               # cb, programmatic dependent
run(wl.make_inputs("large", T=37, B=1024))                         # cb, nts > 1 (carry exchange)
run(wl.make_inputs("stress", T=70, B=64))                          # cb, fp32, A = 9
run(wl.make_inputs("dmlab", T=30, B=32))                           # cb, bf16 A = 9 (8-col segments)
run(wl.make_inputs("dmlab", T=30, B=32), kernel=vt.KERNEL_LOOKBACK)  # look-back, TMA
run(wl.toy_inputs())                                               # look-back, plain loads
run(wl.make_inputs("atari", T=45, B=24, A=24))                     # look-back, runtime A

u = wl.update_inputs(70_001, seed=3, learners=2)
th = torch.from_numpy(u["params"]).cuda()
ms = torch.from_numpy(u["mean_square"]).cuda()
gs = [torch.from_numpy(g).cuda() for g in u["grads"]]
pkg.rmsprop_step(th, ms, gs[0], 6e-4, 0.99, 0.01, 40.0)
pkg.rmsprop_step(th, ms, gs, 6e-4, 0.99, 0.01, 40.0)
torch.cuda.synchronize()
print("ok rmsprop", flush=True)

h = torch.randn(1000, 256, device="cuda").to(torch.bfloat16)
w = torch.randn(19, 256, device="cuda").to(torch.bfloat16)
b = torch.randn(19, device="cuda")
z, v = pkg.output_layer(h, w, b)
torch.cuda.synchronize()
print("ok output_layer", float(z.sum()), flush=True)
