"""Per-CTA timeline of one column-block launch (timing build: VTRACE_DEFINES=CB_TIMING).
usage: python tools/cb_stamps.py [config[:B=..,T=..]] [--pdl]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_01561_b200 as pkg  # noqa: E402
from paper_1802_01561_b200 import workload as wl  # noqa: E402

spec = next((a for a in sys.argv[1:] if not a.startswith("--")), "large")
pdl = "--pdl" in sys.argv
name, _, kv = spec.partition(":")
kw = {k: int(v) for k, v in (x.split("=") for x in kv.split(",") if x)}
inp = wl.make_inputs(name, **kw)
sets = [pkg.tensors_from_workload(inp, "cuda") for _ in range(3)]
ws = pkg.Workspace(inp["T"], inp["B"], inp["A"], inp["dtype"])
lib = pkg.load_library()
lib.vtrace_debug_cb_stamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
outs = [pkg.loss_and_grad(*[d[k] for k in pkg.vtrace.INPUT_NAMES], workspace=ws,
                          reward_mode=inp["reward_mode"]) for d in sets]
for rep in range(3):
    for i in range(6):
        d = sets[i % 3]
        pkg.loss_and_grad(*[d[k] for k in pkg.vtrace.INPUT_NAMES], workspace=ws, out=outs[i % 3],
                          reward_mode=inp["reward_mode"], overlap_previous=pdl)
    torch.cuda.synchronize()
n = 4096
buf = (ctypes.c_ulonglong * (8 * n))()
assert lib.vtrace_debug_cb_stamps(buf, n) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
grid = int((a[:, 0] > 0).sum())
a = a[:grid]
t0 = a[:, 0].min()
r = (a - t0) / 1000.0
last = r[:, 4].max()
print(f"{spec} pdl={pdl} grid={grid}")
for k, nm in enumerate(["start", "first data", "last stage released", "published"]):
    print(f"  {nm:22s} min {r[:, k].min():7.2f}  median {np.median(r[:, k]):7.2f}  max {r[:, k].max():7.2f} us")
li = int(np.argmax(r[:, 4]))
print(f"  last CTA {li}: published {r[li, 3]:.2f}, all warps in {r[li, 5]:.2f}, warp 0 records "
      f"summed {r[li, 6]:.2f}, all warps summed {r[li, 7]:.2f}, done {r[li, 4]:.2f} us")
