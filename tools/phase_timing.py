"""Per-phase cycle timing of the fused kernel (dev tool, uses the debug hook
vtrace_debug_set_timing).  usage: python tools/phase_timing.py [config] [B]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_01561_b200 as pkg  # noqa: E402
from paper_1802_01561_b200 import workload as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
inp = wl.make_inputs(name, B=int(sys.argv[2]) if len(sys.argv) > 2 else None)
dev = pkg.tensors_from_workload(inp, "cuda")
args = [dev[k] for k in pkg.vtrace.INPUT_NAMES]
ws = pkg.Workspace(inp["T"], inp["B"], inp["A"], inp["dtype"])
for _ in range(3):
    pkg.loss_and_grad(*args, workspace=ws, reward_mode=inp["reward_mode"])
torch.cuda.synchronize()
ITERS = 64
GRID = 148 * 8
buf = torch.zeros(GRID * ITERS * 8, dtype=torch.int64, device="cuda")
lib = pkg.load_library()
lib.vtrace_debug_set_timing.argtypes = [ctypes.c_void_p, ctypes.c_int32]
lib.vtrace_debug_set_timing(ctypes.c_void_p(buf.data_ptr()), ITERS)
pkg.loss_and_grad(*args, workspace=ws, reward_mode=inp["reward_mode"])
torch.cuda.synchronize()
lib.vtrace_debug_set_timing(None, 0)
t = buf.view(GRID, ITERS, 8).cpu().numpy().astype(np.int64)
used = t[:, :ITERS - 1, 0] != 0
rows = []
for c in range(GRID):
    for i in range(ITERS - 1):
        if not used[c, i]:
            continue
        r = t[c, i]
        rows.append(dict(p1=r[1] - r[0], scan=r[5] - r[4], scan_local=r[7] - r[4],
                         scan_rest=r[5] - r[7], p3_rows=r[6] - r[2], p3_tail=r[3] - r[6],
                         wait_row=r[2] - r[1],
                         wait_scan=r[2] - r[5], p3=r[3] - r[2],
                         iter=(t[c, i + 1, 0] - r[0]) if i + 1 < ITERS - 1 and used[c, i + 1] else 0))
g = t[:, ITERS - 1, :4]
ok = g[:, 0] > 0
if ok.any():
    g0 = g[ok, 0].min()
    print("globaltimer (ns from first CTA start): start med %.0f max %.0f | first data med %.0f max %.0f | loop end med %.0f max %.0f | last CTA done %.0f" % (
        np.median(g[ok, 0] - g0), (g[ok, 0] - g0).max(), np.median(g[ok, 3] - g0), (g[ok, 3] - g0).max(),
        np.median(g[ok, 1] - g0), (g[ok, 1] - g0).max(), (g[ok, 2].max() - g0) if (g[ok, 2] > 0).any() else -1))
keys = ["p1", "scan", "scan_local", "scan_rest", "wait_row", "p3", "p3_rows", "p3_tail", "iter"]
print(name, "CTAs used", int(used[:, 0].sum()), "iterations/CTA", int(used.sum(1).max()))
for k in keys:
    v = np.array([r[k] for r in rows if r[k] > 0])
    if v.size:
        print(f"{k:10s} median {np.median(v):8.0f}  p10 {np.percentile(v, 10):8.0f}  p90 {np.percentile(v, 90):8.0f} cycles  (n={v.size})")
