"""Per-task globaltimer stamps of the column-task kernel (dev tool, debug hook
vtrace_debug_set_timing): [start, own end (after the group ticket), group
reduced (last arrivals), total written], relative to the first start.  usage: python tools/ct_timing.py [config]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_01561_b200 as pkg  # noqa: E402
from paper_1802_01561_b200 import workload as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
inp = wl.make_inputs(name)
dev = pkg.tensors_from_workload(inp, "cuda")
args = [dev[k] for k in pkg.vtrace.INPUT_NAMES]
ws = pkg.Workspace(inp["T"], inp["B"], inp["A"], inp["dtype"])
for _ in range(5):
    pkg.loss_and_grad(*args, workspace=ws, reward_mode=inp["reward_mode"])
torch.cuda.synchronize()
tasks = inp["B"] // 4
buf = torch.zeros(tasks * 4, dtype=torch.int64, device="cuda")
lib = pkg.load_library()
lib.vtrace_debug_set_timing.argtypes = [ctypes.c_void_p, ctypes.c_int32]
lib.vtrace_debug_set_timing(ctypes.c_void_p(buf.data_ptr()), 1)
pkg.loss_and_grad(*args, workspace=ws, reward_mode=inp["reward_mode"])
torch.cuda.synchronize()
lib.vtrace_debug_set_timing(None, 0)
t = buf.view(tasks, 4).cpu().numpy().astype(np.int64)
t0 = t[:, 0].min()
r = np.where(t > 0, t - t0, -1) / 1000.0  # us
st, en = r[:, 0], r[:, 1]
print(f"start: min {st.min():.2f} max {st.max():.2f} us; own end: min {en.min():.2f} "
      f"median {np.median(en):.2f} max {en.max():.2f}")
print("slowest tasks (own end):", [(int(i), round(float(en[i]), 2), round(float(st[i]), 2))
                                   for i in np.argsort(-en)[:8]])
gr = r[:, 2]
gi = np.where(gr >= 0)[0]
print("group reducers done: ", "n", len(gi), "min", gr[gi].min() if len(gi) else None,
      "max", gr[gi].max() if len(gi) else None)
print("  worst groups:", [(int(i), round(float(gr[i]), 2), round(float(en[i]), 2),
                           round(float(en[(i // 32) * 32:(i // 32) * 32 + 32].max()), 2))
                          for i in gi[np.argsort(-gr[gi])][:6]])
print("top done:", r[:, 3].max())
hist = np.histogram(en, bins=12)
print("own-end histogram:", list(zip(np.round(hist[1], 1).tolist(), hist[0].tolist())))
