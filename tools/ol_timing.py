"""Times vtrace_output_layer (NEXT #3) through the Python binding at the `large` config
(M = T*B = 819,200, H = 256, A = 18): CUDA events on the launching stream, 50 launches after
5 warm-ups; h (419 MB) exceeds L2, so no flush is needed.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1802_01561_b200 as pkg

M, H, A = 100 * 8192, 256, int(os.environ.get("OL_A", 18))
g = torch.Generator(device="cuda:0").manual_seed(0)
if os.environ.get("OL_DATA") == "dyadic":  # A/B: value pattern of the h stream
    h = (torch.randint(-48, 49, (M, H), generator=g, device="cuda:0") / 64.0).to(torch.bfloat16)
else:
    h = torch.randn((M, H), generator=g, device="cuda:0").to(torch.bfloat16)
w = (torch.randn((A + 1, H), generator=g, device="cuda:0") * 0.1).to(torch.bfloat16)
b = None if os.environ.get("OL_NOBIAS") else torch.randn(A + 1, generator=g, device="cuda:0")
z = torch.empty((M, A), device="cuda:0")
v = torch.empty(M, device="cuda:0")
for _ in range(5):
    pkg.output_layer(h, w, b, z, v)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
n = 50
e0.record(s)
for _ in range(n):
    pkg.output_layer(h, w, b, z, v)
e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / n
nbytes = M * H * 2 + (A + 1) * H * 2 + M * (A + 1) * 4 + (A + 1) * 4
print(json.dumps({"kernel": "vtrace_output_layer", "data": os.environ.get("OL_DATA", "normal"), "bias": b is not None, "defines": os.environ.get("VTRACE_DEFINES", ""), "M": M, "H": H, "A": A, "us": round(us, 2),
                  "algorithmic_bytes": nbytes, "GBps": round(nbytes / us / 1e3, 1),
                  "frac_of_measured_hbm": round(nbytes / us / 1e3 / 6544.7, 3)}))
