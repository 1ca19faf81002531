"""Timing of vtrace_head_loss_and_grad (dev tool): CUDA events around N eager calls
alternating two input sets, median of 5 repeats.  usage: python tools/hf_time.py [T B H A]..."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_01561_b200 as pkg  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]


def run(T, B, H, A, n=40):
    g = torch.Generator(device="cuda").manual_seed(1)
    w = (torch.randn((A + 1, H), generator=g, device="cuda") * 0.1).to(torch.bfloat16)
    bias = torch.randn(A + 1, generator=g, device="cuda") * 0.1
    sets = []
    for _ in range(2):
        h = torch.randn((T, B, H), generator=g, device="cuda").to(torch.bfloat16)
        mu = torch.randn((T, B, A), generator=g, device="cuda")
        act = torch.randint(0, A, (T, B), generator=g, device="cuda", dtype=torch.int32)
        disc = torch.full((T, B), 0.99, device="cuda")
        rew = torch.randn((T, B), generator=g, device="cuda")
        boot = torch.randn(B, generator=g, device="cuda")
        sets.append((h, mu, act, disc, rew, boot))
    ws = pkg.HeadWorkspace(T, B, H, A)
    out = pkg.head_loss_and_grad(*sets[0][:1], w, bias, *sets[0][1:], workspace=ws)
    res = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for i in range(n):
            s = sets[i % 2]
            pkg.head_loss_and_grad(s[0], w, bias, *s[1:], workspace=ws, out=out)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1e3 / n)
    res.sort()
    M = T * B
    alg = 2 * M * H * 2 + M * A * 4 + 3 * M * 4 + B * 4 + (A + 1) * H * 6 + (A + 1) * 8 + 64
    us = res[2]
    print(json.dumps({"T": T, "B": B, "H": H, "A": A, "us_per_call": round(us, 2),
                      "all": [round(x, 2) for x in res], "GBps": round(alg / us / 1e3, 1),
                      "frac": round(alg / us / 1e3 / PEAK, 4)}), flush=True)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]] or [100, 8192, 256, 18]
    for k in range(0, len(a), 4):
        run(*a[k:k + 4])
