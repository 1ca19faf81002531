"""NEXT #4 at N > 1, timing build (RMS_TIMING): per-call stamps of the learners' update
(CTA 0: start, ready published, peers ready seen, norm known, updates stored; last CTA:
done published, peers done seen) in an eager loop and in CUDA-graph replay.  Dev tool;
run under torchrun (one rank per GPU).  usage: python tools/rms_stamps.py [sharded]"""
import ctypes
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_01561_b200 as pkg  # noqa: E402
from paper_1802_01561_b200 import workload as wl  # noqa: E402


def main():
    sharded = len(sys.argv) > 1 and sys.argv[1] == "sharded"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # rotated state copies (as bench.py)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    import torch.distributed._symmetric_memory as symm_mem
    n = wl.UPDATE_SIZES["deep"]
    inp = wl.update_inputs(n, seed=1 + rank, norm=60.0)
    gs = [torch.from_numpy(inp["grads"][0]).cuda() for _ in range(R)]
    red = symm_mem.empty(n, dtype=torch.float32, device="cuda")
    ptrs = [int(p) for p in symm_mem.rendezvous(red, dist.group.WORLD.group_name).buffer_ptrs]
    flg = symm_mem.empty(2, dtype=torch.int32, device="cuda")
    flg.zero_()
    fptrs = [int(p) for p in symm_mem.rendezvous(flg, dist.group.WORLD.group_name).buffer_ptrs]
    th = symm_mem.empty(n, dtype=torch.float32, device="cuda")
    th.copy_(torch.from_numpy(inp["params"]))
    tptrs = [int(p) for p in symm_mem.rendezvous(th, dist.group.WORLD.group_name).buffer_ptrs]
    nmb = symm_mem.empty(pkg.vtrace.rmsprop_norm_mailbox_bytes(world) // 8, dtype=torch.float64,
                         device="cuda")
    nmb.zero_()
    nptrs = [int(p) for p in symm_mem.rendezvous(nmb, dist.group.WORLD.group_name).buffer_ptrs]
    mss = [torch.from_numpy(inp["mean_square"]).cuda() for _ in range(R)]
    ths = [th] + [torch.from_numpy(inp["params"]).cuda() for _ in range(R - 1)]
    ws = pkg.RmspropWorkspace(n)
    it = [0]
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.Stream()

    def step():
        j = it[0] % R
        it[0] += 1
        torch.mul(gs[j], 1.0, out=red)
        if sharded:
            pkg.vtrace.rmsprop_step_sharded(tptrs, mss[j], ptrs, 6e-4, 0.99, 0.01, 40.0,
                                            flags=fptrs, norm_mailboxes=nptrs, self_index=rank,
                                            n=n, workspace=ws)
        else:
            pkg.rmsprop_step(ths[j], mss[j], ptrs, 6e-4, 0.99, 0.01, 40.0, workspace=ws,
                             learner_flags=fptrs, self_index=rank)

    with torch.cuda.stream(s):
        for _ in range(300):
            step()
    torch.cuda.synchronize()
    dist.barrier()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(30):
            step()
    torch.cuda.synchronize()
    dist.barrier()
    import time
    host_us = []
    t_all = time.perf_counter()
    with torch.cuda.stream(s):
        for _ in range(8):
            t0 = time.perf_counter()
            gr.replay()
            host_us.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    wall_us = (time.perf_counter() - t_all) * 1e6
    lib = pkg.load_library()
    buf = (ctypes.c_ulonglong * (8 * 4096))()
    lib.vtrace_debug_rms_stamps.argtypes = [ctypes.c_void_p]
    lib.vtrace_debug_rms_stamps(ctypes.addressof(buf))
    st = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)

    def summary(lo, hi):
        a = st[lo:hi]
        d = lambda i, j: np.median(a[:, j] - a[:, i]) / 1e3  # noqa: E731
        per = np.median(np.diff(a[:, 0])) / 1e3
        gap = np.median(a[1:, 0] - a[:-1, 6]) / 1e3
        per_mean = float(np.mean(np.diff(a[:, 0]))) / 1e3
        per_max = float(np.max(np.diff(a[:, 0]))) / 1e3
        return {"period_us": round(per, 2), "period_mean_us": round(per_mean, 2),
                "period_max_us": round(per_max, 2), "ready_pub": round(d(0, 1), 2),
                "wait_peers_ready": round(d(1, 2), 2), "reads_norm": round(d(2, 3), 2),
                "update": round(d(3, 4), 2), "to_done_pub": round(d(4, 5), 2),
                "wait_peers_done": round(d(5, 6), 2), "gap_to_next_start": round(gap, 2)}
    # eager calls: epochs 3 (after the setup call) .. 300; graph: the replays' calls
    out = {"rank": rank, "sharded": sharded, "R": R, "eager": summary(100, 300),
           "graph_capture_epochs": "replays of 30 steps x 8",
           "graph": summary(330, 539), "graph_replay_host_us": [round(x) for x in host_us],
           "graph_wall_us_per_step": round(wall_us / 240, 2)}
    print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
