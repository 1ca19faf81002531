#!/usr/bin/env python
"""bench.py -- V-trace + loss + grad trajectory-steps/s and HBM GB/s on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` (torchrun for
N > 1, one rank per GPU, NCCL) prints ONE JSON line on rank 0.

A "step" is one learner update's hot path over one batch: the fused
vtrace_loss_and_grad kernel on this rank's [T, B/N, A] trajectories (all SURVEY
8(a) rows a1-a12), plus, for N > 1, the NCCL all-reduce of the 8 fp64 partial
sums (row a13, issued on a side stream so it overlaps the next step's kernel) --
the product's learner.LearnerStep.  Default at N > 1: strong scaling, the
BASELINE config's B = 8192 trajectories column-sharded over the N synchronous
learners; --weak gives every rank its own B = 8192.
Without WORLD_SIZE in the environment, ``--gpus N`` (N > 1) launches the N ranks
itself (torch.distributed.run, 127.0.0.1) and exits with their status.

Workload (default): BASELINE.json configs[3], "large": T=100, B=8192, A=18,
bf16 logits, clip[-1,1] rewards; inputs resident in HBM, rotated over R copies
so every step reads cold data (R x working set >= 4 x L2).

``--impl reference``: the CPU oracle (oracle/, the only reference this tier
has) timed on the host cores on bounded column samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
PREROLL_S = 0.2  # untimed graph replays before the timed region (clock settle)
SPIN_CYCLES = 400_000  # device spin (~0.2 ms) queued ahead of a timed region's start event
METRIC = "V-trace+loss+grad trajectory-steps/s and HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "trajectory-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="large")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank gets the config's B (default at N > 1: "
                         "strong scaling, the config's B is the GLOBAL batch)")
    ap.add_argument("--strong", action="store_true", help=argparse.SUPPRESS)  # (the default)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--reserve-sms", type=int, default=1,
                    help="N > 1: SMs the kernel leaves to the per-step NCCL collective so that "
                         "steps can overlap (0: no overlap at N > 1)")
    ap.add_argument("--collective", choices=["nvlink", "fused", "nccl", "off"], default="nvlink",
                    help="N > 1: how the step's 8 partials are summed over the learners: "
                         "vtrace_partials_allreduce over NVLink peer memory (default), inside "
                         "the V-trace kernel's last CTA (fused), or NCCL")
    ap.add_argument("--no-guard", action="store_true", help=argparse.SUPPRESS)  # (A/B only)
    ap.add_argument("--exchange-every", type=int, default=0,
                    help="N > 1, --collective nvlink: steps whose partials are exchanged together "
                         "in one side-stream kernel (1 = every step; 0 = auto: 4 when at least 8 "
                         "input sets rotate, else 1)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="plain stream order between steps (no programmatic dependent launch)")
    ap.add_argument("--path", choices=["vtrace", "update", "head", "head_fused"], default="vtrace",
                    help="update: the learner's parameter update after the backward "
                         "(SURVEY 8(f) NEXT #4: gradient all-reduce at N > 1, global-norm "
                         "clip, RMSProp) instead of the V-trace path; head: the tcgen05 output "
                         "layer [z|V] = hW + b in front of the path (NEXT #3)")
    ap.add_argument("--update-collective", choices=["symm", "symm_push", "symm_sharded", "nccl"],
                    default="symm",
                    help="N > 1 on the update path: symm = the kernel sums every learner's "
                         "gradient over NVLink from symmetric memory (fused); nccl = NCCL "
                         "all_reduce then the single-gradient kernel")
    ap.add_argument("--update-size", default="deep",
                    help="parameters of the update path: shallow (1.2M), deep (1.6M, "
                         "P:285-286) or an integer")
    ap.add_argument("--behaviour", choices=["logits", "log_probs"], default="logits",
                    help="log_probs: the actors ship log mu(a_t) [T,B] instead of mu's "
                         "[T,B,A] logits (SURVEY 8(f) NEXT #2 input mode)")
    return ap.parse_args()


def with_behaviour_log_probs(inp):
    """Input preparation for --behaviour log_probs (outside any timed region): the
    actors' log mu(a_t) for the sampled actions, by a plain numpy fp64 log-softmax of
    the generated behaviour logits, rounded to fp32."""
    import numpy as np
    from paper_1802_01561_b200 import workload as wl
    zm = inp["behaviour_logits"]
    if inp["dtype"] == wl.DTYPE_BF16:
        zm = (zm.astype(np.uint32) << 16).view(np.float32)
    zm = zm.astype(np.float64)
    mx = zm.max(-1, keepdims=True)
    lse = np.log(np.exp(zm - mx).sum(-1)) + mx[..., 0]
    za = np.take_along_axis(zm, inp["actions"][..., None].astype(np.int64), -1)[..., 0]
    return dict(inp, behaviour_log_probs=(za - lse).astype(np.float32))


# ---------------------------------------------------------------------------
# distributed plumbing


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(world, local):
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()

    def summary(self, t0=None, t1=None):
        out = self._summary(t0, t1)
        if out["samples"] == 0 and t0 is not None:
            # a timed region shorter than the 50 ms sampling period (e.g. --steps 20) can
            # fall between two samples: take the samples within 100 ms of it (the GPU is under
            # the same load then: the untimed graph pre-roll runs right before it), stated
            out = self._summary(t0 - 0.1, t1 + 0.04)
            out["window"] = "timed region +- 100 ms (shorter than the 50 ms sampling period)"
        return out

    def _summary(self, t0=None, t1=None):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, line in self.lines:
            if t0 is not None and (ts < t0 or ts > t1 + 0.06):
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_traffic(config_name: str):
    """dram bytes per launch of the fused kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(config_name)
    except (OSError, ValueError):
        return None


def algorithmic_bytes(T, B, A, elem, mu_lp=False):
    """Bytes the method must move per call: read both logits rows,
    a, r, gamma, V; write dlogits, dV; plus the bootstrap row and 64 B partials.
    Behaviour as log mu(a_t): one logits row + 4 B of log-prob instead of two rows."""
    if mu_lp:
        return T * B * (2 * A * elem + 24) + 4 * B + 64
    return T * B * (3 * A * elem + 20) + 4 * B + 64


def make_rank_inputs(cfg, rank, world, strong):
    """Strong scaling: this rank's column shard of the config's global batch (shards of
    8-column units, so every shard keeps 16-byte TMA segments); weak: its own batch."""
    from paper_1802_01561_b200 import learner
    from paper_1802_01561_b200 import workload as wl
    if strong and world > 1:
        full = wl.make_inputs(cfg.name)
        b0, b1 = learner.shard_columns(cfg.B, world, rank, align=8 if cfg.B % 8 == 0 else 1)
        return wl.column_slice(full, b0, b1)
    return wl.make_inputs(cfg.name, seed=cfg.seed + 7919 * rank)


# ---------------------------------------------------------------------------
# our arm


def run_ours(args):
    world, rank, local = dist_env()
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    import paper_1802_01561_b200 as pkg
    from paper_1802_01561_b200 import learner
    from paper_1802_01561_b200 import vtrace as vt
    from paper_1802_01561_b200 import workload as wl

    cfg = wl.CONFIGS[args.config]
    strong = not args.weak
    inp = make_rank_inputs(cfg, rank, world, strong)
    mu_lp = args.behaviour == "log_probs"
    if mu_lp:
        inp = with_behaviour_log_probs(inp)
    T, B, A = inp["T"], inp["B"], inp["A"]
    B_global = B * world if not strong else cfg.B
    elem = 2 if inp["dtype"] == wl.DTYPE_BF16 else 4
    host = pkg.tensors_from_workload(inp, "cpu", pin=True)
    base = {k: v.to("cuda", non_blocking=True) for k, v in host.items()}
    in_bytes = sum(v.numel() * v.element_size() for v in base.values())
    out_bytes = T * B * A * elem + T * B * 4 + 64
    working = in_bytes + out_bytes
    R = max(1, math.ceil(4 * L2_BYTES / working))
    sets = [base] + [{k: v.clone() for k, v in base.items()} for _ in range(R - 1)]
    outs = [{"grad_target_logits": torch.empty(T, B, A, dtype=base["target_logits"].dtype,
                                               device="cuda"),
             "grad_values": torch.empty(T, B, dtype=torch.float32, device="cuda"),
             "partials": torch.zeros(8, dtype=torch.float64, device="cuda")} for _ in range(R)]
    kw = dict(reward_mode=inp["reward_mode"], baseline_cost=wl.BASELINE_COST,
              entropy_cost=wl.ENTROPY_COST, rho_bar=wl.RHO_BAR, c_bar=wl.C_BAR)
    # the product's learner step: kernel on the main stream, step k's partials
    # all-reduce on a side stream under step k+1's kernel, consecutive steps overlapped
    # (programmatic dependent launch: every step reads a fresh rotated batch), one SM
    # left to the collective at N > 1
    overlap = not args.no_overlap
    step_obj = learner.LearnerStep(T, B, A, inp["dtype"], overlap=overlap,
                                   reserve_sms=(args.reserve_sms if world > 1 else 0),
                                   collective=args.collective,
                                   guard_partials=not args.no_guard,
                                   exchange_every=(1 if args.collective != "nvlink" else
                                                   args.exchange_every if args.exchange_every > 0
                                                   else (4 if R >= 8 else 1)),
                                   **kw)
    ws = step_obj.workspace
    s_main = step_obj.stream

    def step(i):
        step_obj(sets[i % R], outs[i % R])

    # eager warm-up (also creates the NCCL communicator before any capture)
    for i in range(max(args.warmup, 1)):
        step(i)
    step_obj.join()
    torch.cuda.synchronize()
    barrier(world)

    # graphs of C steps (C a multiple of R) + a remainder graph: exactly K steps
    K = args.steps
    C = R * max(1, math.ceil(min(K, 100) / R))
    n_full, rem = divmod(K, C)
    graph_mode = "cuda-graph"

    def capture(nsteps):
        return step_obj.capture([(sets[i % R], outs[i % R]) for i in range(nsteps)])

    try:
        g_full = capture(C) if n_full else None
        g_rem = capture(rem) if rem else None
    except Exception as e:  # noqa: BLE001
        graph_mode = f"eager ({type(e).__name__} in capture)"
        g_full = g_rem = None
    torch.cuda.synchronize()

    def run_timed_body():
        if g_full is None and g_rem is None:
            for i in range(K):
                step(i)
            step_obj.join()
        else:
            with torch.cuda.stream(s_main):
                for _ in range(n_full):
                    g_full.replay()
                if g_rem is not None:
                    g_rem.replay()

    # warm the graphs (untimed): replays for at least PREROLL_S of GPU time, so that the
    # timed K steps run at the settled SM clock (a 20-step region right after a cold start
    # otherwise catches the clock ramp: 31.3 vs 27.3 us per step at `large`)
    # The replay count is agreed over the ranks (the graphs hold the collectives: ranks
    # that replayed different counts would wait for each other forever).
    preroll_reps = 0
    if g_full is not None or g_rem is not None:
        gw = g_rem or g_full
        for _ in range(2):  # the first replay uploads the graph: time the second
            t_pre = time.time()
            with torch.cuda.stream(s_main):
                gw.replay()
            torch.cuda.synchronize()
        one = max(time.time() - t_pre, 1e-6)
        reps = min(10000, max(2, math.ceil(PREROLL_S / one)))
        reps = int(max_over_ranks(float(reps), world))
        for _ in range(reps - 2):
            with torch.cuda.stream(s_main):
                gw.replay()
        preroll_reps = reps
    torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
    barrier(world)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    tw0 = time.time()
    # a ~0.2 ms device-side spin ahead of the start event: the graphs are queued behind it,
    # so the timed region holds the K steps and not the host's first graph submission
    # (which a 20-step run would otherwise count: 30.7 vs 27.5 us per step at `large`)
    with torch.cuda.stream(s_main):
        torch.cuda._sleep(SPIN_CYCLES)
    ev0.record(s_main)
    run_timed_body()
    ev1.record(s_main)
    ev1.synchronize()
    torch.cuda.synchronize()
    tw1 = time.time()
    barrier(world)
    if sampler:
        sampler.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    elapsed_max = max_over_ranks(elapsed_ms, world)
    kw_step = dict(kw, overlap_previous=overlap, sm_budget=step_obj.kw["sm_budget"])

    # multi-GPU correctness of the step's collective (untimed): one more step through the
    # product API against an NCCL all_reduce of the same per-rank partials
    collective_check = None
    if world > 1 and step_obj.collective != "off":
        o = outs[0]
        pkg.loss_and_grad(*[sets[0][k] for k in vt.INPUT_NAMES], workspace=ws, out=o, **kw)
        torch.cuda.synchronize()
        local = o["partials"].clone()
        step_obj(sets[0], o)
        step_obj.join()
        torch.cuda.synchronize()
        ref = local.clone()
        dist.all_reduce(ref, op=dist.ReduceOp.SUM)
        torch.cuda.synchronize()
        rel = float(((o["partials"] - ref).abs() / ref.abs().clamp_min(1e-300)).max())
        agree = torch.tensor([o["partials"].sum().item()], dtype=torch.float64, device="cuda")
        gathered = [torch.zeros_like(agree) for _ in range(world)]
        dist.all_gather(gathered, agree)
        collective_check = {"max_rel_diff_vs_nccl": rel,
                            "identical_on_every_rank": all(bool(torch.equal(gathered[0], g))
                                                           for g in gathered[1:])}

    # kernel-only timing for the roofline: the same kernels, no collective
    Kk = min(K, 2000)
    gk = None
    try:
        gk = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gk, stream=s_main):
            for i in range(min(Kk, C)):
                o = outs[i % R]
                x = sets[i % R]
                pkg.loss_and_grad(*[x[k] for k in vt.INPUT_NAMES], workspace=ws, out=o, **kw_step)
    except Exception:  # noqa: BLE001
        gk = None
    torch.cuda.synchronize()
    # at least 200 launches (a replay first, untimed: the graph upload), queued behind a
    # device spin like the main timed region
    reps = max(1, Kk // min(Kk, C), math.ceil(200 / min(Kk, C)))
    if gk is not None:
        with torch.cuda.stream(s_main):
            gk.replay()
        torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_main):
        torch.cuda._sleep(SPIN_CYCLES)
    e0.record(s_main)
    with torch.cuda.stream(s_main):
        for r_ in range(reps):
            if gk is not None:
                gk.replay()
            else:  # (capture failed: the same launches eagerly)
                for i in range(min(Kk, C)):
                    x = sets[i % R]
                    pkg.loss_and_grad(*[x[k] for k in vt.INPUT_NAMES], workspace=ws,
                                      out=outs[i % R], **kw_step)
    e1.record(s_main)
    torch.cuda.synchronize()
    kernel_ms = e0.elapsed_time(e1) / (reps * min(Kk, C))

    # eager launches (no graph): the latency-bound configs' per-call time
    Ke = min(K, 500)
    for i in range(5):
        step(i)
    step_obj.join()
    torch.cuda.synchronize()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record(s_main)
    for i in range(Ke):
        step(i)
    step_obj.join()
    ee1.record(s_main)
    torch.cuda.synchronize()
    eager_ms = max_over_ranks(ee0.elapsed_time(ee1), world) / Ke

    # end-to-end through the public host-input API
    e2e = None
    if not args.no_e2e:
        Ke = args.e2e_steps
        part_h = torch.zeros(8, dtype=torch.float64).pin_memory()
        o = outs[0]
        with torch.cuda.stream(s_main):
            pkg.loss_and_grad_from_host(host, sets[0], o, ws, part_h, **kw)
        torch.cuda.synchronize()
        barrier(world)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(s_main)
        with torch.cuda.stream(s_main):
            for i in range(Ke):
                pkg.loss_and_grad_from_host(host, sets[i % R], o, ws, part_h, **kw)
                if world > 1:
                    dist.all_reduce(o["partials"])
        eb.record(s_main)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(ea.elapsed_time(eb), world) / Ke
        e2e = {"value": T * B_global / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": 64,
               "ms_per_step": e2e_ms}

    # status check (data errors would void the run)
    code, idx = pkg.read_device_status(ws)
    if code != 0:
        raise SystemExit(f"device status reported data error {code} at row {idx}")

    cpu = cpu_par = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(inp, args.cpu_seconds)
        cpu_par = cpu_baseline_parallel(inp)

    if rank != 0:
        return
    ms_per_step = elapsed_max / K
    value = T * B_global / (ms_per_step * 1e-3)
    peak, peak_src = load_peak()
    alg = algorithmic_bytes(T, B, A, elem, mu_lp)
    achieved = alg / (kernel_ms * 1e-3) / 1e9
    traffic = load_traffic(args.config + ("+behaviour_log_probs" if mu_lp else ""))
    clocks = sampler.summary(tw0, tw1) if sampler else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if strong and world > 1 else "weak", "vs_baseline": None,
        "dtype": ("bf16" if elem == 2 else "f32") + " logits; f32 exps with compensated "
                 "(exact-order) sums, f64 ratio and scan, f32 gradient epilogue",
        "data": "synthetic (seeded, DMLab/Atari-shaped; DESIGN.md input recipe)",
        "config": {"workload": cfg.name + ("+behaviour_log_probs" if mu_lp else ""),
                   "T": T, "B_per_gpu": B, "A": A, "behaviour": args.behaviour,
                   "logits_dtype": "bf16" if elem == 2 else "fp32",
                   "global_batch": B_global, "seq_len": T, "parallelism": f"dp{world}",
                   "l2": f"inputs rotated over {R} HBM-resident copies "
                         f"({R} x {working / 1e6:.1f} MB >= 4 x L2)",
                   "timing": graph_mode + " (queued behind a 0.2 ms device spin: the host's "
                                          "graph submission is outside the timed region)",
                   "warmup_detail": f"{args.warmup} eager steps + {preroll_reps} untimed graph "
                                    f"replays (>= {PREROLL_S} s, clock settle)",
                   "step_overlap": "programmatic dependent launch (overlap_previous: inputs are "
                                   "fresh batches)" if overlap else "none",
                   "collective": ("none" if world == 1 else
                                  ("vtrace_partials_allreduce: 8 fp64 partials per step through "
                                   "peer-mapped mailboxes over NVLink, one 32-thread kernel"
                                   + (f" per {step_obj.exchange_every} steps (batched)"
                                      if step_obj.exchange_every > 1 else " per step")
                                   if step_obj.collective == "nvlink" else
                                   "inside the V-trace kernel: its last CTA exchanges the 8 "
                                   "partials through peer-mapped mailboxes over NVLink "
                                   "(vtrace_loss_and_grad_learners)"
                                   if step_obj.collective == "fused" else
                                   "NCCL all_reduce of 8 fp64 partials per step")
                                  + " (side stream"
                                  + (f", {args.reserve_sms} SM reserved)" if args.reserve_sms
                                     else ")")),
                   "step": "paper_1802_01561_b200.learner.LearnerStep",
                   **({"collective_fallback": step_obj.collective_fallback}
                      if getattr(step_obj, "collective_fallback", None) else {})},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": vt.kernel_for(T, B, A, inp["dtype"]), "kernel_ms": kernel_ms,
                     "algorithmic_bytes_per_launch": alg, "peak_source": peak_src},
        "gpu_launches": K,  # one fused kernel per step
        "collective_check": collective_check,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "cpu_baseline_parallel": cpu_par,
        "eager_ms_per_step": eager_ms,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the oracle on the host cores


def cpu_baseline(inp, seconds):
    """The oracle as it stands (single-threaded fp64) on the host cores: whole-batch
    passes (or a column sample of one) repeated for about `seconds`."""
    import oracle
    from paper_1802_01561_b200 import workload as wl
    T, B = inp["T"], inp["B"]
    small = wl.column_slice(inp, 0, min(B, 64))
    t0 = time.perf_counter()
    oracle.loss_and_grad(small, reward_mode=inp["reward_mode"])
    dt = time.perf_counter() - t0
    rate_cols = small["B"] / max(dt, 1e-6)
    ncols = int(max(1, min(B, rate_cols * seconds)))
    sample = wl.column_slice(inp, 0, ncols)
    reps, t_all = 0, 0.0
    while reps == 0 or (t_all < seconds and reps < 50):
        t0 = time.perf_counter()
        oracle.loss_and_grad(sample, reward_mode=inp["reward_mode"])
        t_all += time.perf_counter() - t0
        reps += 1
    return {"value": T * ncols * reps / t_all, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"columns [0,{ncols}) of the {inp['T']}x{B} batch (T={T}), "
                      f"oracle.loss_and_grad single-threaded fp64, {reps} pass(es) in {t_all:.1f} s",
            "host_cpu": _cpu_model()}


def cpu_baseline_parallel(inp, passes=3):
    """the same oracle function over column ranges on every host core
    (ctypes releases the GIL during the call); whole-batch passes."""
    import concurrent.futures as cf
    import oracle
    from paper_1802_01561_b200 import workload as wl
    T, B = inp["T"], inp["B"]
    n = max(1, min(os.cpu_count() or 1, B))
    bounds = [(i * B // n, (i + 1) * B // n) for i in range(n)]
    parts = [wl.column_slice(inp, b0, b1) for b0, b1 in bounds if b1 > b0]
    oracle.loss_and_grad(parts[0], reward_mode=inp["reward_mode"])  # build / load first
    with cf.ThreadPoolExecutor(max_workers=len(parts)) as ex:
        t0 = time.perf_counter()
        for _ in range(passes):
            list(ex.map(lambda x: oracle.loss_and_grad(x, reward_mode=inp["reward_mode"]), parts))
        dt = time.perf_counter() - t0
    return {"value": T * B * passes / dt, "unit": UNIT, "cores": len(parts), "kind": "oracle",
            "sample": f"the whole {T}x{B} batch, {passes} passes, columns split over "
                      f"{len(parts)} threads, {dt:.1f} s", "host_cpu": _cpu_model()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle
    import oracle
    from paper_1802_01561_b200 import workload as wl
    cfg = wl.CONFIGS[args.config]
    inp = wl.make_inputs(cfg.name)
    if args.behaviour == "log_probs":
        inp = with_behaviour_log_probs(inp)
    T, B = inp["T"], inp["B"]
    # size each step's column sample so the whole run takes ~1-2 minutes
    probe = wl.column_slice(inp, 0, min(B, 32))
    t0 = time.perf_counter()
    oracle.loss_and_grad(probe, reward_mode=inp["reward_mode"])
    per_col = (time.perf_counter() - t0) / probe["B"]
    budget = 90.0 / max(1, args.steps + args.warmup)
    ncols = int(max(1, min(B, budget / max(per_col, 1e-9))))
    sample = wl.column_slice(inp, 0, ncols)
    for _ in range(args.warmup):
        oracle.loss_and_grad(sample, reward_mode=inp["reward_mode"])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.loss_and_grad(sample, reward_mode=inp["reward_mode"])
    dt = time.perf_counter() - t0
    value = args.steps * T * ncols / dt
    desc = (f"each step: oracle.loss_and_grad (fp64, single-threaded) on columns [0,{ncols}) "
            f"of the {T}x{B} '{cfg.name}' batch")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name + ("+behaviour_log_probs" if args.behaviour == "log_probs" else ""), "T": T, "B_sample": ncols, "A": inp["A"],
                       "global_batch": ncols, "seq_len": T, "parallelism": "cpu-1core"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": desc, "host_cpu": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# --path update: the learner's parameter update


def _rms_stamp_summary(e0, e1, rank):
    """(dev) medians of the RMS_TIMING stamps of calls [e0, e1) (the last 4000 at most)."""
    import ctypes
    import numpy as np
    import paper_1802_01561_b200 as pkg
    lib = pkg.load_library()
    buf = (ctypes.c_ulonglong * (8 * 4096))()
    lib.vtrace_debug_rms_stamps.argtypes = [ctypes.c_void_p]
    lib.vtrace_debug_rms_stamps(ctypes.addressof(buf))
    st = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)
    ep = np.arange(max(e0, e1 - 4000), e1)
    a = st[ep % 4096]
    d = lambda i, j: float(np.median(a[:, j] - a[:, i]) / 1e3)  # noqa: E731
    per = np.diff(a[:, 0]) / 1e3
    print(json.dumps({"rank": rank, "calls": int(len(ep)),
                      "period_us": float(np.median(per)), "period_mean_us": float(per.mean()),
                      "period_max_us": float(per.max()),
                      "gaps_over_100us": int((per > 100).sum()),
                      "gap_positions": [int(i) for i in np.nonzero(per > 100)[0][:12]],
                      "ready_pub": d(0, 1), "wait_peers_ready": d(1, 2), "reads_norm": d(2, 3),
                      "update": d(3, 4), "to_done_pub": d(4, 5), "wait_peers_done": d(5, 6),
                      "gap_to_next_start": float(np.median(a[1:, 0] - a[:-1, 6]) / 1e3)}),
          file=sys.stderr, flush=True)


def run_update(args):
    """K synchronous learner updates of n parameters: (N > 1) NCCL SUM all-reduce of
    the fp32 gradient, then vtrace_rmsprop_step (clip 40, RMSProp) on every
    replica.  `value` = parameters updated per second (the replicas update the same
    parameters: the job's rate, not N times it)."""
    world, rank, local = dist_env()
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    import paper_1802_01561_b200 as pkg
    from paper_1802_01561_b200 import learner
    from paper_1802_01561_b200 import workload as wl
    size = args.update_size
    n = wl.UPDATE_SIZES[size] if size in wl.UPDATE_SIZES else int(size)
    # replicas start equal (one seed for parameters and mean squares); each learner
    # has its own gradient (its shard of the batch)
    inp = wl.update_inputs(n, seed=1, norm=80.0 / math.sqrt(world))
    if rank > 0:
        inp["grads"] = wl.update_inputs(n, seed=1 + rank, norm=80.0 / math.sqrt(world))["grads"]
    lr, decay, eps, clip = 6e-4, 0.99, 0.01, 40.0  # P:950-953 (decay: reading r9)
    per = 3 * 4 * n  # params, mean square, grads resident per copy
    R = max(1, math.ceil(4 * L2_BYTES / per))
    theta = [torch.from_numpy(inp["params"]).cuda() for _ in range(R)]
    ms = [torch.from_numpy(inp["mean_square"]).cuda() for _ in range(R)]
    grads = [torch.from_numpy(inp["grads"][0]).cuda() for _ in range(R)]
    norm = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = pkg.RmspropWorkspace(n)
    s_main = torch.cuda.Stream()

    symm = world > 1 and args.update_collective in ("symm", "symm_sharded", "symm_push")
    sharded = world > 1 and args.update_collective == "symm_sharded"
    push = world > 1 and args.update_collective == "symm_push"
    red = hdl = ptrs = None
    if symm:
        # the learners' gradient buffers in symmetric memory: every GPU maps every
        # other's, and the update kernel sums them (rank order) over NVLink
        import torch.distributed._symmetric_memory as symm_mem
        red = symm_mem.empty(n, dtype=torch.float32, device="cuda")
        hdl = symm_mem.rendezvous(red, dist.group.WORLD.group_name)
        ptrs = [int(p) for p in hdl.buffer_ptrs]
        # each learner's {ready, done} words: the learners synchronise inside the kernel
        flg = symm_mem.empty(2, dtype=torch.int32, device="cuda")
        flg.zero_()
        hdl_f = symm_mem.rendezvous(flg, dist.group.WORLD.group_name)
        fptrs = [int(p) for p in hdl_f.buffer_ptrs]
        if push:
            # every learner's receive buffer [N][n]: slot j holds learner j's pushed gradient
            recv = symm_mem.empty(world * n, dtype=torch.float32, device="cuda")
            hdl_r = symm_mem.rendezvous(recv, dist.group.WORLD.group_name)
            rptrs = [int(p) for p in hdl_r.buffer_ptrs]
            lslots = [rptrs[rank] + 4 * j * n for j in range(world)]
        if sharded:
            # every learner's R parameter copies in one symmetric allocation: a learner
            # writes its shard of the new theta into all of them (NVLink stores)
            th_all = symm_mem.empty(R * n, dtype=torch.float32, device="cuda")
            hdl_t = symm_mem.rendezvous(th_all, dist.group.WORLD.group_name)
            for j in range(R):
                th_all[j * n:(j + 1) * n].copy_(theta[j])
            theta = [th_all[j * n:(j + 1) * n] for j in range(R)]
            tptrs = [[int(p) + 4 * j * n for p in hdl_t.buffer_ptrs] for j in range(R)]
            nmb = symm_mem.empty(pkg.vtrace.rmsprop_norm_mailbox_bytes(world) // 8,
                                 dtype=torch.float64, device="cuda")
            nmb.zero_()
            hdl_n = symm_mem.rendezvous(nmb, dist.group.WORLD.group_name)
            nptrs = [int(p) for p in hdl_n.buffer_ptrs]
        torch.cuda.synchronize()
        barrier(world)
    elif world > 1:
        red = torch.empty_like(grads[0])

    def step(i, allreduce=True):
        j = i % R
        if symm:
            if allreduce:
                # this step's local gradient (the backward's output) -- an SM kernel: a
                # captured D2D copy_ measured ~70 us per 6.4 MB in graph replay at N = 2
                torch.mul(grads[j], 1.0, out=red)
            if push:  # the gradient pushed into every learner's slot, then local reads only
                if allreduce:
                    pkg.vtrace.grad_push(grads[j], rptrs, rank)
                pkg.rmsprop_step(theta[j], ms[j], lslots, lr, decay, eps, clip,
                                 global_norm_out=norm, workspace=ws, learner_flags=fptrs,
                                 self_index=rank)
                return
            if sharded:  # this learner's 1/N of the parameters, new theta to every learner
                pkg.vtrace.rmsprop_step_sharded(tptrs[j], ms[j], ptrs, lr, decay, eps, clip,
                                                flags=fptrs, norm_mailboxes=nptrs,
                                                self_index=rank, n=n, workspace=ws,
                                                global_norm_out=norm)
                return
            # every learner's buffer summed over NVLink in rank order; ready / done flags
            # inside the kernel replace the barriers around it
            pkg.rmsprop_step(theta[j], ms[j], ptrs, lr, decay, eps, clip,
                             global_norm_out=norm, workspace=ws, learner_flags=fptrs,
                             self_index=rank)
            return
        g = grads[j]
        if allreduce and world > 1:
            # a fresh local gradient each step (the backward's output), summed in place
            torch.mul(grads[j], 1.0, out=red)  # (an SM kernel, as on the fused path)
            learner.allreduce_grads(red)
            g = red
        pkg.rmsprop_step(theta[j], ms[j], g, lr, decay, eps, clip,
                         global_norm_out=norm, workspace=ws)

    with torch.cuda.stream(s_main):
        for i in range(max(args.warmup, 3)):
            step(i)
    torch.cuda.synchronize()
    barrier(world)
    K = args.steps

    # eager Python loop (host launch rate included)
    Ke = min(K, 500)
    q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q0.record(s_main)
    with torch.cuda.stream(s_main):
        for i in range(Ke):
            step(i)
    q1.record(s_main)
    torch.cuda.synchronize()
    eager_ms = max_over_ranks(q0.elapsed_time(q1), world) / Ke

    # CUDA graphs of R consecutive steps (one per rotated copy), replayed: exactly K
    def capture(nsteps, allreduce=True):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s_main):
            for i in range(nsteps):
                step(i, allreduce)
        return g

    n_full, rem = divmod(K, R)
    timing_mode = "cuda-graph of R steps, replayed (eager loop: eager_ms_per_step)"
    try:
        g_full, g_rem = capture(R), (capture(rem) if rem else None)
    except Exception as e:  # (a collective that cannot be captured: eager timing)
        g_full = g_rem = None
        timing_mode = f"eager (capture failed: {type(e).__name__})"
    torch.cuda.synchronize()
    barrier(world)

    def timed(gf, gr, allreduce=True):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        barrier(world)  # (the learners sync inside the kernels: start the region together)
        t0.record(s_main)
        with torch.cuda.stream(s_main):
            if gf is None:
                for i in range(K):
                    step(i, allreduce)
            else:
                th = []
                for _ in range(n_full):
                    h0 = time.perf_counter()
                    gf.replay()
                    th.append((time.perf_counter() - h0) * 1e6)
                if gr is not None:
                    gr.replay()
                if os.environ.get("VT_RMS_STAMPS"):
                    print(json.dumps({"rank": rank, "graph_replay_host_us": [round(x) for x in th[:12]],
                                      "host_total_us": round(sum(th))}), file=sys.stderr)
        t1.record(s_main)
        torch.cuda.synchronize()
        return max_over_ranks(t0.elapsed_time(t1), world) / K

    # the clock sampler starts BEFORE the ranks line up: its start (a subprocess) took ~150 ms
    # on rank 0, during which the other rank's first update waited inside the kernel for
    # rank 0's ready flag -- 150 ms / 2000 steps was the "graph penalty" of the round-1
    # N = 2 update numbers (profiles/r2_update_n2_stamps.txt)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    barrier(world)
    torch.cuda.synchronize()
    tw0 = time.time()
    e_first = int(ws.tensor[:4].view(torch.int32).item()) if os.environ.get("VT_RMS_STAMPS") else 0
    step_ms = timed(g_full, g_rem)
    if os.environ.get("VT_RMS_STAMPS"):  # RMS_TIMING builds only: per-call stamps of the region
        _rms_stamp_summary(e_first, int(ws.tensor[:4].view(torch.int32).item()), rank)
    tw1 = time.time()
    barrier(world)
    if sampler:
        sampler.stop()
    # the replicas must agree bitwise (same buffers, same order, same arithmetic)
    replicas_equal = None
    if world > 1:
        # exact checksums of the bits (int64 sums of the fp32 words, two weightings); the
        # sharded update keeps theta replicated and each learner's own shard of ms
        def bits(t):
            w = t.view(torch.int32).long()
            idx = torch.arange(w.numel(), device=w.device, dtype=torch.int64) % 1009
            return [int(w.sum()), int((w * idx).sum())]
        h = torch.tensor(bits(theta[0]) + ([] if sharded else bits(ms[0])), dtype=torch.int64,
                         device="cuda")
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        replicas_equal = all(bool(torch.equal(hs[0], x)) for x in hs[1:])
    graph_ms = step_ms
    if world > 1 and eager_ms < step_ms:
        # (at N = 2 graph replay measured slower than the eager loop for both the NCCL
        # and the fused path -- DESIGN.md 9b; the faster of the two real runs is kept)
        step_ms = eager_ms
        timing_mode = "eager loop (faster than graph replay at this N; both reported)"
    # the update kernel alone (roofline): the same graphs without the collective
    if world > 1:
        if g_full is None:
            kernel_ms = timed(None, None, False)
        else:
            k_full, k_rem = capture(R, False), (capture(rem, False) if rem else None)
            kernel_ms = timed(k_full, k_rem)
    else:
        kernel_ms = step_ms

    # end to end: this step's gradient from pinned host memory, the norm read back
    e2e = None
    if not args.no_e2e:
        g_host = torch.from_numpy(inp["grads"][0]).pin_memory()
        n_host = torch.zeros(1, dtype=torch.float64).pin_memory()
        Ke = min(K, 200)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s_main)
        with torch.cuda.stream(s_main):
            for i in range(Ke):
                grads[i % R].copy_(g_host, non_blocking=True)
                step(i)
                n_host.copy_(norm, non_blocking=True)
        a1.record(s_main)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(a0.elapsed_time(a1), world) / Ke
        e2e = {"value": n / (e2e_ms * 1e-3), "unit": "params/s", "h2d_bytes_per_step": 4 * n,
               "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import rmsprop_oracle as ro
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < min(args.cpu_seconds, 5.0) or reps == 0:
            ro.rmsprop_step(inp["params"], inp["mean_square"], inp["grads"][0], lr, decay, eps,
                            clip)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        cpu = {"value": n / dt, "unit": "params/s", "cores": 1, "kind": "oracle",
               "sample": f"{reps} full updates of the same {n} parameters (numpy fp64)"}
    if rank != 0:
        return
    peak, peak_src = load_peak()
    alg = 20 * n  # g 4 B + ms 4+4 B + theta 4+4 B per parameter
    achieved = alg / (kernel_ms * 1e-3) / 1e9
    line = {
        "metric": "learner_update_params_per_s", "value": n / (step_ms * 1e-3),
        "unit": "params/s", "n_gpus": world, "steps": K, "warmup": max(args.warmup, 3),
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "replicated",
        "vs_baseline": None, "dtype": "f32 (f64 global norm)", "path": "update",
        "data": "synthetic (seeded gradient of global norm 80, N(0, 0.05^2) parameters)",
        "config": {"workload": f"learner update, {size} model ({n} parameters)",
                   "n_params": n, "optimizer": "RMSProp momentum 0, decay 0.99, eps 0.01, "
                   "lr 6e-4, clip global norm 40 (P:950-953)",
                   "collective": (("per step: the local gradient pushed into every learner's "
                                   "receive slot (NVLink stores, vtrace_grad_push); ONE kernel "
                                   "syncs the learners and sums the local slots (rank order)")
                                  if push else
                                  ("per step: local gradient into symmetric memory; ONE kernel "
                                   "per learner updates its 1/N shard from every learner's "
                                   "gradient (NVLink reads), adds the shards' norms through "
                                   "mailboxes and stores the new theta into every replica "
                                   "(NVLink writes)") if sharded else
                                  "per step: local gradient into symmetric memory; ONE kernel "
                                  "syncs the learners (ready/done flags over NVLink), sums "
                                  "every learner's buffer (rank order) and updates" if symm else
                                  "per step: copy of the local fp32 gradient + NCCL all_reduce "
                                  "SUM of it, then the update kernel") if world > 1 else "none",
                   "l2": f"state rotated over {R} HBM-resident copies ({R} x {per / 1e6:.1f} MB "
                         ">= 4 x L2)", "parallelism": f"dp{world}",
                   "timing": timing_mode},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": load_traffic("update:" + str(size)),
                     "kernel": "rmsprop_reg_kernel" if n <= 148 * 512 * 24 else "rmsprop_kernel",
                     "kernel_ms": kernel_ms, "algorithmic_bytes_per_launch": alg,
                     "peak_source": peak_src},
        "gpu_launches": K,
        "clocks": sampler.summary(tw0, tw1) if sampler else None,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "eager_ms_per_step": eager_ms,
        "replicas_bitwise_equal": replicas_equal,
        "graph_ms_per_step": graph_ms,
    }
    print(json.dumps(line), flush=True)


# --path head: the output layer in front of the path


def run_head(args):
    """K launches of vtrace_output_layer at the `large` config's T*B rows (H = 256, A = 18).
    Each rank computes its own T*B rows (weak scaling, no collective).  h (419 MB) is
    larger than L2, and two copies are alternated, so no flush is needed."""
    world, rank, local = dist_env()
    init_dist(world, local)
    torch.cuda.set_device(local)
    import paper_1802_01561_b200 as pkg
    T, B, H, A = 100, 8192, 256, 18
    M = T * B
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    hs = [torch.randn((M, H), generator=g, device="cuda").to(torch.bfloat16) for _ in range(2)]
    w = (torch.randn((A + 1, H), generator=g, device="cuda") * 0.1).to(torch.bfloat16)
    b = torch.randn(A + 1, generator=g, device="cuda")
    z = torch.empty((M, A), device="cuda")
    v = torch.empty(M, device="cuda")
    s_main = torch.cuda.Stream()
    K, W = args.steps, max(args.warmup, 3)
    with torch.cuda.stream(s_main):
        for i in range(W):
            pkg.output_layer(hs[i % 2], w, b, z, v)
    torch.cuda.synchronize()
    barrier(world)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    tw0 = time.time()
    e0.record(s_main)
    with torch.cuda.stream(s_main):
        for i in range(K):
            pkg.output_layer(hs[i % 2], w, b, z, v)
    e1.record(s_main)
    torch.cuda.synchronize()
    tw1 = time.time()
    if sampler:
        sampler.stop()
    barrier(world)
    step_ms = max_over_ranks(e0.elapsed_time(e1), world) / K
    e2e = None
    if not args.no_e2e:  # h from pinned host memory, V read back, every step
        h_host = hs[0].cpu().pin_memory()
        v_host = torch.empty(M, dtype=torch.float32).pin_memory()
        Ke = min(K, 10)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s_main)
        with torch.cuda.stream(s_main):
            for i in range(Ke):
                hs[0].copy_(h_host, non_blocking=True)
                pkg.output_layer(hs[0], w, b, z, v)
                v_host.copy_(v, non_blocking=True)
        a1.record(s_main)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(a0.elapsed_time(a1), world) / Ke
        e2e = {"value": world * M / (e2e_ms * 1e-3), "unit": "rows/s",
               "h2d_bytes_per_step": M * H * 2, "d2h_bytes_per_step": M * 4, "ms_per_step": e2e_ms}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import output_layer_oracle as ol
        rows = 16384
        hh = hs[0][:rows].float().cpu().numpy().astype("float64").reshape(rows, 1, H)
        Wn = w.float().cpu().numpy().astype("float64").T
        bn = b.cpu().numpy().astype("float64")
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < min(args.cpu_seconds, 5.0) or reps == 0:
            ol.output_layer(hh, Wn, bn)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        cpu = {"value": rows / dt, "unit": "rows/s", "cores": torch.get_num_threads(),
               "kind": "oracle", "sample": f"{reps} x oracle.output_layer_oracle.output_layer on "
               f"rows [0, {rows}) (numpy fp64 matmul, BLAS threads)"}
    if rank != 0:
        return
    peak, peak_src = load_peak()
    alg = M * H * 2 + (A + 1) * H * 2 + M * (A + 1) * 4 + (A + 1) * 4
    achieved = alg / (step_ms * 1e-3) / 1e9
    line = {
        "metric": "output_layer_rows_per_s", "value": world * M / (step_ms * 1e-3),
        "unit": "rows/s", "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16 in, f32 accumulate (tcgen05), f32 out", "path": "head",
        "data": "synthetic (seeded N(0,1) hidden, N(0,0.01) weights)",
        "config": {"workload": "output layer at large: T=100 B=8192 H=256 A=18",
                   "parallelism": f"dp{world}", "collective": "none",
                   "l2": "h (419 MB per copy, 2 copies alternated) exceeds L2", "timing": "eager"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": load_traffic("head:large"),
                     "kernel": "output_layer_kernel",
                     "kernel_ms": step_ms, "algorithmic_bytes_per_launch": alg,
                     "peak_source": peak_src},
        "gpu_launches": K,
        "clocks": sampler.summary(tw0, tw1) if sampler else None,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_head_fused(args):
    """K calls of vtrace_head_loss_and_grad (NEXT #3 second half) at the `large` config:
    T=100, B=8192 trajectories, H=256 hidden, A=18 -- the output layer with the V-trace loss
    and gradients as its epilogue and the head backward (dh, dW, db).  Each rank its own
    batch (weak scaling, no collective).  Two input sets alternated; h (419 MB) exceeds L2."""
    world, rank, local = dist_env()
    init_dist(world, local)
    torch.cuda.set_device(local)
    import paper_1802_01561_b200 as pkg
    T, B, H, A = 100, 8192, 256, 18
    M = T * B
    g = torch.Generator(device="cuda").manual_seed(200 + rank)
    w = (torch.randn((A + 1, H), generator=g, device="cuda") * 0.1).to(torch.bfloat16)
    bias = torch.randn(A + 1, generator=g, device="cuda") * 0.1
    sets = []
    for _ in range(2):
        h = torch.randn((T, B, H), generator=g, device="cuda").to(torch.bfloat16)
        z, _v = pkg.output_layer(h, w, bias)
        mu = (z + 0.3 * torch.randn(z.shape, generator=g, device="cuda")).contiguous()
        u = torch.rand(mu.shape, generator=g, device="cuda").clamp_(min=1e-12)
        act = torch.argmax(mu - torch.log(-torch.log(u)), dim=-1).to(torch.int32).contiguous()
        done = torch.rand((T, B), generator=g, device="cuda") < 0.01
        disc = torch.where(done, 0.0, 0.99).to(torch.float32).contiguous()
        rew = torch.randn((T, B), generator=g, device="cuda").contiguous()
        boot = torch.randn(B, generator=g, device="cuda")
        sets.append((h, mu, act, disc, rew, boot))
        del z, _v, u
    torch.cuda.empty_cache()
    ws = pkg.HeadWorkspace(T, B, H, A)
    out = {"grad_hidden": torch.empty((T, B, H), dtype=torch.bfloat16, device="cuda"),
           "grad_w_t": torch.empty((A + 1, H), device="cuda"),
           "grad_bias": torch.empty(A + 1, device="cuda"),
           "partials": torch.empty(8, dtype=torch.float64, device="cuda")}
    kw = dict(rho_bar=1.0, c_bar=1.0, baseline_cost=0.5, entropy_cost=0.01, workspace=ws, out=out)

    def step(i):
        h, mu, act, disc, rew, boot = sets[i % 2]
        pkg.head_loss_and_grad(h, w, bias, mu, act, disc, rew, boot, **kw)

    s_main = torch.cuda.Stream()
    K, W = args.steps, max(args.warmup, 3)
    with torch.cuda.stream(s_main):
        for i in range(W):
            step(i)
    torch.cuda.synchronize()
    barrier(world)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    tw0 = time.time()
    with torch.cuda.stream(s_main):
        torch.cuda._sleep(SPIN_CYCLES)  # (the first call's host launch outside the timing)
    e0.record(s_main)
    with torch.cuda.stream(s_main):
        for i in range(K):
            step(i)
    e1.record(s_main)
    torch.cuda.synchronize()
    tw1 = time.time()
    if sampler:
        sampler.stop()
    barrier(world)
    step_ms = max_over_ranks(e0.elapsed_time(e1), world) / K
    e2e = None
    if not args.no_e2e:  # the step's inputs from pinned host memory, the partials back
        host = [t.cpu().pin_memory() for t in sets[0]]
        p_host = torch.empty(8, dtype=torch.float64).pin_memory()
        Ke = min(K, 10)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s_main)
        with torch.cuda.stream(s_main):
            for i in range(Ke):
                for dst, src in zip(sets[0], host):
                    dst.copy_(src, non_blocking=True)
                step(0)
                p_host.copy_(out["partials"], non_blocking=True)
        a1.record(s_main)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(a0.elapsed_time(a1), world) / Ke
        e2e = {"value": world * M / (e2e_ms * 1e-3), "unit": "trajectory-steps/s",
               "h2d_bytes_per_step": sum(t.numel() * t.element_size() for t in host),
               "d2h_bytes_per_step": 64, "ms_per_step": e2e_ms}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import numpy as np
        import oracle
        from oracle import output_layer_oracle as ol
        cols = 64
        h, mu, act, disc, rew, boot = sets[0]
        inp = dict(T=T, B=cols, A=A, dtype=oracle.DTYPE_F32,
                   target_logits=np.zeros((T, cols, A), np.float32),
                   behaviour_logits=mu[:, :cols].cpu().numpy(),
                   actions=act[:, :cols].cpu().numpy(), rewards=rew[:, :cols].cpu().numpy(),
                   values=np.zeros((T, cols), np.float32),
                   bootstrap_value=boot[:cols].cpu().numpy(),
                   discounts=disc[:, :cols].cpu().numpy())
        hh = h[:, :cols].float().cpu().numpy().astype(np.float64)
        Wn = w.float().cpu().numpy().astype(np.float64).T
        bn = bias.cpu().numpy().astype(np.float64)
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < min(args.cpu_seconds, 5.0) or reps == 0:
            ol.loss_and_grad_from_hidden(inp, hh, Wn, bn, baseline_cost=0.5, entropy_cost=0.01)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        cpu = {"value": T * cols / dt, "unit": "trajectory-steps/s",
               "cores": torch.get_num_threads(), "kind": "oracle",
               "sample": f"{reps} x oracle.output_layer_oracle.loss_and_grad_from_hidden on "
                         f"trajectories [0, {cols}) x T={T}"}
    if rank != 0:
        return
    peak, peak_src = load_peak()
    # algorithmic bytes per call: h read + dh write (bf16), behaviour logits (fp32), a, r,
    # gamma, bootstrap, W^T, bias; grad_w_t, grad_bias, partials
    alg = (2 * M * H * 2 + M * A * 4 + 3 * M * 4 + B * 4 + (A + 1) * H * 2 + (A + 1) * 4
           + (A + 1) * H * 4 + (A + 1) * 4 + 64)
    # the same work unfused: the head forward writes z^pi, V (fp32), the path reads them
    # back with the behaviour logits and writes dz, dV, the backward reads dZ and h again
    unfused = (M * H * 2 + M * (A + 1) * 4                      # head forward
               + M * (A + 1) * 4 + M * A * 4 + 3 * M * 4 + M * (A + 1) * 4  # V-trace path
               + M * (A + 1) * 4 + M * H * 2 + M * H * 2)          # dh, dW (reads dZ, h)
    achieved = alg / (step_ms * 1e-3) / 1e9
    line = {
        "metric": "fused head + V-trace + loss + grad + head backward trajectory-steps/s",
        "value": world * M / (step_ms * 1e-3), "unit": "trajectory-steps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16 h, W; f32 accumulate (tcgen05); f32 path; bf16 hi+lo dZ backward",
        "path": "head_fused",
        "data": "synthetic (seeded N(0,1) hidden, N(0,0.01) weights, behaviour = z + N(0,0.3^2))",
        "config": {"workload": "head + path at large: T=100 B=8192 H=256 A=18",
                   "parallelism": f"dp{world}", "collective": "none",
                   "l2": "h (419 MB per copy, 2 copies alternated) exceeds L2", "timing": "eager",
                   "fused_bytes_per_call": alg, "unfused_bytes_per_call": unfused},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": load_traffic("head_fused:large"),
                     "kernel": "head_fused_kernel",
                     "kernel_ms": step_ms, "algorithmic_bytes_per_launch": alg,
                     "peak_source": peak_src},
        "gpu_launches": K,
        "clocks": sampler.summary(tw0, tw1) if sampler else None,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """--gpus N without a launcher: start the N ranks with torch.distributed.run on
    127.0.0.1 (one process per GPU) and return their exit status."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    a = parse()
    _world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        if torch.cuda.device_count() < a.gpus:
            print(f"bench.py: --gpus {a.gpus} but only {torch.cuda.device_count()} CUDA devices",
                  file=sys.stderr)
            sys.exit(2)
        sys.exit(spawn_ranks(a))
    if _world != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={_world}", file=sys.stderr)
        sys.exit(2)
    if os.environ.get("VT_BENCH_WATCHDOG"):  # diagnostics: every thread's stack, then exit
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["VT_BENCH_WATCHDOG"]), exit=True)
    try:
        if a.path == "head_fused":
            if a.impl == "reference":
                print(json.dumps({"impl": "reference", "path": "head_fused", "unavailable":
                                  "the fused head's CPU baseline is in the ours line"}))
            else:
                run_head_fused(a)
        elif a.path == "head":
            if a.impl == "reference":
                print(json.dumps({"impl": "reference", "path": "head", "unavailable":
                                  "the head path's CPU baseline is in the ours line"}))
            else:
                run_head(a)
        elif a.path == "update":
            if a.impl == "reference":
                print(json.dumps({"impl": "reference", "path": "update", "unavailable":
                                  "the update path's CPU baseline is in the ours line"}))
            else:
                run_update(a)
        elif a.impl == "reference":
            run_reference(a)
        else:
            run_ours(a)
    except BaseException:  # noqa: BLE001
        # a failed rank must not hang in NCCL teardown (the others would wait for it):
        # report and leave at once with a non-zero status
        import traceback
        traceback.print_exc()
        sys.stderr.flush()
        sys.stdout.flush()
        os._exit(1)
    import torch.distributed as _dist
    if _dist.is_available() and _dist.is_initialized():
        _dist.destroy_process_group()
