"""Data-parallel learner step (the paper's synchronous learners).

Each rank (one process per GPU) owns a contiguous block of trajectories (columns
of the [T, B] batch) and runs the fused V-trace + loss + gradient kernel on it
with no data-path collective: trajectories are independent through every step of
Section 4.  The one exchange is the sum of the 8 fp64 partials (losses and
gradient-norm sums; the losses add over learners because the loss is summed over
the batch), all-reduced over the process group.

:class:`LearnerStep` is the product API of that step on a GPU: the kernel on a
main stream, step k's 64-byte partials all-reduce on a side stream so that it runs
under step k+1's kernel (nothing on the path consumes the reduced scalars), the
kernel launched as a programmatic dependent of the previous step
(``overlap_previous``: a step's inputs are a fresh trajectory batch), an SM left
free for the collective, and CUDA-graph capture of a sequence of steps.  The
functions below it are backend-agnostic (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch


def shard_columns(B: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Column block [b0, b1) of rank `rank`: equal blocks of whole `align`-column units
    (the first ranks get one extra unit when they do not divide evenly).  align = 8
    keeps every shard on the column-block kernel's 16-byte TMA segments."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if align < 1 or B % align:
        raise ValueError("B must be a multiple of align")
    units = B // align
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    return u0 * align, (u0 + base + (1 if rank < extra else 0)) * align


def allreduce_partials(partials: torch.Tensor, group=None, async_op: bool = False):
    """SUM all-reduce of the [8] fp64 partials in place.  Every entry is a sum
    over trajectories (the total loss is linear in the others), so the shard
    sums add up to the global batch's partials."""
    import torch.distributed as dist
    if partials.dtype != torch.float64 or partials.numel() != 8:
        raise ValueError("partials must be a float64 tensor of 8 entries")
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def max_over_ranks(x: float, device="cpu", group=None) -> float:
    """Max of a host float over ranks (the slowest rank's time)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gradient_norm(partials: torch.Tensor) -> float:
    """sqrt(sum dL/dz^2 + sum dL/dV^2) of the (reduced) partials (reading c17)."""
    p = partials.detach().to("cpu", torch.float64)
    return float(torch.sqrt(p[4] + p[5]))


def allreduce_grads(grads: torch.Tensor, group=None, async_op: bool = False):
    """SUM all-reduce, in place, of a learner's parameter gradient before the
    update: the loss is summed over the batch, so the
    whole batch's gradient is the sum of the learners' shard gradients (reading
    r11); every learner then runs the same vtrace_rmsprop_step on its replica
    (synchronous update).  NCCL on GPUs, gloo in the CPU tests."""
    import torch.distributed as dist
    if not grads.is_floating_point():
        raise ValueError("grads must be a floating-point tensor")
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def _world(group=None) -> tuple[int, int]:
    import torch.distributed as dist
    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


class LearnerStep:
    """One learner's step on its trajectory shard: the fused kernel, then the
    partials all-reduce (row a13) overlapped with the next step.

    ``kernel`` computes one shard: ``kernel(inputs, out, **kw)`` with the seven
    input tensors in ``inputs`` and the outputs (grad_target_logits, grad_values,
    partials) in ``out``; the default is :func:`vtrace.loss_and_grad` on the GPU
    (the CPU tests pass the oracle).  On a CUDA device the kernel runs on
    ``self.stream`` and the collective on ``self.comm_stream``; call :meth:`join`
    (or synchronise) before reading a reduced ``partials``.

    overlap:      launch each step's kernel as a programmatic dependent of the
                  previous one (its prologue overlaps the previous step's tail;
                  valid because every step reads a fresh batch, never the
                  previous step's outputs).
    reserve_sms:  SMs the kernel leaves free at N > 1 so that step k's collective
                  is not queued behind step k+1's CTAs (default 1).
    collective:   how the partials are summed over the learners at N > 1 on GPUs:
                  "nvlink" (default) -- vtrace_partials_allreduce, one 32-thread kernel
                  that exchanges the 64 bytes through peer-mapped mailboxes in
                  symmetric memory; "fused" -- inside the V-trace kernel's last CTA
                  (vtrace_loss_and_grad_learners); "nccl" -- torch.distributed.all_reduce.
    exchange_every: with "nvlink" and > 1, exchange the partials of this many steps
                  together in one side-stream kernel (vtrace_partials_allreduce_batched;
                  each step's sums are still produced, in place, once its batch is
                  exchanged; join() exchanges a partial batch).
    A step's kernel never overwrites a partials buffer whose previous collective is
    still pending: it waits for that collective's event (with buffers rotated over R
    sets, the collective of R steps ago).
    """

    def __init__(self, T: int, B: int, A: int, logits_dtype, *, device=None, group=None,
                 overlap: bool = True, reserve_sms: int | None = None,
                 kernel: Callable | None = None, collective: str = "nvlink",
                 guard_partials: bool = True, exchange_every: int = 1, **method_kw):
        self.T, self.B, self.A = int(T), int(B), int(A)
        self.group = group
        self.world, self.rank = _world(group)
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        self.cuda = self.device.type == "cuda"
        self.kw = dict(method_kw)
        if kernel is None:
            from . import vtrace
            code = logits_dtype if isinstance(logits_dtype, int) else {
                torch.float32: vtrace.VT_FLOAT32, torch.bfloat16: vtrace.VT_BFLOAT16}[logits_dtype]
            self.workspace = vtrace.Workspace(T, B, A, code, self.device)
            self._kernel = vtrace.loss_and_grad
            reserve = (1 if self.world > 1 else 0) if reserve_sms is None else int(reserve_sms)
            sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            self.kw.update(workspace=self.workspace, overlap_previous=bool(overlap),
                           sm_budget=(sms - reserve) if reserve > 0 else 0)
        else:
            self.workspace = None
            self._kernel = kernel
        if self.cuda:
            self.stream = torch.cuda.Stream(self.device)
            self.comm_stream = torch.cuda.Stream(self.device)
        else:
            self.stream = self.comm_stream = None
        if collective not in ("nvlink", "nccl", "fused", "off"):
            raise ValueError("collective must be 'nvlink', 'fused', 'nccl' (or 'off': A/B only, "
                             "no exchange)")
        self.collective = collective if (self.cuda and self.world > 1) else "none"
        if self.collective == "fused" and kernel is not None:
            raise ValueError("collective='fused' runs the library kernel")
        if self.collective == "fused":
            from . import vtrace
            if not vtrace.kernel_for(T, B, A, self.workspace_dtype(logits_dtype)).startswith(
                    "vtrace_cb_kernel"):
                self.collective = "nvlink"  # (the in-kernel exchange is column-block only)
        self._pending: dict = {}  # partials data_ptr -> event after its collective
        self.guard_partials = bool(guard_partials)
        self.exchange_every = int(exchange_every)
        if not 1 <= self.exchange_every <= 32:
            raise ValueError("exchange_every must be in 1..32")
        if self.exchange_every > 1 and self.collective == "nccl":
            raise ValueError("exchange_every > 1 needs collective='nvlink'")
        self._batch: list = []  # (key, partials) of the steps not exchanged yet
        self._batch_id = 0      # batches exchanged so far (side stream, in order)
        self._waited = 0        # the last batch the step's stream has waited for
        self.collective_fallback = None
        if self.collective in ("nvlink", "fused"):
            try:
                self._setup_mailboxes()
            except Exception as e:  # noqa: BLE001 -- no peer-mapped memory: NCCL, stated
                # (symmetric memory failing is a property of the node, the same on every rank)
                self.collective_fallback = f"{type(e).__name__}: {e}"[:200]
                self.collective, self.exchange_every = "nccl", 1
        if self.collective == "fused":
            self.kw.update(mailboxes=self._mbox_ptrs, self_index=self.rank)

    @staticmethod
    def workspace_dtype(logits_dtype):
        from . import vtrace
        if isinstance(logits_dtype, int):
            return logits_dtype
        return {torch.float32: vtrace.VT_FLOAT32, torch.bfloat16: vtrace.VT_BFLOAT16}[logits_dtype]

    def _setup_mailboxes(self):
        """Every learner's mailbox in symmetric memory (peer-mapped over NVLink)."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        from . import vtrace
        nbytes = (vtrace.partials_mailbox_bytes(self.world) if self.exchange_every == 1 else
                  vtrace.partials_mailbox_bytes_batched(self.world, self.exchange_every))
        if nbytes <= 0:
            raise ValueError(f"collective='nvlink' supports up to 16 learners, not {self.world}")
        with torch.cuda.device(self.device):
            self._mbox = symm_mem.empty(nbytes // 8, dtype=torch.float64, device=self.device)
            self._mbox.zero_()
            name = (self.group or dist.group.WORLD).group_name
            hdl = symm_mem.rendezvous(self._mbox, name)
            self._mbox_ptrs = [int(p) for p in hdl.buffer_ptrs]
            self._counter = torch.zeros(1, dtype=torch.int64, device=self.device)
            torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)

    def _launch(self, inputs: dict, out: dict):
        from .vtrace import INPUT_NAMES
        self._kernel(*[inputs[k] for k in INPUT_NAMES], out=out, **self.kw)

    def __call__(self, inputs: dict, out: dict):
        """Enqueue one step: the shard's kernel, then (N > 1) the SUM all-reduce of
        out['partials'] over the group."""
        if not self.cuda:
            self._launch(inputs, out)
            allreduce_partials(out["partials"], self.group)
            return
        key = out["partials"].data_ptr()
        if any(k == key for k, _ in self._batch):  # (reused before its exchange: flush first)
            self._flush()
        if self.collective == "nvlink" and self.exchange_every > 1 and self.world > 1:
            # batched exchange on the side stream; a kernel waits only for the first batch
            # not yet waited for that last read its buffer (batches finish in order on the
            # side stream, so one wait covers every earlier batch): in a captured graph only
            # one kernel in exchange_every has a cross-stream edge in and one an edge out
            pend = self._pending.pop(key, None)
            if pend is not None and self.guard_partials and pend[0] > self._waited:
                self.stream.wait_event(pend[1])
                self._waited = pend[0]
            with torch.cuda.stream(self.stream):
                self._launch(inputs, out)
            self._batch.append((key, out["partials"]))
            if len(self._batch) == self.exchange_every:
                self._flush()
            return
        ev = self._pending.pop(key, None)
        if ev is not None and self.guard_partials:  # its previous collective must have read it
            self.stream.wait_event(ev)
        with torch.cuda.stream(self.stream):
            self._launch(inputs, out)
        if self.world > 1 and self.collective not in ("fused", "off"):
            self.comm_stream.wait_stream(self.stream)
            with torch.cuda.stream(self.comm_stream):
                if self.collective == "nvlink":
                    from . import vtrace
                    vtrace.partials_allreduce(out["partials"], self._mbox_ptrs, self.rank,
                                              self._counter)
                else:
                    allreduce_partials(out["partials"], self.group)
                ev = torch.cuda.Event()
                ev.record(self.comm_stream)
            self._pending[key] = ev

    def _flush(self):
        """Exchange the batched steps' partials: one kernel on the side stream after the
        batch's last kernel."""
        if not self._batch:
            return
        from . import vtrace
        self.comm_stream.wait_stream(self.stream)
        with torch.cuda.stream(self.comm_stream):
            vtrace.partials_allreduce_batched([p for _, p in self._batch], self._mbox_ptrs,
                                              self.rank, self._counter,
                                              batch_max=self.exchange_every)
            ev = torch.cuda.Event()
            ev.record(self.comm_stream)
        self._batch_id += 1
        for k, _ in self._batch:
            self._pending[k] = (self._batch_id, ev)
        self._batch = []

    def join(self):
        """The main stream waits for the outstanding collectives (a partial batch is
        exchanged first: every learner joins at the same points)."""
        if self.cuda and self.world > 1:
            self._flush()
            self.stream.wait_stream(self.comm_stream)
            self._pending.clear()
            self._waited = self._batch_id

    def run(self, batches: Sequence[tuple[dict, dict]]):
        """Enqueue the steps over (inputs, out) pairs, then join."""
        for inputs, out in batches:
            self(inputs, out)
        self.join()

    def capture(self, batches: Sequence[tuple[dict, dict]]) -> "torch.cuda.CUDAGraph":
        """A CUDA graph of the step sequence (kernels, cross-stream events and the
        NCCL collectives), joined at the end; replay with ``g.replay()`` on any
        stream (it runs in the graph's own stream order)."""
        if not self.cuda:
            raise RuntimeError("graph capture needs a CUDA device")
        g = torch.cuda.CUDAGraph()
        self.join()  # no event of an eager step may be waited on inside the capture
        with torch.cuda.graph(g, stream=self.stream):
            self.run(batches)  # (ends with join: no captured event leaks out)
        return g
