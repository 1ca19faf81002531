"""Data-parallel learner plumbing (the paper's synchronous learners).

Each rank (one process per GPU) owns a contiguous block of trajectories
(columns of the [T, B] batch) and runs the fused kernel on it with no
data-path collective; the one exchange is the sum of the 8 fp64 partials
(losses and gradient-norm sums), all-reduced over the process group.  The
functions here are backend-agnostic (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import torch


def shard_columns(B: int, world: int, rank: int) -> tuple[int, int]:
    """Column block [b0, b1) of rank `rank`: equal blocks, the first B % world
    ranks get one extra column."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(B, world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


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
    """Max of a host float over ranks (used for the slowest rank's time)."""
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
