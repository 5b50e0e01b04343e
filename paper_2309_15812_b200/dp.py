"""Batch-sharded data parallelism for the oriented 1D depthwise conv layer
(SURVEY.md §8(e), row a8).

One process per GPU.  Rank r owns samples [r*N/g, (r+1)*N/g) of the global batch.
forward and backward_input are per-sample, so they need no communication.
backward_weight yields a local partial dW[C][K] (fp32) per rank; the only
collective of the path is one all-reduce (sum) of dW over the process group
(NCCL over NVLink/NVSwitch on B200; gloo in the CPU / single-GPU tests).

`DPLayerStep` runs one layer training step on the rank's shard through
liboriented1d and overlaps the dW all-reduce with backward_input: backward_weight
goes first, its dW is handed to the collective asynchronously (NCCL runs it on its
own stream), and backward_input runs on the compute stream while the reduction is
in flight.  torch.distributed is the plumbing; every pass runs in liboriented1d.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_range(N: int, world: int, rank: int):
    """Contiguous, balanced shard [lo, hi) of N samples for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(N, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def allreduce_weight_grad(dW: torch.Tensor, group: Optional[dist.ProcessGroup] = None,
                          async_op: bool = False):
    """Sum the per-rank partial dW over the group, in place (row a8).  Returns the work
    handle for async_op=True (None when there is nothing to reduce)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(dW, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def dp_layer_step(x_shard: torch.Tensor, w: torch.Tensor, dy_shard: torch.Tensor,
                  forward: Callable, backward_input: Callable, backward_weight: Callable,
                  group: Optional[dist.ProcessGroup] = None):
    """One data-parallel training step of the layer on this rank's shard with arbitrary
    pass callables (used by the CPU tests): y = forward(x), dW = allreduce(backward_weight
    (x, dy)) overlapped with dx = backward_input(dy).  Returns (y, dx, dW); dW is the
    global-batch gradient."""
    y = forward(x_shard, w)
    dW = backward_weight(x_shard, dy_shard)
    work = allreduce_weight_grad(dW, group, async_op=True)
    dx = backward_input(dy_shard, w)
    if work is not None:
        work.wait()
    return y, dx, dW


class DPLayerStep:
    """Data-parallel layer step through liboriented1d for one rank.

    plan: a binding.Plan for this rank's shard (N = shard size).  __call__(x, w, dy)
    returns (y, dx, dW) with dW summed over the group.  With fused=True the backward
    runs as one o1d_backward pass (x and dy read once, NEXT-2) and the all-reduce
    follows it; otherwise backward_weight runs first and its all-reduce overlaps
    backward_input.  Buffers are allocated once and reused."""

    def __init__(self, plan, group: Optional[dist.ProcessGroup] = None, fused: bool = False):
        from . import binding as B
        self.B = B
        self.plan = plan
        self.group = group
        self.fused = fused
        dev = plan.device
        self.y = torch.empty(plan.y_shape(), dtype=plan.dtype, device=dev)
        self.dx = torch.empty(plan.x_shape(), dtype=plan.dtype, device=dev)
        self.dW = torch.empty((plan.C, plan.K), dtype=torch.float32, device=dev)
        self.ws = B.workspace(plan)

    def __call__(self, x: torch.Tensor, w: torch.Tensor, dy: torch.Tensor):
        B = self.B
        B.forward(self.plan, x, w, self.y)
        if self.fused:
            B.backward(self.plan, x, dy, w, self.dx, self.dW, self.ws)
            allreduce_weight_grad(self.dW, self.group)
            return self.y, self.dx, self.dW
        B.backward_weight(self.plan, x, dy, self.dW, self.ws)
        work = allreduce_weight_grad(self.dW, self.group, async_op=True)
        B.backward_input(self.plan, dy, w, self.dx)
        if work is not None:
            work.wait()
        return self.y, self.dx, self.dW
