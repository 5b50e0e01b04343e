"""Batch-sharded data parallelism for the oriented 1D depthwise conv layer
(SURVEY.md §8(e), row a8).

One process per GPU.  Rank r owns samples [r*N/g, (r+1)*N/g) of the global
batch.  forward and backward_input are per-sample, so they need no
communication.  backward_weight yields a local partial dW[C][K] (fp32) per
rank; the only collective of the path is one all-reduce (sum) of dW over the
process group (NCCL over NVLink/NVSwitch on B200).  torch.distributed is the
plumbing; the compute runs in liboriented1d.
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
    """Sum the per-rank partial dW over the group, in place (row a8)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(dW, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def dp_layer_step(x_shard: torch.Tensor, w: torch.Tensor, dy_shard: torch.Tensor,
                  forward: Callable, backward_input: Callable, backward_weight: Callable,
                  group: Optional[dist.ProcessGroup] = None):
    """One data-parallel training step of the layer on this rank's shard:
    y = forward(x), dx = backward_input(dy), dW = allreduce(backward_weight(x, dy)).
    The three callables are the library passes (binding.forward etc., partially
    applied to a plan); returns (y, dx, dW) where dW is the global-batch gradient."""
    y = forward(x_shard, w)
    dx = backward_input(dy_shard, w)
    dW = backward_weight(x_shard, dy_shard)
    allreduce_weight_grad(dW, group)
    return y, dx, dW
