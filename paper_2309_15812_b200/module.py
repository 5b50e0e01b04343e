"""PyTorch operators, autograd and nn.Module over the C ABI (the paper's
"plug-and-play PyTorch module").  Marshalling only: every pass runs in
liboriented1d.

* `torch.library` custom ops `o1d::forward`, `o1d::backward_input`,
  `o1d::backward_weight` with fake (meta) implementations, so the op is visible to
  torch.compile / FakeTensor tracing and passes `torch.library.opcheck`.  A plan is an
  immutable host object, so the ops take an integer plan id (`register_plan`).
* `o1d::forward` has an autograd formula: dx = backward_input(dy), dW =
  backward_weight(x, dy) -- or, for plans created with O1D_FUSED=1, the fused
  single-pass backward (o1d_backward, NEXT-2) behind one `o1d::backward` op.
* `Oriented1dDWConv`: the nn.Module (C channels, K taps, D directions).
"""
from __future__ import annotations

import itertools
import math
import threading
import weakref
from collections import OrderedDict

import numpy as np
import torch

from . import binding as B

# plan id -> Plan, weakly: a plan lives while its owner (a module's plan cache, an autograd
# graph that saved it, the caller) holds it
_PLANS = weakref.WeakValueDictionary()
_ids = itertools.count(1)
_lock = threading.Lock()


def register_plan(plan: B.Plan) -> int:
    """Make `plan` addressable by the custom ops; returns its id (the caller keeps the plan
    alive; the registry holds a weak reference)."""
    with _lock:
        pid = getattr(plan, "_op_id", None)
        if pid is None:
            pid = next(_ids)
            plan._op_id = pid
        _PLANS[pid] = plan
    return pid


def unregister_plan(pid: int) -> None:
    with _lock:
        _PLANS.pop(pid, None)


def _plan(pid: int) -> B.Plan:
    p = _PLANS.get(pid)
    if p is None:
        raise KeyError(f"o1d plan id {pid} is not registered")
    return p


@torch.library.custom_op("o1d::forward", mutates_args=())
def forward_op(x: torch.Tensor, w: torch.Tensor, plan_id: int) -> torch.Tensor:
    """y = Def. 1 of x with fp32 weights w [C][K]."""
    return B.forward(_plan(plan_id), x, w)


@forward_op.register_fake
def _(x, w, plan_id):
    p = _plan(plan_id)
    return x.new_empty(p.y_shape())


@torch.library.custom_op("o1d::backward_input", mutates_args=())
def backward_input_op(dy: torch.Tensor, w: torch.Tensor, plan_id: int) -> torch.Tensor:
    return B.backward_input(_plan(plan_id), dy, w)


@backward_input_op.register_fake
def _(dy, w, plan_id):
    p = _plan(plan_id)
    return dy.new_empty(p.x_shape())


@torch.library.custom_op("o1d::backward_weight", mutates_args=())
def backward_weight_op(x: torch.Tensor, dy: torch.Tensor, plan_id: int) -> torch.Tensor:
    return B.backward_weight(_plan(plan_id), x, dy)


@backward_weight_op.register_fake
def _(x, dy, plan_id):
    p = _plan(plan_id)
    return x.new_empty((p.C, p.K), dtype=torch.float32)


@torch.library.custom_op("o1d::backward", mutates_args=())
def backward_op(x: torch.Tensor, dy: torch.Tensor, w: torch.Tensor, plan_id: int) -> tuple[torch.Tensor, torch.Tensor]:
    """(dx, dW) from one pass over x and dy (o1d_backward)."""
    return B.backward(_plan(plan_id), x, dy, w)


@backward_op.register_fake
def _(x, dy, w, plan_id):
    p = _plan(plan_id)
    return x.new_empty(p.x_shape()), x.new_empty((p.C, p.K), dtype=torch.float32)


def _setup_context(ctx, inputs, output):
    x, w, plan_id = inputs
    ctx.save_for_backward(x, w)
    ctx.plan_id = plan_id
    ctx.plan = _plan(plan_id)  # keeps the plan alive until the backward ran


def _backward(ctx, dy):
    x, w = ctx.saved_tensors
    # The gradient arriving from autograd may be a non-contiguous view; the library takes
    # NCHW-contiguous buffers only (binding: no silent copies), so the copy is made here,
    # explicitly, at the autograd boundary -- never inside the library.
    if not dy.is_contiguous():
        dy = dy.contiguous()
    need_x, need_w = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
    if need_x and need_w and ctx.plan.fused_step:
        dx, dW = backward_op(x, dy, w, ctx.plan_id)
        return dx, dW, None
    dx = backward_input_op(dy, w, ctx.plan_id) if need_x else None
    dW = backward_weight_op(x, dy, ctx.plan_id) if need_w else None
    return dx, dW, None


forward_op.register_autograd(_backward, setup_context=_setup_context)


def oriented1d_dwconv(x: torch.Tensor, w: torch.Tensor, plan: B.Plan) -> torch.Tensor:
    return forward_op(x, w, register_plan(plan))


class Oriented1dDWConv(torch.nn.Module):
    """Depthwise convolution of oriented 1D kernels (Def. 1).

    C channels, kernel length K, D directions assigned "contiguous"
    (paper) or "cycled"; `shift_deg` = layer-wise rotation;
    `discretization` = "rotation" (Def. 1), "shear" (Appendix) or
    "bilinear".  Weights are fp32 [C][K]; activations NCHW-contiguous
    fp32/bf16/fp16.  Plans are cached per input shape in a bounded LRU (`max_plans`);
    plans that differ only in the batch size share their compiled kernels (the
    library's module cache), so a ragged last batch costs a plan, not a compile."""

    def __init__(self, C: int, K: int, D: int = 8, stride: int = 1, assign: str = "contiguous",
                 shift_deg: float = 0.0, angles_deg=None, discretization: str = "rotation", max_plans: int = 8):
        super().__init__()
        self.C, self.K, self.stride = C, K, stride
        self.discretization = discretization
        if angles_deg is None:
            angles_deg = B.direction_angles(D, C, assign, shift_deg)
        # kept as float64 numpy (not a buffer: Module.to(dtype) must not round the angles)
        self.angles_deg = np.asarray(angles_deg, dtype=np.float64).copy()
        self.weight = torch.nn.Parameter(torch.empty(C, K))
        torch.nn.init.uniform_(self.weight, -1.0 / math.sqrt(K), 1.0 / math.sqrt(K))
        self._plans: OrderedDict = OrderedDict()
        self.max_plans = max_plans

    def plan_for(self, x: torch.Tensor) -> B.Plan:
        N, C, H, W = x.shape
        key = (N, H, W, x.dtype, x.device)
        p = self._plans.get(key)
        if p is None:
            p = B.Plan(N, C, H, W, self.K, self.angles_deg, stride=self.stride, dtype=x.dtype,
                       device=x.device, discretization=self.discretization)
            self._plans[key] = p
            while len(self._plans) > self.max_plans:
                self._plans.popitem(last=False)  # freed once no autograd graph holds it
        else:
            self._plans.move_to_end(key)
        return p

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return oriented1d_dwconv(x, self.weight, self.plan_for(x))
