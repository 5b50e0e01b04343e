"""PyTorch autograd + nn.Module over the C ABI (the paper's "plug-and-play PyTorch
module").  Marshalling only: the three passes run in liboriented1d."""
from __future__ import annotations

import math

import numpy as np
import torch

from . import binding as B


class _Oriented1dFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, plan):
        ctx.plan = plan
        ctx.save_for_backward(x, w)
        return B.forward(plan, x, w)

    @staticmethod
    def backward(ctx, dy):
        x, w = ctx.saved_tensors
        plan = ctx.plan
        dy = dy.contiguous()
        dx = B.backward_input(plan, dy, w) if ctx.needs_input_grad[0] else None
        dW = B.backward_weight(plan, x, dy) if ctx.needs_input_grad[1] else None
        return dx, dW, None


def oriented1d_dwconv(x: torch.Tensor, w: torch.Tensor, plan: B.Plan) -> torch.Tensor:
    return _Oriented1dFn.apply(x, w, plan)


class Oriented1dDWConv(torch.nn.Module):
    """Depthwise convolution of oriented 1D kernels (Def. 1).

    C channels, kernel length K, D directions assigned "contiguous"
    (paper) or "cycled"; `shift_deg` = layer-wise rotation;
    `discretization` = "rotation" (Def. 1) or "shear" (Appendix).  Weights
    are fp32 [C][K]; activations NCHW-contiguous fp32/bf16/fp16."""

    def __init__(self, C: int, K: int, D: int = 8, stride: int = 1, assign: str = "contiguous",
                 shift_deg: float = 0.0, angles_deg=None, discretization: str = "rotation"):
        super().__init__()
        self.C, self.K, self.stride = C, K, stride
        self.discretization = discretization
        if angles_deg is None:
            angles_deg = B.direction_angles(D, C, assign, shift_deg)
        # kept as float64 numpy (not a buffer: Module.to(dtype) must not round the angles)
        self.angles_deg = np.asarray(angles_deg, dtype=np.float64).copy()
        self.weight = torch.nn.Parameter(torch.empty(C, K))
        torch.nn.init.uniform_(self.weight, -1.0 / math.sqrt(K), 1.0 / math.sqrt(K))
        self._plans = {}

    def plan_for(self, x: torch.Tensor) -> B.Plan:
        N, C, H, W = x.shape
        key = (N, H, W, x.dtype, x.device)
        p = self._plans.get(key)
        if p is None:
            p = B.Plan(N, C, H, W, self.K, self.angles_deg, stride=self.stride, dtype=x.dtype,
                       device=x.device, discretization=self.discretization)
            self._plans[key] = p
        return p

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return oriented1d_dwconv(x, self.weight, self.plan_for(x))
