"""ConvNeXt-1D measurement harness (SURVEY.md §8(d).1 workloads T-full / B-DP).

Not a model zoo: a synthetic-data training step that puts the oriented 1D
depthwise layer (liboriented1d through `module.Oriented1dDWConv`) inside the
network it was designed for, so the model-level throughput (images/s) of the
BASELINE metric can be measured.  Everything except the oriented depthwise
convolutions is stock PyTorch (cuBLAS GEMMs for the pointwise layers).

Architecture (PAPER.md "Model Instantiation"):
  * ConvNeXt-T-1D: C = (96, 192, 384, 768), B = (3, 3, 9, 3) (Table model_size);
    ConvNeXt-B-1D: C = (128, 256, 512, 1024), B = (3, 3, 27, 3).
  * 1D Block = oriented dw 1xK -> LN -> pw 4C -> GELU -> pw C -> layer scale -> residual
    (ConvNeXt block with the 7x7 dw replaced).
  * K per stage [31, 31, 27, 15], D = 8 directions, layer-wise
    rotation +90 deg on alternate layers (reading R11: per block).
  * Depthwise 1D Stem with C0 = 64 (figure only): the layer sequence
    is SPEC's reading: pw(3->C0) -> dw 1x5 s2 (0 deg) -> dw 1x5 (90 deg) ->
    pw -> GELU -> dw 1x5 s2 (90 deg) -> dw 1x5 (0 deg) -> pw(C0->C1) -> LN.
  * Downsampling between stages: LN + 2x2 stride-2 conv (kept from ConvNeXt).
Weights are random (no checkpoints); inputs are synthetic images.
"""
from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F

from .module import Oriented1dDWConv

CONFIGS = {
    "convnext_t_1d": dict(dims=(96, 192, 384, 768), depths=(3, 3, 9, 3)),
    "convnext_b_1d": dict(dims=(128, 256, 512, 1024), depths=(3, 3, 27, 3)),
}
STAGE_K = (31, 31, 27, 15)


def make_dw(C, K, angles=None, D=8, stride=1, shift_deg=0.0, impl="oriented"):
    """The depthwise layer of a block / the stem: the oriented 1D conv (liboriented1d), or -- as
    the comparator of PAPER.md:1027 ("1xK" PyTorch depthwise conv) -- torch's depthwise conv2d
    with a horizontal 1xK kernel of the same length and stride (cuDNN), same surrounding network."""
    if impl == "torch1xk":
        return nn.Conv2d(C, C, (1, K), stride=stride, padding=(0, K // 2), groups=C, bias=False)
    if angles is not None:
        return Oriented1dDWConv(C, K, angles_deg=angles, stride=stride)
    return Oriented1dDWConv(C, K, D=D, assign="contiguous", shift_deg=shift_deg, stride=stride)


class LayerNorm2d(nn.Module):
    """LayerNorm over channels of an NCHW tensor."""

    def __init__(self, C):
        super().__init__()
        self.ln = nn.LayerNorm(C, eps=1e-6)

    def forward(self, x):
        return self.ln(x.permute(0, 2, 3, 1)).permute(0, 3, 1, 2).contiguous()


class Block1D(nn.Module):
    def __init__(self, C, K, D, shift_deg, impl="oriented"):
        super().__init__()
        self.dw = make_dw(C, K, D=D, shift_deg=shift_deg, impl=impl)
        self.norm = nn.LayerNorm(C, eps=1e-6)
        self.pw1 = nn.Linear(C, 4 * C)
        self.pw2 = nn.Linear(4 * C, C)
        self.gamma = nn.Parameter(1e-6 * torch.ones(C))

    def forward(self, x):
        y = self.dw(x).permute(0, 2, 3, 1)
        y = self.pw2(F.gelu(self.pw1(self.norm(y))))
        return x + (self.gamma * y).permute(0, 3, 1, 2).contiguous()


class DepthwiseStem1D(nn.Module):
    def __init__(self, C0, C1, impl="oriented"):
        super().__init__()
        self.pw_in = nn.Conv2d(3, C0, 1)
        self.dw1 = make_dw(C0, 5, angles=[0.0] * C0, stride=2, impl=impl)
        self.dw2 = make_dw(C0, 5, angles=[90.0] * C0, impl=impl)
        self.pw_mid = nn.Conv2d(C0, C0, 1)
        self.dw3 = make_dw(C0, 5, angles=[90.0] * C0, stride=2, impl=impl)
        self.dw4 = make_dw(C0, 5, angles=[0.0] * C0, impl=impl)
        self.pw_out = nn.Conv2d(C0, C1, 1)
        self.norm = LayerNorm2d(C1)

    def forward(self, x):
        x = self.dw2(self.dw1(self.pw_in(x).contiguous()))
        x = F.gelu(self.pw_mid(x)).contiguous()
        x = self.dw4(self.dw3(x))
        return self.norm(self.pw_out(x))


class ConvNeXt1D(nn.Module):
    def __init__(self, name="convnext_t_1d", num_classes=1000, D=8, C0=64, impl="oriented"):
        super().__init__()
        cfg = CONFIGS[name]
        dims, depths = cfg["dims"], cfg["depths"]
        self.stem = DepthwiseStem1D(C0, dims[0], impl=impl)
        self.stages = nn.ModuleList()
        self.downs = nn.ModuleList()
        layer = 0
        for i, (C, n) in enumerate(zip(dims, depths)):
            blocks = []
            for _ in range(n):
                blocks.append(Block1D(C, STAGE_K[i], D, 90.0 if layer % 2 else 0.0, impl=impl))
                layer += 1
            self.stages.append(nn.Sequential(*blocks))
            if i < 3:
                self.downs.append(nn.Sequential(LayerNorm2d(C), nn.Conv2d(C, dims[i + 1], 2, stride=2)))
        self.head_norm = nn.LayerNorm(dims[-1], eps=1e-6)
        self.head = nn.Linear(dims[-1], num_classes)

    def forward(self, x):
        x = self.stem(x)
        for i, st in enumerate(self.stages):
            x = st(x)
            if i < 3:
                x = self.downs[i](x).contiguous()
        return self.head(self.head_norm(x.mean((2, 3))))


def oriented_layers(model: nn.Module):
    return [m for m in model.modules() if isinstance(m, Oriented1dDWConv)]
