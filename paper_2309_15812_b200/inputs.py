"""Seeded synthetic inputs shared by the tests, bench.py and smoke().

This module is the ONLY code shared between the CUDA path and the oracle
(`oracle/`).  It holds none of the method's arithmetic: it produces random
numbers and the workload shapes named in BASELINE.json / SURVEY.md §8(d).1.

Generator: SplitMix64 ("SplitMix64-derived 64-bit stream mapped to the
unit interval"), element i (0-based) is mix(seed + (i+1)·0x9E3779B97F4A7C15),
mapped to U[-1, 1) with 53 random bits, then rounded to the activation dtype.
Recipe: x seed 0 U[-1,1); w seed 1 U[-1,1)/sqrt(K); dy seed 2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """n outputs of SplitMix64 seeded with `seed` (uint64 array)."""
    with np.errstate(over="ignore"):
        idx = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(shape, seed: int) -> np.ndarray:
    """float64 array, U[-1, 1), 53-bit resolution."""
    n = int(np.prod(shape)) if len(shape) else 1
    z = splitmix64(seed, n)
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return (2.0 * u - 1.0).reshape(shape)


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even); returns
    float32 values that are exactly representable in bf16."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


def round_to_f16(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).astype(np.float16).astype(np.float32)


def activation(shape, seed: int, dtype: str = "f32") -> np.ndarray:
    """Activations (x or dy) as float32 values exactly representable in `dtype`."""
    a = uniform_pm1(shape, seed).astype(np.float32)
    if dtype == "f32":
        return a
    if dtype == "bf16":
        return round_to_bf16(a)
    if dtype == "f16":
        return round_to_f16(a)
    raise ValueError(dtype)


def weights(C: int, K: int, seed: int = 1) -> np.ndarray:
    """fp32 weights laid out [C][K] (k fastest), U[-1,1)/sqrt(K)."""
    return (uniform_pm1((C, K), seed) / math.sqrt(K)).astype(np.float32)


@dataclass(frozen=True)
class Workload:
    """Shape recipe of one BASELINE.json config."""
    name: str
    N: int
    C: int
    H: int
    W: int
    K: int
    D: int
    assign: str  # "cycled" (BASELINE) or "contiguous" (paper P:1271)
    stride: int = 1

    @property
    def pad(self) -> int:
        return self.K // 2


# configs[0]: tiny oracle check (BASELINE.json configs[0]); angles {0,45,90,135} = D=4
TINY = Workload("tiny", 1, 8, 14, 14, 7, 4, "cycled")
# configs[1]: ConvNeXt-T-1D stage-1 layer, 8 angles cycled over channels
S1 = Workload("convnext_t_1d_stage1", 64, 96, 56, 56, 31, 8, "cycled")


def ksweep(K: int) -> Workload:
    """configs[2]: kernel-length sweep at C=384, 14x14, N=128."""
    return Workload(f"ksweep_k{K}", 128, 384, 14, 14, K, 8, "cycled")


# the 1D++ block of ConvNeXt1D++ (P:1469-1483): the block's main oriented
# conv shrinks to K=15, and a residual depthwise oriented 1x31 conv is inserted on the
# 4C-expanded inverted bottleneck (C = 4 x 96 = 384 at stage 1 of the T model).
PP_MAIN = Workload("convnext_t_1dpp_stage1_main", 64, 96, 56, 56, 15, 8, "cycled")
PP_RES = Workload("convnext_t_1dpp_stage1_residual", 64, 384, 56, 56, 31, 8, "cycled")

WORKLOADS = {"s1": S1, "pp_main": PP_MAIN, "pp_res": PP_RES}
