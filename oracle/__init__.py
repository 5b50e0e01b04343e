"""CPU oracle of the depthwise oriented 1D convolution (arXiv 2309.15812).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import, call, link or execute anything
under oracle/.  The product path (paper_2309_15812_b200/) never does, and the
two share no code (only the seeded inputs in paper_2309_15812_b200/inputs.py,
which hold none of the method's arithmetic).

Contents
  taps.py    exact tap tables (Def. 1 Eq. coordinate) and the
             direction-group angle assignment
  oracle.c   f64 triple loops: forward, backward_input (adjoint, scatter
             form), backward_weight (adjoint in w); the same three for the bilinear
             discretisation: interpolated samples at the real offsets

Pins (tests/test_oracle_*.py, -m "not gpu"): SPEC worked examples, the paper's
theta=-45/pad=0 example, symbolic (sympy) floors, closed forms at 0/90 deg,
torch f64 conv2d (horizontal, vertical, masked KxK) and its autograd, adjoint
identities, finite differences; bilinear: torch grid_sample (bilinear, zeros,
align_corners) and its autograd, the rotation oracle at the axis angles, partition of
unity.  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from .taps import bilinear_exact, bilinear_table, direction_angles, taps_exact, taps_exact_shear, taps_table  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
# timing-only variant (bench.py cpu_baseline): fp32 accumulators in forward / backward_weight
_LIB_F32ACC = os.path.join(_HERE, "_build", "liboracle_f32acc.so")
_lock = threading.Lock()
_lib = None
_variant = "f64"


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, no fast-math: IEEE f64, order as written); also the
    f32-accumulator timing variant."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    for path, extra in ((_LIB_PATH, []), (_LIB_F32ACC, ["-DORACLE_ACC=float"])):
        if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC):
            tmp = path + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
                                   "-shared", "-fPIC"] + extra + ["-o", tmp, _SRC])
            os.replace(tmp, path)
    return _LIB_PATH


def use_variant(name: str) -> None:
    """"f64" (the oracle; every parity check) or "f32acc" (bench.py timing only)."""
    global _lib, _variant
    if name not in ("f64", "f32acc"):
        raise ValueError(name)
    with _lock:
        if name != _variant:
            _variant, _lib = name, None


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH if _variant == "f64" else _LIB_F32ACC)
            i32p = ctypes.POINTER(ctypes.c_int32)
            f64p = ctypes.POINTER(ctypes.c_double)
            for name in ("oracle_forward", "oracle_backward_input", "oracle_backward_weight"):
                fn = getattr(lib, name)
                fn.restype = None
                fn.argtypes = [ctypes.c_int] * 6 + [i32p, i32p, f64p, f64p, f64p, ctypes.c_int]
            for name in ("oracle_forward_bilinear", "oracle_backward_input_bilinear", "oracle_backward_weight_bilinear"):
                fn = getattr(lib, name)
                fn.restype = None
                fn.argtypes = [ctypes.c_int] * 6 + [i32p, i32p, f64p, f64p, f64p, f64p, f64p, ctypes.c_int]
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def out_shape(H: int, W: int, stride: int):
    """P = floor((H-1)/str) + 1, Q likewise (reading R2)."""
    return (H - 1) // stride + 1, (W - 1) // stride + 1


def forward(x, w, oh, ow, stride: int = 1, threads: int = 1):
    """y[N][C][P][Q] (f64) of Def. 1.  x: [N][C][H][W], w: [C][K], oh/ow: [C][K] ints."""
    x = _f64(x)
    N, C, H, W = x.shape
    w = _f64(w)
    K = w.shape[1]
    oh, ow = _i32(oh), _i32(ow)
    assert w.shape == (C, K) and oh.shape == (C, K) and ow.shape == (C, K)
    P, Q = out_shape(H, W, stride)
    y = np.empty((N, C, P, Q), np.float64)
    _load().oracle_forward(N, C, H, W, K, stride, _ptr(oh, ctypes.c_int32), _ptr(ow, ctypes.c_int32),
                           _ptr(x, ctypes.c_double), _ptr(w, ctypes.c_double), _ptr(y, ctypes.c_double),
                           threads)
    return y


def backward_input(dy, w, oh, ow, H: int, W: int, stride: int = 1, threads: int = 1):
    """dx[N][C][H][W] (f64): adjoint of forward in x (scatter form)."""
    dy = _f64(dy)
    N, C, P, Q = dy.shape
    w = _f64(w)
    K = w.shape[1]
    oh, ow = _i32(oh), _i32(ow)
    assert (P, Q) == out_shape(H, W, stride)
    dx = np.empty((N, C, H, W), np.float64)
    _load().oracle_backward_input(N, C, H, W, K, stride, _ptr(oh, ctypes.c_int32), _ptr(ow, ctypes.c_int32),
                                  _ptr(dy, ctypes.c_double), _ptr(w, ctypes.c_double),
                                  _ptr(dx, ctypes.c_double), threads)
    return dx


def backward_weight(x, dy, oh, ow, stride: int = 1, threads: int = 1):
    """dW[C][K] (f64): adjoint of forward in w."""
    x, dy = _f64(x), _f64(dy)
    N, C, H, W = x.shape
    oh, ow = _i32(oh), _i32(ow)
    K = oh.shape[1]
    assert dy.shape[:2] == (N, C) and dy.shape[2:] == out_shape(H, W, stride)
    dW = np.empty((C, K), np.float64)
    _load().oracle_backward_weight(N, C, H, W, K, stride, _ptr(oh, ctypes.c_int32), _ptr(ow, ctypes.c_int32),
                                   _ptr(x, ctypes.c_double), _ptr(dy, ctypes.c_double),
                                   _ptr(dW, ctypes.c_double), threads)
    return dW


def _bil(h0, w0, fa, fb):
    return _i32(h0), _i32(w0), _f64(fa), _f64(fb)


def forward_bilinear(x, w, h0, w0, fa, fb, stride: int = 1, threads: int = 1):
    """y[N][C][P][Q] (f64), bilinear discretisation: tables from taps.bilinear_table."""
    x, w = _f64(x), _f64(w)
    N, C, H, W = x.shape
    K = w.shape[1]
    h0, w0, fa, fb = _bil(h0, w0, fa, fb)
    assert h0.shape == (C, K) and fa.shape == (C, K)
    P, Q = out_shape(H, W, stride)
    y = np.empty((N, C, P, Q), np.float64)
    _load().oracle_forward_bilinear(N, C, H, W, K, stride, _ptr(h0, ctypes.c_int32), _ptr(w0, ctypes.c_int32),
                                    _ptr(fa, ctypes.c_double), _ptr(fb, ctypes.c_double), _ptr(x, ctypes.c_double),
                                    _ptr(w, ctypes.c_double), _ptr(y, ctypes.c_double), threads)
    return y


def backward_input_bilinear(dy, w, h0, w0, fa, fb, H: int, W: int, stride: int = 1, threads: int = 1):
    """dx (f64): adjoint in x of forward_bilinear (scatter form)."""
    dy, w = _f64(dy), _f64(w)
    N, C, P, Q = dy.shape
    K = w.shape[1]
    h0, w0, fa, fb = _bil(h0, w0, fa, fb)
    assert (P, Q) == out_shape(H, W, stride)
    dx = np.empty((N, C, H, W), np.float64)
    _load().oracle_backward_input_bilinear(N, C, H, W, K, stride, _ptr(h0, ctypes.c_int32), _ptr(w0, ctypes.c_int32),
                                           _ptr(fa, ctypes.c_double), _ptr(fb, ctypes.c_double),
                                           _ptr(dy, ctypes.c_double), _ptr(w, ctypes.c_double),
                                           _ptr(dx, ctypes.c_double), threads)
    return dx


def backward_weight_bilinear(x, dy, h0, w0, fa, fb, stride: int = 1, threads: int = 1):
    """dW[C][K] (f64): adjoint in w of forward_bilinear."""
    x, dy = _f64(x), _f64(dy)
    N, C, H, W = x.shape
    h0, w0, fa, fb = _bil(h0, w0, fa, fb)
    K = h0.shape[1]
    assert dy.shape[2:] == out_shape(H, W, stride)
    dW = np.empty((C, K), np.float64)
    _load().oracle_backward_weight_bilinear(N, C, H, W, K, stride, _ptr(h0, ctypes.c_int32), _ptr(w0, ctypes.c_int32),
                                            _ptr(fa, ctypes.c_double), _ptr(fb, ctypes.c_double),
                                            _ptr(x, ctypes.c_double), _ptr(dy, ctypes.c_double),
                                            _ptr(dW, ctypes.c_double), threads)
    return dW
