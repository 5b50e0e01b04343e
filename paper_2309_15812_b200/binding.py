"""Thin Python binding of liboriented1d (include/oriented1d.h).

Argument marshalling only: every step of the oriented 1D convolution runs in the
library's CUDA kernels.  PyTorch provides device memory and streams.  There is no
CPU fallback: if the shared library is missing or a call fails, this module raises.

Function names follow the C ABI without the `o1d_` prefix (both spellings exported).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboriented1d.so")

O1D_OK = 0
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "INVALID_SHAPE", 3: "INVALID_CONFIG", 4: "SHAPE_MISMATCH",
          5: "UNSUPPORTED", 6: "MISALIGNED", 7: "WORKSPACE_TOO_SMALL", 8: "CUDA_ERROR", 9: "JIT_ERROR"}
DTYPES = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}
FLAG_FORCE_GENERIC = 0x1
FLAG_NO_TMA = 0x2
FLAG_SHEAR = 0x4
FLAG_BILINEAR = 0x8
TAPS = {"rotation": 0, "shear": 1, "bilinear": 2}
ASSIGN = {"contiguous": 0, "cycled": 1}

EXPORTS = ["o1d_make_taps", "o1d_direction_angles", "o1d_plan_create", "o1d_plan_out_shape",
           "o1d_plan_get_taps", "o1d_plan_describe", "o1d_workspace_bytes", "o1d_forward",
           "o1d_backward_input", "o1d_backward_weight", "o1d_step_host_workspace_bytes", "o1d_step_host",
           "o1d_launches_per_call", "o1d_plan_destroy", "o1d_last_error", "o1d_version", "o1d_spec_source",
           "o1d_debug_trace", "o1d_make_taps_ex", "o1d_step", "o1d_make_bilinear", "o1d_plan_stats",
           "o1d_backward"]


class O1DError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Desc(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_int32) for n in ("N", "C", "H", "W", "K", "stride")] + [("pad", ctypes.c_double)]
                + [(n, ctypes.c_int32) for n in ("dtype", "layout", "flags")])


_lib = None
_lock = threading.Lock()


def lib():
    """Load liboriented1d.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                  "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            st, vp, i32, i16p, f64p = ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p
            sig = {
                "o1d_make_taps": (st, [i32, ctypes.c_double, i32, f64p, i16p, i16p]),
                "o1d_direction_angles": (st, [i32, i32, i32, ctypes.c_double, f64p]),
                "o1d_plan_create": (st, [ctypes.POINTER(_Desc), f64p, ctypes.POINTER(vp)]),
                "o1d_plan_out_shape": (st, [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
                "o1d_plan_get_taps": (st, [vp, i16p, i16p]),
                "o1d_plan_describe": (ctypes.c_char_p, [vp]),
                "o1d_workspace_bytes": (ctypes.c_size_t, [vp]),
                "o1d_forward": (st, [vp, vp, vp, vp, vp]),
                "o1d_backward_input": (st, [vp, vp, vp, vp, vp]),
                "o1d_backward_weight": (st, [vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
                "o1d_step_host_workspace_bytes": (ctypes.c_size_t, [vp]),
                "o1d_step_host": (st, [vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
                "o1d_launches_per_call": (i32, [vp, i32]),
                "o1d_plan_destroy": (None, [vp]),
                "o1d_last_error": (ctypes.c_char_p, []),
                "o1d_version": (ctypes.c_char_p, []),
                "o1d_debug_trace": (ctypes.c_size_t, [vp, vp, ctypes.c_size_t]),
                "o1d_make_taps_ex": (st, [i32, ctypes.c_double, i32, f64p, i32, i16p, i16p]),
                "o1d_make_bilinear": (st, [i32, ctypes.c_double, i32, f64p, i16p, i16p, f64p, f64p]),
                "o1d_plan_stats": (st, [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)]),
                "o1d_step": (st, [vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
                "o1d_backward": (st, [vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
                "o1d_spec_source": (st, [ctypes.POINTER(_Desc), f64p, i32, ctypes.c_char_p, ctypes.POINTER(ctypes.c_size_t)]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _check(status: int):
    if status != O1D_OK:
        raise O1DError(status, lib().o1d_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def version() -> str:
    return lib().o1d_version().decode()


def make_taps(K: int, angles_deg, pad: float = -1, discretization: str = "rotation"):
    """Tap tables (oh, ow) int16 [C][K] from the library's host tap generator;
    discretization "rotation" (Def. 1), "shear" (Appendix) or "bilinear"
    (the base corners).  pad: a real number, negative = floor(K/2)."""
    a = np.ascontiguousarray(angles_deg, dtype=np.float64)
    C = a.shape[0]
    oh = np.empty((C, K), np.int16)
    ow = np.empty((C, K), np.int16)
    if discretization not in TAPS:
        raise ValueError("discretization must be 'rotation', 'shear' or 'bilinear'")
    _check(lib().o1d_make_taps_ex(K, float(pad), C, _ptr(a), TAPS[discretization], _ptr(oh), _ptr(ow)))
    return oh, ow


def make_bilinear(K: int, angles_deg, pad: float = -1):
    """Bilinear taps: base corners h0, w0 int16 [C][K] and fractional parts
    fa, fb float64 [C][K] of the real offsets (-(k-pad) sin t, (k-pad) cos t)."""
    a = np.ascontiguousarray(angles_deg, dtype=np.float64)
    C = a.shape[0]
    h0, w0 = np.empty((C, K), np.int16), np.empty((C, K), np.int16)
    fa, fb = np.empty((C, K), np.float64), np.empty((C, K), np.float64)
    _check(lib().o1d_make_bilinear(K, float(pad), C, _ptr(a), _ptr(h0), _ptr(w0), _ptr(fa), _ptr(fb)))
    return h0, w0, fa, fb


def direction_angles(D: int, C: int, assign: str = "contiguous", shift_deg: float = 0.0) -> np.ndarray:
    out = np.empty(C, np.float64)
    _check(lib().o1d_direction_angles(D, C, ASSIGN[assign], float(shift_deg), _ptr(out)))
    return out


def spec_source(N, C, H, W, K, angles_deg, pass_id: int, stride=1, pad=-1, dtype=torch.float32, flags=0) -> str:
    """CUDA source of the specialised kernel for one pass (0 fwd, 1 bwd_in, 2 bwd_w, 3 fused
    backward; host only, diagnostics)."""
    a = np.ascontiguousarray(angles_deg, dtype=np.float64)
    d = _Desc(N, C, H, W, K, stride, float(pad), DTYPES[dtype], 0, flags)
    n = ctypes.c_size_t(0)
    _check(lib().o1d_spec_source(ctypes.byref(d), _ptr(a), pass_id, None, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _check(lib().o1d_spec_source(ctypes.byref(d), _ptr(a), pass_id, buf, ctypes.byref(n)))
    return buf.value.decode()


def _stream_handle(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


class Plan:
    """An immutable o1d_plan for one problem shape, dtype and angle set."""

    def __init__(self, N, C, H, W, K, angles_deg, stride=1, pad=-1, dtype=torch.float32, flags=0, device=None,
                 discretization="rotation"):
        if discretization not in TAPS:
            raise ValueError("discretization must be 'rotation', 'shear' or 'bilinear'")
        if discretization == "shear":
            flags |= FLAG_SHEAR
        if discretization == "bilinear":
            flags |= FLAG_BILINEAR
        a = np.ascontiguousarray(angles_deg, dtype=np.float64)
        if a.shape != (C,):
            raise ValueError("angles must have shape [C]")
        if dtype not in DTYPES:
            raise ValueError(f"unsupported dtype {dtype}")
        self.N, self.C, self.H, self.W, self.K, self.stride = N, C, H, W, K, stride
        self.dtype = dtype
        self.angles = a
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device = dev
        d = _Desc(N, C, H, W, K, stride, float(pad), DTYPES[dtype], 0, flags)
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _check(lib().o1d_plan_create(ctypes.byref(d), _ptr(a), ctypes.byref(h)))
        self._h = h
        P, Q = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().o1d_plan_out_shape(h, ctypes.byref(P), ctypes.byref(Q)))
        self.P, self.Q = P.value, Q.value
        self.pad = K // 2 if pad < 0 else pad
        self.discretization = discretization

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.o1d_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def describe(self) -> str:
        return lib().o1d_plan_describe(self._h).decode()

    @property
    def fused_step(self) -> bool:
        """o1d_step / the module's autograd use the fused single-pass backward (O1D_FUSED=1 at
        plan creation); otherwise backward_input + backward_weight."""
        return "step=fused" in self.describe()

    def taps(self):
        oh = np.empty((self.C, self.K), np.int16)
        ow = np.empty((self.C, self.K), np.int16)
        _check(lib().o1d_plan_get_taps(self._h, _ptr(oh), _ptr(ow)))
        return oh, ow

    def debug_trace(self) -> np.ndarray:
        """O1D_TRACE event records since the last call: uint64 [n, 2] (time ns, tag); empty if tracing is off."""
        buf = np.zeros(1 + 2 * (1 << 21), np.uint64)
        got = lib().o1d_debug_trace(self._h, buf.ctypes.data, buf.nbytes)
        if not got:
            return np.zeros((0, 2), np.uint64)
        rec = buf[1:].reshape(-1, 2)
        return rec[rec[:, 0] != 0]

    def stats(self):
        """(plan-creation host ms, JIT module-cache hit: 1 / 0, -1 = no specialised kernels)."""
        ms, hit = ctypes.c_double(), ctypes.c_int32()
        _check(lib().o1d_plan_stats(self._h, ctypes.byref(ms), ctypes.byref(hit)))
        return ms.value, hit.value

    def workspace_bytes(self) -> int:
        return int(lib().o1d_workspace_bytes(self._h))

    def launches_per_call(self, pass_id: int) -> int:
        return int(lib().o1d_launches_per_call(self._h, pass_id))

    def x_shape(self):
        return (self.N, self.C, self.H, self.W)

    def y_shape(self):
        return (self.N, self.C, self.P, self.Q)


def plan_create(*args, **kw) -> Plan:
    return Plan(*args, **kw)


def _check_tensor(t: torch.Tensor, name: str, shape, dtype, device):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        # a silent copy would hide the paper's own .permute() throughput bug
        raise ValueError(f"{name} must be contiguous (NCHW); no silent copies")


def forward(plan: Plan, x, w, y=None, stream=None):
    _check_tensor(x, "x", plan.x_shape(), plan.dtype, plan.device)
    _check_tensor(w, "w", (plan.C, plan.K), torch.float32, plan.device)
    if y is None:
        y = torch.empty(plan.y_shape(), dtype=plan.dtype, device=plan.device)
    _check_tensor(y, "y", plan.y_shape(), plan.dtype, plan.device)
    _check(lib().o1d_forward(plan.handle, x.data_ptr(), w.data_ptr(), y.data_ptr(), _stream_handle(stream)))
    return y


def backward_input(plan: Plan, dy, w, dx=None, stream=None):
    _check_tensor(dy, "dy", plan.y_shape(), plan.dtype, plan.device)
    _check_tensor(w, "w", (plan.C, plan.K), torch.float32, plan.device)
    if dx is None:
        dx = torch.empty(plan.x_shape(), dtype=plan.dtype, device=plan.device)
    _check_tensor(dx, "dx", plan.x_shape(), plan.dtype, plan.device)
    _check(lib().o1d_backward_input(plan.handle, dy.data_ptr(), w.data_ptr(), dx.data_ptr(), _stream_handle(stream)))
    return dx


def workspace(plan: Plan):
    n = max(plan.workspace_bytes(), 16)
    return torch.empty((n + 3) // 4, dtype=torch.float32, device=plan.device)


def backward_weight(plan: Plan, x, dy, dW=None, ws=None, stream=None):
    _check_tensor(x, "x", plan.x_shape(), plan.dtype, plan.device)
    _check_tensor(dy, "dy", plan.y_shape(), plan.dtype, plan.device)
    if dW is None:
        dW = torch.empty((plan.C, plan.K), dtype=torch.float32, device=plan.device)
    _check_tensor(dW, "dW", (plan.C, plan.K), torch.float32, plan.device)
    if ws is None:
        ws = workspace(plan)
    _check(lib().o1d_backward_weight(plan.handle, x.data_ptr(), dy.data_ptr(), dW.data_ptr(), ws.data_ptr(),
                                     ws.numel() * ws.element_size(), _stream_handle(stream)))
    return dW


def backward(plan: Plan, x, dy, w, dx=None, dW=None, ws=None, stream=None):
    """backward_input and backward_weight in one pass over x and dy (o1d_backward, NEXT-2)."""
    _check_tensor(x, "x", plan.x_shape(), plan.dtype, plan.device)
    _check_tensor(dy, "dy", plan.y_shape(), plan.dtype, plan.device)
    _check_tensor(w, "w", (plan.C, plan.K), torch.float32, plan.device)
    dx = torch.empty(plan.x_shape(), dtype=plan.dtype, device=plan.device) if dx is None else dx
    dW = torch.empty((plan.C, plan.K), dtype=torch.float32, device=plan.device) if dW is None else dW
    _check_tensor(dx, "dx", plan.x_shape(), plan.dtype, plan.device)
    _check_tensor(dW, "dW", (plan.C, plan.K), torch.float32, plan.device)
    ws = workspace(plan) if ws is None else ws
    _check(lib().o1d_backward(plan.handle, x.data_ptr(), dy.data_ptr(), w.data_ptr(), dx.data_ptr(), dW.data_ptr(),
                              ws.data_ptr(), ws.numel() * ws.element_size(), _stream_handle(stream)))
    return dx, dW


def step(plan: Plan, x, w, dy, y=None, dx=None, dW=None, ws=None, stream=None):
    """One layer training step on device tensors (o1d_step): forward, backward_input and
    backward_weight with the later passes overlapping the earlier ones' tails."""
    _check_tensor(x, "x", plan.x_shape(), plan.dtype, plan.device)
    _check_tensor(dy, "dy", plan.y_shape(), plan.dtype, plan.device)
    _check_tensor(w, "w", (plan.C, plan.K), torch.float32, plan.device)
    y = torch.empty(plan.y_shape(), dtype=plan.dtype, device=plan.device) if y is None else y
    dx = torch.empty(plan.x_shape(), dtype=plan.dtype, device=plan.device) if dx is None else dx
    dW = torch.empty((plan.C, plan.K), dtype=torch.float32, device=plan.device) if dW is None else dW
    _check_tensor(y, "y", plan.y_shape(), plan.dtype, plan.device)
    _check_tensor(dx, "dx", plan.x_shape(), plan.dtype, plan.device)
    _check_tensor(dW, "dW", (plan.C, plan.K), torch.float32, plan.device)
    ws = workspace(plan) if ws is None else ws
    _check(lib().o1d_step(plan.handle, x.data_ptr(), w.data_ptr(), dy.data_ptr(), y.data_ptr(), dx.data_ptr(),
                          dW.data_ptr(), ws.data_ptr(), ws.numel() * ws.element_size(), _stream_handle(stream)))
    return y, dx, dW


def step_host_workspace(plan: Plan):
    n = int(lib().o1d_step_host_workspace_bytes(plan.handle))
    return torch.empty((n + 3) // 4, dtype=torch.float32, device=plan.device)


def step_host(plan: Plan, x_h, w_h, dy_h, y_h, dx_h, dW_h, dev_ws, stream=None):
    """One layer training step through HOST (pinned) buffers: H2D, fwd, bwd_in, bwd_w, D2H, sync."""
    for t, n in ((x_h, "x_h"), (w_h, "w_h"), (dy_h, "dy_h"), (y_h, "y_h"), (dx_h, "dx_h"), (dW_h, "dW_h")):
        if t.device.type != "cpu" or not t.is_contiguous():
            raise ValueError(f"{n} must be a contiguous host tensor")
    _check(lib().o1d_step_host(plan.handle, x_h.data_ptr(), w_h.data_ptr(), dy_h.data_ptr(), y_h.data_ptr(),
                               dx_h.data_ptr(), dW_h.data_ptr(), dev_ws.data_ptr(),
                               dev_ws.numel() * dev_ws.element_size(), _stream_handle(stream)))


# C-ABI spellings
o1d_make_taps = make_taps
o1d_direction_angles = direction_angles
o1d_plan_create = plan_create
o1d_forward = forward
o1d_backward_input = backward_input
o1d_backward_weight = backward_weight
o1d_backward = backward
o1d_make_bilinear = make_bilinear
o1d_step_host = step_host
