"""Pins for the oracle's bilinear discretisation (Sec. "Discretization and
Interpolation"; Table "bilinear" P:322-334) and for real-valued pads (Eq. coordinate1d,
P:346-351).

Each pin is something other than the oracle's own formula: torch.nn.functional.grid_sample
(bilinear, zero padding, align_corners=True) as a library routine sampling x at the real
coordinates of Eq. coordinate2d, its autograd, f64 trig evaluated independently (numpy),
the rotation oracle where all fractional parts vanish (the axis angles), sympy floors for
rational pads, partition of unity, and the adjoint identities of a linear map.
"""
import math

import numpy as np
import pytest
import sympy
import torch
import torch.nn.functional as F

import oracle
from oracle import taps as T
from paper_2309_15812_b200 import inputs

ANGLES = [0.0, 30.0, 45.0, 90.0, 112.5, 135.0, 200.0, 17.3, -61.0, 270.0]


def _tables(K, angles, pad=None):
    pad = K // 2 if pad is None else pad
    h0, w0, fa, fb = T.bilinear_table(K, pad, angles)
    return np.array(h0), np.array(w0), np.array(fa), np.array(fb)


def test_tables_vs_independent_trig():
    """Base corner = the exact floor taps; h0 + a and w0 + b reproduce the real offsets
    -(k-pad) sin t, (k-pad) cos t evaluated with numpy f64 trig; a, b in [0, 1)."""
    for K in (3, 7, 31):
        pad = K // 2
        for t in ANGLES + [i * 7.5 for i in range(48)]:
            rows = T.bilinear_exact(K, pad, t)
            assert [(r[0], r[1]) for r in rows] == T.taps_exact(K, pad, t)
            r = math.radians(t)
            for k, (h0, w0, a, b) in enumerate(rows):
                assert 0.0 <= a < 1.0 and 0.0 <= b < 1.0
                assert abs(h0 + a - (-(k - pad) * np.sin(r))) < 1e-12
                assert abs(w0 + b - ((k - pad) * np.cos(r))) < 1e-12


def test_niven_fractions_exact():
    # 30 deg: -(k-3) sin 30 = (3-k)/2 -> a in {0, 1/2} exactly; 90 deg: cos = 0 -> b == 0
    for h0, w0, a, b in T.bilinear_exact(7, 3, 30.0):
        assert a in (0.0, 0.5)
    assert all(b == 0.0 and a == 0.0 for _, _, a, b in T.bilinear_exact(9, 4, 90.0))
    assert all(b == 0.0 and a == 0.0 for _, _, a, b in T.bilinear_exact(9, 4, 0.0))


def _grid_sample_forward(x, w, K, angles, stride, pad=None):
    """y = sum_k w_k * bilinear sample of x at (str*p - (k-pad) sin t, str*q + (k-pad) cos t),
    via torch grid_sample (f64, zero padding, align_corners=True); independent of oracle.c."""
    pad = K // 2 if pad is None else pad
    xt = torch.from_numpy(x)
    N, C, H, W = x.shape
    P, Q = oracle.out_shape(H, W, stride)
    y = torch.zeros((N, C, P, Q), dtype=torch.float64)
    pp = torch.arange(P, dtype=torch.float64) * stride
    qq = torch.arange(Q, dtype=torch.float64) * stride
    for c in range(C):
        r = math.radians(angles[c])
        for k in range(K):
            u, v = -(k - pad) * math.sin(r), (k - pad) * math.cos(r)
            hh = (pp + u)[:, None].expand(P, Q)
            ww = (qq + v)[None, :].expand(P, Q)
            grid = torch.stack([2 * ww / (W - 1) - 1, 2 * hh / (H - 1) - 1], dim=-1)[None].expand(N, P, Q, 2)
            s = F.grid_sample(xt[:, c:c + 1], grid, mode="bilinear", padding_mode="zeros", align_corners=True)
            y[:, c] += w[c, k] * s[:, 0]
    return y.numpy()


@pytest.mark.parametrize("stride", [1, 2])
def test_forward_vs_grid_sample(stride):
    K, C = 7, len(ANGLES)
    x = inputs.uniform_pm1((2, C, 9, 11), 0)
    w = inputs.uniform_pm1((C, K), 1)
    h0, w0, fa, fb = _tables(K, ANGLES)
    y = oracle.forward_bilinear(x, w, h0, w0, fa, fb, stride)
    ref = _grid_sample_forward(x, w, K, ANGLES, stride)
    assert np.max(np.abs(y - ref)) < 1e-12


def test_axis_angles_equal_rotation_oracle():
    K = 9
    angles = [0.0, 90.0, 180.0, 270.0]
    x = inputs.uniform_pm1((1, 4, 10, 12), 3)
    w = inputs.uniform_pm1((4, K), 4)
    h0, w0, fa, fb = _tables(K, angles)
    oh, ow = T.taps_table(K, K // 2, angles)
    assert np.array_equal(oracle.forward_bilinear(x, w, h0, w0, fa, fb), oracle.forward(x, w, np.array(oh), np.array(ow)))


def test_partition_of_unity():
    # constant image, outputs whose taps stay inside: y = sum_k w_k (the four weights sum to 1)
    K = 5
    x = np.ones((1, 3, 20, 20))
    w = inputs.uniform_pm1((3, K), 5)
    h0, w0, fa, fb = _tables(K, [17.0, 63.0, 141.0])
    y = oracle.forward_bilinear(x, w, h0, w0, fa, fb)
    assert np.allclose(y[:, :, 5:15, 5:15], w.sum(axis=1)[None, :, None, None], atol=1e-13)


@pytest.mark.parametrize("stride", [1, 2])
def test_backward_vs_autograd_and_adjoint(stride):
    K, C = 5, 6
    angles = ANGLES[:C]
    x = inputs.uniform_pm1((2, C, 8, 9), 6)
    w = inputs.uniform_pm1((C, K), 7)
    h0, w0, fa, fb = _tables(K, angles)
    P, Q = oracle.out_shape(8, 9, stride)
    dy = inputs.uniform_pm1((2, C, P, Q), 8)
    dx = oracle.backward_input_bilinear(dy, w, h0, w0, fa, fb, 8, 9, stride)
    dW = oracle.backward_weight_bilinear(x, dy, h0, w0, fa, fb, stride)
    # torch autograd through the grid_sample formulation
    xt = torch.from_numpy(x).requires_grad_(True)
    wt = torch.from_numpy(w).requires_grad_(True)
    N, _, H, W = x.shape
    pp = torch.arange(P, dtype=torch.float64) * stride
    qq = torch.arange(Q, dtype=torch.float64) * stride
    ys = []
    for c in range(C):
        r = math.radians(angles[c])
        acc = 0
        for k in range(K):
            u, v = -(k - K // 2) * math.sin(r), (k - K // 2) * math.cos(r)
            grid = torch.stack([2 * (qq + v)[None, :].expand(P, Q) / (W - 1) - 1,
                                2 * (pp + u)[:, None].expand(P, Q) / (H - 1) - 1], dim=-1)[None].expand(N, P, Q, 2)
            acc = acc + wt[c, k] * F.grid_sample(xt[:, c:c + 1], grid, mode="bilinear", padding_mode="zeros",
                                                 align_corners=True)[:, 0]
        ys.append(acc)
    torch.stack(ys, 1).backward(torch.from_numpy(dy))
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-12
    assert np.max(np.abs(dW - wt.grad.numpy())) < 1e-11
    # adjoint / bilinearity identities
    y = oracle.forward_bilinear(x, w, h0, w0, fa, fb, stride)
    assert abs(np.vdot(dy, y) - np.vdot(dx, x)) < 1e-10
    assert abs(np.vdot(dW, w) - np.vdot(dy, y)) < 1e-10


def test_real_pad_taps_sympy():
    """Eq. coordinate1d with a non-integer pad (P:346-351 leaves pad_w real): exact floors
    against sympy with the pad as an exact rational."""
    for K, pad in ((6, 2.5), (7, 1.25), (4, 0.5)):
        for i in range(0, 24):
            t = sympy.Rational(15, 1) * i
            ang = sympy.pi * t / 180
            pr = sympy.Rational(pad)
            want = [(int(sympy.floor(-(k - pr) * sympy.sin(ang))), int(sympy.floor((k - pr) * sympy.cos(ang))))
                    for k in range(K)]
            assert T.taps_exact(K, pad, float(t)) == want, (K, pad, float(t))
