"""Pins for oracle/oracle.c (forward, backward_input, backward_weight).

Pinned against: SPEC worked examples, torch f64 CPU conv2d as a library
routine (horizontal 1xK at 0 deg, vertical Kx1 at 90/270 deg, masked KxK at every
angle, P:1261 + R1 zero padding), torch autograd of that conv2d, and the adjoint /
bilinearity identities of a linear map.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from oracle import taps as T
from paper_2309_15812_b200 import inputs


def _taps(K, angles):
    oh, ow = T.taps_table(K, K // 2, angles)
    return np.array(oh, np.int32), np.array(ow, np.int32)


def _masked_kxk(w, oh, ow, K):
    """Dense K x K depthwise kernel: W2[c][pad+oh][pad+ow] += w[c][k] (duplicates summed)."""
    C = w.shape[0]
    pad = K // 2
    W2 = np.zeros((C, 1, K, K))
    for c in range(C):
        for k in range(K):
            W2[c, 0, pad + oh[c, k], pad + ow[c, k]] += w[c, k]
    return W2


def _rand_case(N, C, H, W, K, angles, seed=0):
    x = inputs.uniform_pm1((N, C, H, W), seed)
    w = inputs.uniform_pm1((C, K), seed + 1)
    oh, ow = _taps(K, angles)
    return x, w, oh, ow


def test_spec_examples():
    a, b, c = 0.3, -1.25, 2.5
    # theta=0, K=3, row x=[a,b,c], w=[1,1,1] -> [a+b, a+b+c, b+c]
    x = np.array([a, b, c]).reshape(1, 1, 1, 3)
    oh, ow = _taps(3, [0.0])
    y = oracle.forward(x, np.ones((1, 3)), oh, ow)
    assert y.ravel().tolist() == [a + b, a + b + c, b + c]
    # 45 deg, 3x3 distinct values: y[1][1] = w0 x[1][0] + w1 x[1][1] + w2 x[0][1]
    x = np.arange(1.0, 10.0).reshape(1, 1, 3, 3)
    w = np.array([[2.0, 3.0, 5.0]])
    oh, ow = _taps(3, [45.0])
    y = oracle.forward(x, w, oh, ow)
    assert y[0, 0, 1, 1] == 2 * x[0, 0, 1, 0] + 3 * x[0, 0, 1, 1] + 5 * x[0, 0, 0, 1]


@pytest.mark.parametrize("K", [3, 7, 31])
def test_delta_kernel_identity(K):
    # w_k = [k == pad] -> y == x (origin tap (0,0))
    angles = [0, 22.5, 45, 90, 135, 200, 300, 359]
    x, _, oh, ow = _rand_case(2, 8, 9, 11, K, angles)
    w = np.zeros((8, K))
    w[:, K // 2] = 1.0
    assert np.array_equal(oracle.forward(x, w, oh, ow), x)


@pytest.mark.parametrize("K", [3, 7, 15])
def test_axis_cases_vs_torch(K):
    pad = K // 2
    x, w, _, _ = _rand_case(2, 4, 13, 17, K, [0.0] * 4)
    xt, wt = torch.from_numpy(x), torch.from_numpy(w)
    # theta=0 == horizontal 1xK depthwise conv
    oh, ow = _taps(K, [0.0] * 4)
    ref = F.conv2d(xt, wt.view(4, 1, 1, K), padding=(0, pad), groups=4).numpy()
    np.testing.assert_allclose(oracle.forward(x, w, oh, ow), ref, rtol=0, atol=1e-13)
    # theta=90 == vertical Kx1 conv with the kernel REVERSED (reading R5)
    oh, ow = _taps(K, [90.0] * 4)
    ref = F.conv2d(xt, wt.flip(1).view(4, 1, K, 1), padding=(pad, 0), groups=4).numpy()
    np.testing.assert_allclose(oracle.forward(x, w, oh, ow), ref, rtol=0, atol=1e-13)
    # theta=270 == vertical Kx1 conv, same order
    oh, ow = _taps(K, [270.0] * 4)
    ref = F.conv2d(xt, wt.view(4, 1, K, 1), padding=(pad, 0), groups=4).numpy()
    np.testing.assert_allclose(oracle.forward(x, w, oh, ow), ref, rtol=0, atol=1e-13)


ANGLE_SETS = {
    "tiny_cycled": [0, 45, 90, 135, 0, 45, 90, 135],
    "tiny_contig": [0, 0, 45, 45, 90, 90, 135, 135],
    "d8": [i * 22.5 for i in range(8)],
    "thirties": [0, 30, 60, 120, 150, 210, 240, 330],
    "integer_deg": [7, 91, 178, 199, 263, 301, 333, 13],
}


@pytest.mark.parametrize("name", sorted(ANGLE_SETS))
@pytest.mark.parametrize("K,stride", [(3, 1), (7, 1), (7, 2), (15, 1), (15, 2)])
def test_forward_vs_masked_conv2d(name, K, stride):
    angles = ANGLE_SETS[name]
    x, w, oh, ow = _rand_case(2, 8, 14, 15, K, angles)
    W2 = torch.from_numpy(_masked_kxk(w, oh, ow, K))
    ref = F.conv2d(torch.from_numpy(x), W2, padding=K // 2, stride=stride, groups=8).numpy()
    y = oracle.forward(x, w, oh, ow, stride=stride)
    assert y.shape == ref.shape
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", sorted(ANGLE_SETS))
@pytest.mark.parametrize("K,stride", [(7, 1), (7, 2), (15, 1)])
def test_backward_vs_autograd(name, K, stride):
    angles = ANGLE_SETS[name]
    N, C, H, W = 2, 8, 13, 14
    x, w, oh, ow = _rand_case(N, C, H, W, K, angles, seed=3)
    P, Q = oracle.out_shape(H, W, stride)
    dy = inputs.uniform_pm1((N, C, P, Q), 7)
    xt = torch.from_numpy(x).requires_grad_(True)
    W2 = torch.from_numpy(_masked_kxk(w, oh, ow, K)).requires_grad_(True)
    y = F.conv2d(xt, W2, padding=K // 2, stride=stride, groups=C)
    y.backward(torch.from_numpy(dy))
    dx = oracle.backward_input(dy, w, oh, ow, H, W, stride)
    np.testing.assert_allclose(dx, xt.grad.numpy(), rtol=0, atol=1e-12)
    dW = oracle.backward_weight(x, dy, oh, ow, stride)
    pad = K // 2
    g = W2.grad.numpy()
    want = np.array([[g[c, 0, pad + oh[c, k], pad + ow[c, k]] for k in range(K)] for c in range(C)])
    np.testing.assert_allclose(dW, want, rtol=0, atol=1e-11)


@pytest.mark.parametrize("stride", [1, 2])
def test_adjoint_identities(stride):
    angles = [i * 22.5 for i in range(8)]
    N, C, H, W, K = 3, 8, 16, 12, 31
    x, w, oh, ow = _rand_case(N, C, H, W, K, angles, seed=11)
    y = oracle.forward(x, w, oh, ow, stride)
    dy = inputs.uniform_pm1(y.shape, 12)
    dx = oracle.backward_input(dy, w, oh, ow, H, W, stride)
    dW = oracle.backward_weight(x, dy, oh, ow, stride)
    lhs = float(np.sum(dy * y))
    assert abs(lhs - float(np.sum(dx * x))) <= 1e-12 * max(1.0, abs(lhs)) * 100
    assert abs(lhs - float(np.sum(dW * w))) <= 1e-12 * max(1.0, abs(lhs)) * 100


def test_duplicate_taps_equal_grad_and_finite_difference():
    # K=7 at 135 deg has a duplicated centre tap: its two weights get equal dW
    oh, ow = _taps(7, [135.0])
    assert (oh[0, 2], ow[0, 2]) == (oh[0, 3], ow[0, 3])
    x = inputs.uniform_pm1((1, 1, 9, 9), 5)
    dy = inputs.uniform_pm1((1, 1, 9, 9), 6)
    dW = oracle.backward_weight(x, dy, oh, ow)
    assert dW[0, 2] == dW[0, 3]
    # central finite differences of L(w) = <dy, y(w)> in a random direction
    w = inputs.uniform_pm1((1, 7), 8)
    v = inputs.uniform_pm1((1, 7), 9)
    h = 1e-6
    Lp = np.sum(dy * oracle.forward(x, w + h * v, oh, ow))
    Lm = np.sum(dy * oracle.forward(x, w - h * v, oh, ow))
    fd = (Lp - Lm) / (2 * h)
    assert abs(fd - float(np.sum(dW * v))) <= 1e-6 * max(1.0, abs(fd))


def test_thread_count_independent():
    angles = [i * 22.5 for i in range(8)]
    x, w, oh, ow = _rand_case(4, 8, 20, 20, 15, angles)
    y1 = oracle.forward(x, w, oh, ow, threads=1)
    y4 = oracle.forward(x, w, oh, ow, threads=4)
    assert np.array_equal(y1, y4)
    dy = inputs.uniform_pm1(y1.shape, 3)
    assert np.array_equal(oracle.backward_weight(x, dy, oh, ow, threads=1),
                          oracle.backward_weight(x, dy, oh, ow, threads=4))


def test_inputs_splitmix64_vector():
    # well-known first output of SplitMix64 seeded with 0
    assert int(inputs.splitmix64(0, 1)[0]) == 0xE220A8397B1DCDAF
    a = inputs.uniform_pm1((1000,), 0)
    assert a.min() >= -1.0 and a.max() < 1.0
    b = inputs.round_to_bf16(a.astype(np.float32))
    assert np.all((b.view(np.uint32) & 0xFFFF) == 0)
    assert np.max(np.abs(b - a)) <= 2.0 ** -8
