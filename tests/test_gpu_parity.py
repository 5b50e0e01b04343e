"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on identical
seeded inputs.  Tolerances (BASELINE.json north_star, reading R9): normwise
max|g - r| / max|r| <= 1e-5 for fp32, <= 2e-2 for bf16/fp16 (fp32 accumulation);
tap tables bit-exact; results bitwise deterministic."""
import numpy as np
import pytest
import torch

import oracle
from oracle import taps as T
from paper_2309_15812_b200 import binding as B
from paper_2309_15812_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2, torch.float16: 2e-2}
NP_DT = {torch.float32: "f32", torch.bfloat16: "bf16", torch.float16: "f16"}


def nerr(g: torch.Tensor, r: np.ndarray) -> float:
    g = g.double().cpu().numpy()
    den = float(np.max(np.abs(r)))
    return float(np.max(np.abs(g - r))) / (den if den > 0 else 1.0)


_oracle_cache = {}


def oracle_case(N, C, H, W, K, angles, stride, dt, disc, x, w, dy, threads=None):
    """(oh, ow, y, dx, dW) of the oracle on these inputs (cached for the last key)."""
    key = (N, C, H, W, K, tuple(angles), stride, dt, disc)
    if key not in _oracle_cache:
        th = threads or max(1, oracle.max_threads())
        _oracle_cache.clear()
        if disc == "bilinear":
            h0, w0, fa, fb = (np.array(v) for v in T.bilinear_table(K, K // 2, angles))
            oh, ow = h0.astype(np.int32), w0.astype(np.int32)
            _oracle_cache[key] = (oh, ow, oracle.forward_bilinear(x, w, h0, w0, fa, fb, stride, th),
                                  oracle.backward_input_bilinear(dy, w, h0, w0, fa, fb, H, W, stride, th),
                                  oracle.backward_weight_bilinear(x, dy, h0, w0, fa, fb, stride, th))
        else:
            oh, ow = T.taps_table(K, K // 2, angles, disc)
            oh, ow = np.array(oh, np.int32), np.array(ow, np.int32)
            _oracle_cache[key] = (oh, ow, oracle.forward(x, w, oh, ow, stride, th),
                                  oracle.backward_input(dy, w, oh, ow, H, W, stride, th),
                                  oracle.backward_weight(x, dy, oh, ow, stride, th))
    return _oracle_cache[key]


def run_case(N, C, H, W, K, angles, stride=1, dtype=torch.float32, flags=0, threads=None, check_det=False,
             disc="rotation", expect=None):
    """All passes (forward, backward_input, backward_weight and the fused o1d_backward) vs the
    oracle; `expect`: "spec" / "generic" = the kernel family the plan must select."""
    angles = [float(a) for a in angles]
    plan = B.Plan(N, C, H, W, K, np.array(angles), stride=stride, dtype=dtype, flags=flags, device="cuda:0",
                  discretization=disc)
    if expect == "spec":
        assert plan.describe().startswith("spec"), plan.describe()
    elif expect == "spec-small":
        assert plan.describe().startswith("spec-small"), plan.describe()
    elif expect == "generic":
        assert plan.describe().startswith("generic"), plan.describe()
    P, Q = plan.P, plan.Q
    dt = NP_DT[dtype]
    x = inputs.activation((N, C, H, W), 0, dt)
    w = inputs.weights(C, K, 1)
    dy = inputs.activation((N, C, P, Q), 2, dt)
    oh, ow, ry, rdx, rdW = oracle_case(N, C, H, W, K, angles, stride, dt, disc, x, w, dy, threads)
    poh, pow_ = plan.taps()
    assert np.array_equal(poh, oh) and np.array_equal(pow_, ow), "tap tables must be bit-exact"
    tx = torch.from_numpy(x).to("cuda:0", dtype)
    tdy = torch.from_numpy(dy).to("cuda:0", dtype)
    tw = torch.from_numpy(w).cuda()
    y = B.forward(plan, tx, tw)
    dx = B.backward_input(plan, tdy, tw)
    dW = B.backward_weight(plan, tx, tdy)
    fdx, fdW = B.backward(plan, tx, tdy, tw)
    torch.cuda.synchronize()
    errs = {"y": nerr(y, ry), "dx": nerr(dx, rdx), "dW": nerr(dW, rdW)}
    tol = TOL[dtype]
    assert all(e <= tol for e in errs.values()), (plan.describe(), errs)
    # the fused backward (NEXT-2) computes the same partial sums in the same order: bitwise
    assert torch.equal(fdx, dx) and torch.equal(fdW, dW), plan.describe()
    if check_det:
        y2 = B.forward(plan, tx, tw)
        dx2 = B.backward_input(plan, tdy, tw)
        dW2 = B.backward_weight(plan, tx, tdy)
        assert torch.equal(y, y2) and torch.equal(dx, dx2) and torch.equal(dW, dW2)
    return plan, errs


FLAGS = {"default": 0, "generic": B.FLAG_FORCE_GENERIC}


@pytest.mark.parametrize("flags", sorted(FLAGS))
@pytest.mark.parametrize("assign", ["cycled", "contiguous"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("stride", [1, 2])
def test_tiny(flags, assign, dtype, stride):
    # BASELINE configs[0]: N=1, C=8, 14x14, K=7, {0,45,90,135} deg
    angles = T.direction_angles(4, 8, assign)
    run_case(1, 8, 14, 14, 7, angles, stride, dtype, FLAGS[flags], check_det=True)


@pytest.mark.parametrize("flags", sorted(FLAGS))
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("HW", [(56, 56), (37, 45), (61, 29), (7, 9), (1, 1), (1, 40), (40, 1)])
def test_stage1_like_ragged(flags, dtype, HW):
    """K=31, 8 angles, multiple tiles with ragged edges, degenerate 1-pixel images."""
    H, W = HW
    run_case(2, 16, H, W, 31, T.direction_angles(8, 16, "cycled"), 1, dtype, FLAGS[flags], check_det=True)


@pytest.mark.parametrize("flags", sorted(FLAGS))
@pytest.mark.parametrize("K", [1, 3, 7, 15, 23, 31, 39, 47, 55, 63])
def test_ksweep_shape(flags, K):
    # configs[2] geometry (14x14, D=8 cycled) at a reduced N, C
    run_case(2, 16, 14, 14, K, T.direction_angles(8, 16, "cycled"), 1, torch.float32, FLAGS[flags])


@pytest.mark.parametrize("flags", sorted(FLAGS))
@pytest.mark.parametrize("angle_set", ["thirties_DC96", "integer_deg", "single_45", "neg_and_big"])
@pytest.mark.parametrize("stride", [1, 2])
def test_angle_sets(flags, angle_set, stride):
    if angle_set == "thirties_DC96":
        angles, C = T.direction_angles(96, 96), 96
    elif angle_set == "integer_deg":
        angles, C = [float((37 * c) % 360) for c in range(24)], 24
    elif angle_set == "single_45":
        angles, C = [45.0] * 8, 8
    else:
        angles, C = [-30.0, 725.5, -3600.0, 1e3, 89.999, 90.001, 180.0, 270.0], 8
    run_case(1, C, 30, 23, 15, angles, stride, torch.float32, FLAGS[flags])


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_full_stage1_config(dtype):
    """BASELINE configs[1] at full size, in the launch configuration bench.py times."""
    wl = inputs.S1
    angles = T.direction_angles(wl.D, wl.C, wl.assign)
    plan, errs = run_case(wl.N, wl.C, wl.H, wl.W, wl.K, angles, 1, dtype, 0)
    print(plan.describe(), errs)


@pytest.mark.parametrize("K", [7, 31, 63])
def test_full_ksweep_config(K):
    """BASELINE configs[2] (N=128, C=384, 14x14, D=8) at full size."""
    wl = inputs.ksweep(K)
    angles = T.direction_angles(wl.D, wl.C, wl.assign)
    plan, errs = run_case(wl.N, wl.C, wl.H, wl.W, wl.K, angles, 1, torch.float32, 0)
    print(plan.describe(), errs)


def test_errors_on_gpu():
    plan = B.Plan(1, 8, 14, 14, 7, np.zeros(8), device="cuda:0")
    x = torch.zeros(1, 8, 14, 14, device="cuda:0")
    w = torch.zeros(8, 7, device="cuda:0")
    with pytest.raises(ValueError):
        B.forward(plan, x.transpose(2, 3), w)  # non-contiguous is an error, never a silent copy
    with pytest.raises(ValueError):
        B.forward(plan, x.half(), w)
    ws = torch.zeros(1, device="cuda:0")
    with pytest.raises(B.O1DError) as e:
        B.backward_weight(plan, x, x, ws=ws)
    assert e.value.status == 7
    import ctypes
    L = B.lib()
    st = L.o1d_forward(plan.handle, ctypes.c_void_p(x.data_ptr() + 4), ctypes.c_void_p(w.data_ptr()),
                       ctypes.c_void_p(x.data_ptr()), None)
    assert st == 6  # MISALIGNED


def test_concurrent_streams_same_plan():
    """One plan, launches in flight on several streams at once (work-queue slots)."""
    wl = inputs.S1
    angles = T.direction_angles(wl.D, wl.C, wl.assign)
    plan = B.Plan(8, wl.C, wl.H, wl.W, wl.K, np.array(angles), device="cuda:0")
    xs = [torch.from_numpy(inputs.activation(plan.x_shape(), 20 + i)).cuda() for i in range(4)]
    w = torch.from_numpy(inputs.weights(wl.C, wl.K)).cuda()
    ref = [B.forward(plan, x, w) for x in xs]
    refw = [B.backward_weight(plan, x, x) for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in xs]
    outs, outw = [], []
    for _ in range(3):
        for x, st in zip(xs, streams):
            with torch.cuda.stream(st):
                outs.append(B.forward(plan, x, w, stream=st))
                outw.append(B.backward_weight(plan, x, x, stream=st))
    torch.cuda.synchronize()
    for i, (y, dW) in enumerate(zip(outs, outw)):
        assert torch.equal(y, ref[i % 4]) and torch.equal(dW, refw[i % 4])


def test_module_autograd():
    from paper_2309_15812_b200.module import Oriented1dDWConv
    torch.manual_seed(0)
    m = Oriented1dDWConv(16, 7, D=8).cuda()
    x = torch.randn(2, 16, 20, 20, device="cuda:0", requires_grad=True)
    y = m(x)
    y.square().sum().backward()
    angles = m.angles_deg.tolist()
    oh, ow = T.taps_table(7, 3, angles)
    oh, ow = np.array(oh), np.array(ow)
    xd = x.detach().double().cpu().numpy()
    wd = m.weight.detach().double().cpu().numpy()
    ry = oracle.forward(xd, wd, oh, ow)
    assert nerr(y.detach(), ry) <= 1e-5
    g = 2 * ry
    assert nerr(x.grad, oracle.backward_input(g, wd, oh, ow, 20, 20)) <= 1e-5
    assert nerr(m.weight.grad, oracle.backward_weight(xd, g, oh, ow)) <= 1e-5


def test_step_host_matches_device_path():
    wl = inputs.TINY
    angles = T.direction_angles(wl.D, wl.C, wl.assign)
    plan = B.Plan(wl.N, wl.C, wl.H, wl.W, wl.K, np.array(angles), device="cuda:0")
    x = torch.from_numpy(inputs.activation(plan.x_shape(), 0)).pin_memory()
    w = torch.from_numpy(inputs.weights(wl.C, wl.K)).pin_memory()
    dy = torch.from_numpy(inputs.activation(plan.y_shape(), 2)).pin_memory()
    y, dx, dW = torch.empty_like(x).pin_memory(), torch.empty_like(x).pin_memory(), torch.empty_like(w).pin_memory()
    B.step_host(plan, x, w, dy, y, dx, dW, B.step_host_workspace(plan))
    xd, wd, dyd = x.cuda(), w.cuda(), dy.cuda()
    assert torch.equal(y, B.forward(plan, xd, wd).cpu())
    assert torch.equal(dx, B.backward_input(plan, dyd, wd).cpu())
    assert torch.equal(dW, B.backward_weight(plan, xd, dyd).cpu())


def test_convnext1d_harness_trains():
    """The ConvNeXt-T-1D harness runs a bf16 training step through liboriented1d
    (smaller image; every oriented layer's weight receives a finite gradient)."""
    from paper_2309_15812_b200 import convnext1d
    torch.manual_seed(0)
    m = convnext1d.ConvNeXt1D("convnext_t_1d", num_classes=10).cuda().to(torch.bfloat16)
    for layer in convnext1d.oriented_layers(m):
        layer.weight.data = layer.weight.data.float()
    x = torch.randn(2, 3, 64, 64, device="cuda:0").to(torch.bfloat16)
    out = m(x)
    loss = torch.nn.functional.cross_entropy(out.float(), torch.tensor([1, 3], device="cuda:0"))
    loss.backward()
    assert torch.isfinite(loss)
    for layer in convnext1d.oriented_layers(m):
        assert layer.weight.grad is not None and torch.isfinite(layer.weight.grad).all()


def test_repeated_launches_bitwise():
    """Hundreds of back-to-back steps without host synchronisation (as bench.py runs them)
    give bitwise the first step's results: the persistent kernels' per-launch scheduler
    slots are reset correctly and no item is skipped or repeated."""
    wl = inputs.S1
    angles = T.direction_angles(wl.D, wl.C, wl.assign)
    plan = B.Plan(wl.N, wl.C, wl.H, wl.W, wl.K, np.array(angles), device="cuda:0")
    g = torch.Generator(device="cuda:0").manual_seed(0)
    x = torch.rand(wl.N, wl.C, wl.H, wl.W, device="cuda:0", generator=g)
    dy = torch.rand(wl.N, wl.C, wl.H, wl.W, device="cuda:0", generator=g)
    w = torch.rand(wl.C, wl.K, device="cuda:0", generator=g)
    ws = B.workspace(plan)
    y0 = B.forward(plan, x, w).clone()
    dx0 = B.backward_input(plan, dy, w).clone()
    dW0 = B.backward_weight(plan, x, dy, ws=ws).clone()
    n = 240  # > 64 launch slots per pass, several times over
    ys = torch.empty((8,) + tuple(y0.shape), device="cuda:0")
    dxs = torch.empty((8,) + tuple(dx0.shape), device="cuda:0")
    dWs = torch.empty((n,) + tuple(dW0.shape), device="cuda:0")
    bad = []
    for i in range(n):
        B.forward(plan, x, w, ys[i % 8])
        B.backward_input(plan, dy, w, dxs[i % 8])
        B.backward_weight(plan, x, dy, dWs[i], ws)
        if i % 8 == 7:
            torch.cuda.synchronize()
            for k in range(8):
                if not (torch.equal(ys[k], y0) and torch.equal(dxs[k], dx0)):
                    bad.append(i - 7 + k)
    torch.cuda.synchronize()
    bad += [i for i in range(n) if not torch.equal(dWs[i], dW0)]
    assert not bad, f"steps with different results: {sorted(set(bad))[:20]}"


@pytest.mark.parametrize("flags", sorted(FLAGS))
@pytest.mark.parametrize("HW", [(56, 56), (37, 48), (14, 14)])
@pytest.mark.parametrize("stride", [1, 2])
def test_shear_discretization(flags, HW, stride):
    """Shear-form tap tables (Appendix "Rotation vs Shearing"; plan flag
    O1D_FLAG_SHEAR) through every pass vs the oracle with the same tables."""
    H, W = HW
    angles = T.direction_angles(8, 16, "cycled") if stride == 1 else [-45.0, 10.0, 30.0, 60.0, 100.0, 135.0, 170.0, 225.0]
    C = len(angles) if stride != 1 else 16
    plan, errs = run_case(2, C, H, W, 31 if stride == 1 else 7, angles, stride, torch.float32, FLAGS[flags],
                          check_det=True, disc="shear")
    oh, ow = plan.taps()
    assert all(len(set(zip(oh[c], ow[c]))) == plan.K for c in range(plan.C))  # no redundant taps


def test_shear_full_stage1():
    """BASELINE configs[1] shape with shear tables, in the bench launch configuration."""
    wl = inputs.S1
    run_case(wl.N, wl.C, wl.H, wl.W, wl.K, T.direction_angles(wl.D, wl.C, wl.assign), 1, torch.float32, 0,
             disc="shear")


@pytest.mark.parametrize("which", ["pp_main", "pp_res"])
def test_1dpp_block_workloads(which):
    """the 1D++ block's K=15 main conv (C=96) and its residual 1x31 conv on
    the 4C inverted bottleneck (C=384), 56x56, D=8, at N=4 (every table
    and the bench launch configuration; the full batch only adds planes)."""
    wl = inputs.WORKLOADS[which]
    run_case(4, wl.C, wl.H, wl.W, wl.K, T.direction_angles(wl.D, wl.C, wl.assign), 1, torch.float32, 0,
             check_det=True)


@pytest.mark.parametrize("chunks", ["1", "3", "8"])
def test_step_host_pipelined_bitwise(chunks, monkeypatch):
    """o1d_step_host pipelined over batch chunks (v2 kernels with a batch window; H2D,
    kernels and D2H on three streams) gives bitwise the device path's y, dx and dW
    (the chunks' dW partials land in the full workspace; one finalize)."""
    monkeypatch.setenv("O1D_E2E_CHUNKS", chunks)
    angles = T.direction_angles(8, 16, "cycled")
    plan = B.Plan(8, 16, 56, 56, 31, np.array(angles), device="cuda:0")
    assert plan.describe().startswith("spec")
    x = torch.from_numpy(inputs.activation(plan.x_shape(), 0)).pin_memory()
    w = torch.from_numpy(inputs.weights(16, 31)).pin_memory()
    dy = torch.from_numpy(inputs.activation(plan.y_shape(), 2)).pin_memory()
    y, dx, dW = torch.empty_like(x).pin_memory(), torch.empty_like(x).pin_memory(), torch.empty_like(w).pin_memory()
    for _ in range(2):
        B.step_host(plan, x, w, dy, y, dx, dW, B.step_host_workspace(plan))
        xd, wd, dyd = x.cuda(), w.cuda(), dy.cuda()
        assert torch.equal(y, B.forward(plan, xd, wd).cpu())
        assert torch.equal(dx, B.backward_input(plan, dyd, wd).cpu())
        assert torch.equal(dW, B.backward_weight(plan, xd, dyd).cpu())



def test_step_api_bitwise_and_repeated():
    """o1d_step (the three passes with the later ones overlapping the earlier ones' tails)
    gives bitwise the results of the three separate calls, step after step."""
    wl = inputs.S1
    angles = T.direction_angles(wl.D, wl.C, wl.assign)
    plan = B.Plan(wl.N, wl.C, wl.H, wl.W, wl.K, np.array(angles), device="cuda:0")
    g = torch.Generator(device="cuda:0").manual_seed(1)
    x = torch.rand(wl.N, wl.C, wl.H, wl.W, device="cuda:0", generator=g)
    dy = torch.rand(wl.N, wl.C, wl.H, wl.W, device="cuda:0", generator=g)
    w = torch.rand(wl.C, wl.K, device="cuda:0", generator=g)
    y0, dx0, dW0 = B.forward(plan, x, w), B.backward_input(plan, dy, w), B.backward_weight(plan, x, dy)
    ws = B.workspace(plan)
    y, dx, dW = torch.empty_like(y0), torch.empty_like(dx0), torch.empty_like(dW0)
    for i in range(100):
        B.step(plan, x, w, dy, y, dx, dW, ws)
        if i % 25 == 24:
            torch.cuda.synchronize()
            assert torch.equal(y, y0) and torch.equal(dx, dx0) and torch.equal(dW, dW0), i


# ---------------------------------------------------------------------------------------
# Angle sets, assignments and strides at SPEC-ELIGIBLE shapes (the JIT kernels), VERDICT r1
# item 1(a)/(b): every test asserts which kernel family ran.
SPEC_SETS = {
    # <= 16 distinct tables of the D=C 30-degree family (Niven angles: exact floors matter)
    "thirties_16": [i * 180.0 / 96 for i in range(0, 96, 6)],
    "thirties_exact": [0.0, 30.0, 60.0, 90.0, 120.0, 150.0, 210.0, 330.0],
    "integer_deg": [float((37 * c) % 360) for c in range(16)],
    "near_90": [89.999, 90.001, 89.9999999, 90.0000001, 0.001, -0.001, 179.999, 45.0],
    "neg_and_big": [-30.0, 725.5, -3600.0, 1e3, -1e5 - 30.0, 1e6 + 0.5, 180.0, 270.0],
}


@pytest.mark.parametrize("HW,K", [((56, 56), 31), ((40, 48), 15)])
@pytest.mark.parametrize("angle_set", sorted(SPEC_SETS))
def test_angle_sets_spec(angle_set, K, HW):
    angles = SPEC_SETS[angle_set]
    C = 16
    angles = [angles[c % len(angles)] for c in range(C)]
    H, W = HW
    run_case(2, C, H, W, K, angles, 1, torch.float32, 0, expect="spec")


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("assign", ["contiguous", "cycled"])
def test_assignments_spec(assign, dtype):
    # the model harness uses the paper's contiguous groups
    run_case(2, 16, 56, 56, 31, T.direction_angles(8, 16, assign), 1, dtype, 0, check_det=True, expect="spec")


def test_full_stage1_contiguous():
    wl = inputs.S1
    run_case(wl.N, wl.C, wl.H, wl.W, wl.K, T.direction_angles(wl.D, wl.C, "contiguous"), 1, torch.float32, 0,
             expect="spec")


def test_full_stage1_stride2():
    """S1 at stride 2: the generic kernels (strided gather for dx)."""
    wl = inputs.S1
    run_case(wl.N, wl.C, wl.H, wl.W, wl.K, T.direction_angles(wl.D, wl.C, wl.assign), 2, torch.float32, 0,
             expect="generic")


def test_full_ksweep_bf16():
    wl = inputs.ksweep(31)
    run_case(wl.N, wl.C, wl.H, wl.W, wl.K, T.direction_angles(wl.D, wl.C, wl.assign), 1, torch.bfloat16, 0)


# ---------------------------------------------------------------------------------------
# Bilinear discretisation (NEXT-4): the JIT kernels take weighted taps (each tap
# split over its four neighbours), the generic kernels the expanded table.
@pytest.mark.parametrize("flags", sorted(FLAGS))
@pytest.mark.parametrize("HW", [(56, 56), (37, 45), (14, 14)])
@pytest.mark.parametrize("stride", [1, 2])
def test_bilinear(flags, HW, stride):
    H, W = HW
    angles = T.direction_angles(8, 16, "cycled") if stride == 1 else [17.0, 30.0, 63.5, 90.0, 100.0, 135.0, 170.0, 225.0]
    C = len(angles) if stride != 1 else 16
    K = 15 if stride == 1 else 7
    run_case(2, C, H, W, K, angles, stride, torch.float32, FLAGS[flags], check_det=True, disc="bilinear")


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_bilinear_full_stage1(dtype):
    wl = inputs.S1
    run_case(wl.N, wl.C, wl.H, wl.W, wl.K, T.direction_angles(wl.D, wl.C, wl.assign), 1, dtype, 0,
             disc="bilinear", expect="spec")


# ---------------------------------------------------------------------------------------
def test_plan_module_cache_and_batch_independence():
    """The generated source does not depend on N: a second plan with another batch size (or a
    re-created plan) reuses the compiled modules; its results match the oracle."""
    angles = np.array(T.direction_angles(8, 16, "cycled"))
    p1 = B.Plan(4, 16, 56, 56, 31, angles, device="cuda:0")
    ms1, hit1 = p1.stats()
    p2 = B.Plan(3, 16, 56, 56, 31, angles, device="cuda:0")
    ms2, hit2 = p2.stats()
    assert hit2 == 1 and "module cache hit" in p2.describe(), p2.describe()
    run_case(3, 16, 56, 56, 31, angles, 1, torch.float32, 0, expect="spec")


def test_step_fused_bitwise(monkeypatch):
    """o1d_step with the fused backward (O1D_FUSED=1 at plan creation) gives bitwise the three
    separate calls' results, step after step (the persistent kernels' slots reset)."""
    monkeypatch.setenv("O1D_FUSED", "1")
    wl = inputs.S1
    angles = T.direction_angles(wl.D, wl.C, wl.assign)
    plan = B.Plan(16, wl.C, wl.H, wl.W, wl.K, np.array(angles), device="cuda:0")
    assert "step=fused" in plan.describe(), plan.describe()
    g = torch.Generator(device="cuda:0").manual_seed(2)
    x = torch.rand(16, wl.C, wl.H, wl.W, device="cuda:0", generator=g)
    dy = torch.rand(16, wl.C, wl.H, wl.W, device="cuda:0", generator=g)
    w = torch.rand(wl.C, wl.K, device="cuda:0", generator=g)
    y0, dx0, dW0 = B.forward(plan, x, w), B.backward_input(plan, dy, w), B.backward_weight(plan, x, dy)
    ws = B.workspace(plan)
    y, dx, dW = torch.empty_like(y0), torch.empty_like(dx0), torch.empty_like(dW0)
    for i in range(100):
        B.step(plan, x, w, dy, y, dx, dW, ws)
        if i % 25 == 24:
            torch.cuda.synchronize()
            assert torch.equal(y, y0) and torch.equal(dx, dx0) and torch.equal(dW, dW0), i


@pytest.mark.parametrize("fused", ["0", "1"])
def test_step_host_full_width_windows(fused, monkeypatch):
    """Batch windows of a full-width plan (C=96, N=8: 1-2 planes per table per window, every
    CTA's home table exhausted early): every item is computed once whatever SMs the CTAs land
    on (the scheduler's cross-table stealing)."""
    monkeypatch.setenv("O1D_E2E_CHUNKS", "8")
    monkeypatch.setenv("O1D_FUSED", fused)
    angles = T.direction_angles(8, 96, "cycled")
    plan = B.Plan(8, 96, 56, 56, 31, np.array(angles), device="cuda:0")
    x = torch.from_numpy(inputs.activation(plan.x_shape(), 0)).pin_memory()
    w = torch.from_numpy(inputs.weights(96, 31)).pin_memory()
    dy = torch.from_numpy(inputs.activation(plan.y_shape(), 2)).pin_memory()
    y, dx, dW = torch.empty_like(x).pin_memory(), torch.empty_like(x).pin_memory(), torch.empty_like(w).pin_memory()
    xd, wd, dyd = x.cuda(), w.cuda(), dy.cuda()
    ry, rdx, rdW = B.forward(plan, xd, wd).cpu(), B.backward_input(plan, dyd, wd).cpu(), B.backward_weight(plan, xd, dyd).cpu()
    for _ in range(3):
        B.step_host(plan, x, w, dy, y, dx, dW, B.step_host_workspace(plan))
        assert torch.equal(y, ry) and torch.equal(dx, rdx) and torch.equal(dW, rdW)


def test_torch_library_opcheck():
    """The o1d::* custom ops (schema, fake/meta implementations, autograd registration)
    pass torch.library.opcheck; the autograd formula gives the library passes."""
    from paper_2309_15812_b200 import module as M
    angles = np.array(T.direction_angles(8, 16, "cycled"))
    plan = B.Plan(2, 16, 56, 56, 31, angles, device="cuda:0")
    pid = M.register_plan(plan)
    x = torch.randn(2, 16, 56, 56, device="cuda:0", requires_grad=True)
    w = torch.randn(16, 31, device="cuda:0", requires_grad=True)
    dy = torch.randn(2, 16, 56, 56, device="cuda:0")
    torch.library.opcheck(torch.ops.o1d.forward.default, (x, w, pid))
    torch.library.opcheck(torch.ops.o1d.backward_input.default, (dy, w.detach(), pid))
    torch.library.opcheck(torch.ops.o1d.backward_weight.default, (x.detach(), dy, pid))
    torch.library.opcheck(torch.ops.o1d.backward.default, (x.detach(), dy, w.detach(), pid))
    y = M.oriented1d_dwconv(x, w, plan)
    y.backward(dy)
    assert torch.equal(x.grad, B.backward_input(plan, dy, w.detach()))
    assert torch.equal(w.grad, B.backward_weight(plan, x.detach(), dy))


# small-plane kernels (H, W <= 14, even H*W): 32-plane items, compile-time block positions with
# the out-of-image (output, tap) pairs dropped; partial last groups (N not a multiple of 32),
# ragged blocks, K up to 63 (taps that never reach the image), both activation widths
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("HW,N,K,assign", [((14, 14), 33, 31, "cycled"), ((14, 14), 70, 63, "contiguous"),
                                           ((12, 14), 5, 15, "cycled"), ((8, 8), 40, 7, "contiguous"),
                                           ((6, 4), 3, 31, "cycled"), ((14, 10), 32, 27, "cycled"),
                                           ((2, 2), 2, 7, "cycled"), ((7, 14), 9, 31, "contiguous"),
                                           ((7, 7), 70, 15, "contiguous"), ((7, 9), 33, 31, "cycled"),
                                           ((5, 3), 4, 7, "cycled"), ((1, 1), 3, 5, "cycled")])
def test_small_planes(dtype, HW, N, K, assign):
    C = 16
    angles = B.direction_angles(8, C, assign)
    run_case(N, C, HW[0], HW[1], K, angles, dtype=dtype, check_det=True, expect="spec-small")


@pytest.mark.parametrize("angle_set", sorted(SPEC_SETS))
def test_small_planes_angle_sets(angle_set):
    angles = SPEC_SETS[angle_set]
    run_case(3, len(angles), 14, 14, 31, angles, expect="spec-small")


@pytest.mark.parametrize("disc", ["shear", "bilinear"])
def test_small_planes_discretizations(disc):
    angles = B.direction_angles(8, 16, "cycled")
    run_case(35, 16, 14, 14, 31, angles, disc=disc, expect="spec-small")


@pytest.mark.parametrize("shape", [(2, 16, 56, 56, 31), (33, 16, 14, 14, 31), (3, 8, 40, 48, 15), (70, 16, 14, 14, 63)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_outputs_fully_written(shape, dtype):
    """Every output element is written by the kernels (the TMA box/band stores included: the
    compute-sanitizer initcheck does not track bulk-async writes, profiles/r2/sanitizer_r2.txt):
    outputs pre-filled with NaN come back finite and dW is overwritten, never accumulated."""
    N, C, H, W, K = shape
    plan = B.Plan(N, C, H, W, K, B.direction_angles(8, C, "cycled"), dtype=dtype, device="cuda:0")
    assert plan.describe().startswith("spec"), plan.describe()
    x = torch.randn(N, C, H, W, device="cuda").to(dtype)
    dy = torch.randn(N, C, plan.P, plan.Q, device="cuda").to(dtype)
    w = torch.randn(C, K, device="cuda")
    y = torch.full_like(dy, float("nan"))
    dx = torch.full_like(x, float("nan"))
    dW = torch.full_like(w, float("nan"))
    ws = torch.full((B.workspace(plan).numel(),), float("nan"), device="cuda")
    B.forward(plan, x, w, y)
    B.backward_input(plan, dy, w, dx)
    B.backward_weight(plan, x, dy, dW, ws)
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all() and torch.isfinite(dx.float()).all() and torch.isfinite(dW).all()


@pytest.mark.parametrize("HW,K,stride", [((56, 56), 31, 1), ((14, 14), 27, 1), ((7, 7), 15, 1), ((28, 28), 31, 1),
                                         ((30, 30), 5, 2)])
def test_block1d_parity_vs_masked_conv2d(HW, K, stride):
    """A ConvNeXt-1D block (oriented dw -> LN -> pw 4C -> GELU -> pw -> layer scale -> residual,
    P:1386) through liboriented1d vs the same block with the dw layer as torch's f64 conv2d with
    the masked KxK kernel built from the oracle's exact taps (the oracle's own pin):
    output, input gradient and every parameter gradient (incl. dW) agree."""
    from paper_2309_15812_b200 import convnext1d
    torch.manual_seed(0)
    C, N = 16, 3
    blk = convnext1d.Block1D(C, K, 8, 90.0).cuda()
    if stride != 1:  # the stem's strided layer inside the same block structure
        blk.dw = convnext1d.make_dw(C, K, angles=list(B.direction_angles(8, C, "cycled")), stride=stride)
        blk = blk.cuda()
    blk.gamma.data.fill_(0.5)
    x = torch.randn(N, C, *HW, device="cuda:0", requires_grad=True)
    out = blk(x) if stride == 1 else blk.pw2(torch.nn.functional.gelu(blk.pw1(blk.norm(blk.dw(x).permute(0, 2, 3, 1)))))
    g = torch.randn_like(out)
    (out * g).sum().backward()
    # reference: f64, masked KxK conv2d with the exact taps
    ang = blk.dw.angles_deg
    oh, ow = T.taps_table(K, K // 2, list(ang))
    Wm = torch.zeros(C, 1, K, K, dtype=torch.float64)
    wd = blk.dw.weight.detach().double().cpu()
    for c in range(C):
        for k in range(K):
            Wm[c, 0, K // 2 + oh[c][k], K // 2 + ow[c][k]] += wd[c, k]
    Wm = Wm.cuda().requires_grad_(True)
    xr = x.detach().double().requires_grad_(True)
    ref = {n: p.detach().double().clone().requires_grad_(True) for n, p in blk.named_parameters() if not n.startswith("dw")}
    y = torch.nn.functional.conv2d(xr, Wm, stride=stride, padding=K // 2, groups=C).permute(0, 2, 3, 1)
    y = torch.nn.functional.layer_norm(y, (C,), ref["norm.weight"], ref["norm.bias"], 1e-6)
    y = torch.nn.functional.linear(torch.nn.functional.gelu(torch.nn.functional.linear(y, ref["pw1.weight"], ref["pw1.bias"])),
                                   ref["pw2.weight"], ref["pw2.bias"])
    outr = xr + (ref["gamma"] * y).permute(0, 3, 1, 2) if stride == 1 else y
    (outr * g.double()).sum().backward()

    def rel(a, b):
        return float((a.double() - b).abs().max() / max(float(b.abs().max()), 1e-30))
    assert rel(out, outr) <= 1e-4
    assert rel(x.grad, xr.grad) <= 1e-4
    dWr = torch.stack([torch.stack([Wm.grad[c, 0, K // 2 + oh[c][k], K // 2 + ow[c][k]] for k in range(K)]) for c in range(C)])
    assert rel(blk.dw.weight.grad, dWr) <= 1e-4
    for n, p in blk.named_parameters():
        if not n.startswith("dw"):
            if p.grad is None:  # (the strided variant has no residual / layer scale)
                assert ref[n].grad is None, n
                continue
            assert rel(p.grad, ref[n].grad) <= 1e-4, n


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_small_planes_repeated_bitwise(dtype):
    """The small-plane kernels at the K-sweep shape: 40 back-to-back launches of every pass give
    bitwise-identical results (dynamic scheduling, slot reuse, PDL overlap between launches)."""
    N, C, H, W, K = 128, 384, 14, 14, 31
    plan = B.Plan(N, C, H, W, K, B.direction_angles(8, C, "cycled"), dtype=dtype, device="cuda:0")
    assert plan.describe().startswith("spec-small"), plan.describe()
    x = torch.from_numpy(inputs.activation((N, C, H, W), 0)).to("cuda:0", dtype)
    dy = torch.from_numpy(inputs.activation((N, C, H, W), 2)).to("cuda:0", dtype)
    w = torch.from_numpy(inputs.weights(C, K, 1)).cuda()
    ws = B.workspace(plan)
    y0, dx0, dW0 = B.forward(plan, x, w), B.backward_input(plan, dy, w), B.backward_weight(plan, x, dy, ws=ws)
    y, dx, dW = torch.empty_like(y0), torch.empty_like(dx0), torch.empty_like(dW0)
    bad = 0
    for _ in range(40):
        B.forward(plan, x, w, y)
        B.backward_input(plan, dy, w, dx)
        B.backward_weight(plan, x, dy, dW, ws)
        torch.cuda.synchronize()
        bad += int(not (torch.equal(y, y0) and torch.equal(dx, dx0) and torch.equal(dW, dW0)))
    assert bad == 0, bad


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("shape", [(4, 16, 28, 28, 31, "cycled"), (3, 8, 36, 28, 15, "contiguous"),
                                   (2, 8, 20, 44, 31, "cycled"), (5, 16, 28, 28, 7, "contiguous")])
def test_flat_16bit_planes(shape, dtype):
    """16-bit planes whose rows are not 16-byte multiples (ConvNeXt stage 2: 28 x 2 B) on the specialised
    kernels through flat TMA views (planes as rows of 8 elements) and the element-to-(row, column) widening."""
    N, C, H, W, K, assign = shape
    angles = B.direction_angles(8, C, assign)
    plan, errs = run_case(N, C, H, W, K, angles, dtype=dtype, check_det=True, expect="spec")
    assert "spec-small" not in plan.describe()


def test_disk_cubin_cache(tmp_path):
    """The on-disk cubin cache: a second process building the same plan loads the compiled modules from
    O1D_CACHE_DIR instead of running NVRTC (plan creation several times faster) and computes bitwise
    the same outputs; a damaged cache entry is recompiled."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2309_15812_b200 import binding as B, inputs
ang = B.direction_angles(8, 16, "cycled")
plan = B.Plan(2, 16, 56, 56, 31, ang, device="cuda:0")
x = torch.from_numpy(inputs.activation((2, 16, 56, 56), 0)).cuda()
w = torch.from_numpy(inputs.weights(16, 31, 1)).cuda()
y = B.forward(plan, x, w)
dW = B.backward_weight(plan, x, y)
torch.cuda.synchronize()
print(json.dumps({"ms": plan.stats()[0], "y": float(y.double().sum()), "dW": dW.double().cpu().numpy().tolist()}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {**os.environ, "O1D_CACHE_DIR": str(tmp_path / "cache")}

    def run():
        out = subprocess.run([sys.executable, "-c", code, root], capture_output=True, text=True, env=env, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        return json.loads(out.stdout.strip().splitlines()[-1])

    first = run()
    files = sorted(os.listdir(tmp_path / "cache"))
    assert any(f.endswith(".cubin") for f in files) and any(f.endswith(".log") for f in files), files
    second = run()
    assert second["y"] == first["y"] and second["dW"] == first["dW"]
    assert second["ms"] < first["ms"] / 3, (first["ms"], second["ms"])
    for f in files:  # damage every cubin: the next process must recompile and still be right
        if f.endswith(".cubin"):
            (tmp_path / "cache" / f).write_bytes(b"not a cubin")
    third = run()
    assert third["y"] == first["y"] and third["dW"] == first["dW"]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_many_pair_layout_repeated_bitwise(dtype):
    """Layouts with more than 4 pairs per CTA (28 x 28 planes: one warp per pair, producers serving
    several pairs) over 150 launches -- every scheduler launch slot reused twice: outputs and dW stay
    bitwise equal to the first launch (no counter left behind or overwritten by an exhausted producer)."""
    N, C, H, W, K = 64, 32, 28, 28, 31
    angles = B.direction_angles(8, C, "cycled")
    plan = B.Plan(N, C, H, W, K, angles, dtype=dtype, device="cuda:0")
    assert plan.describe().startswith("spec-v2"), plan.describe()
    x = torch.from_numpy(inputs.activation((N, C, H, W), 0)).to("cuda:0", dtype)
    dy = torch.from_numpy(inputs.activation((N, C, H, W), 2)).to("cuda:0", dtype)
    w = torch.from_numpy(inputs.weights(C, K, 1)).cuda()
    y0, dx0, dW0 = B.forward(plan, x, w), B.backward_input(plan, dy, w), B.backward_weight(plan, x, dy)
    y, dx, dW = torch.empty_like(y0), torch.empty_like(dx0), torch.empty_like(dW0)
    ws = B.workspace(plan)
    bad = 0
    for _ in range(150):
        y.fill_(float("nan")), dx.fill_(float("nan")), dW.fill_(float("nan"))
        B.forward(plan, x, w, y)
        B.backward_input(plan, dy, w, dx)
        B.backward_weight(plan, x, dy, dW, ws)
        bad += int(not (torch.equal(y, y0) and torch.equal(dx, dx0) and torch.equal(dW, dW0)))
    torch.cuda.synchronize()
    assert bad == 0, bad
