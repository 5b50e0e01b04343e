"""Small cases of every kernel family for compute-sanitizer (memcheck / racecheck / initcheck /
synccheck): spec-v2 (56-wide planes: forward, backward_input, backward_weight, fused backward),
spec-small (14x14 fp32 TMA boxes and bf16 cp.async units), generic (stride 1 and 2).
usage: compute-sanitizer --tool X python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_15812_b200 import binding as B

CASES = [  # N, C, H, W, K, stride, dtype, flags
    (2, 16, 56, 56, 31, 1, torch.float32, 0),
    (1, 8, 40, 48, 15, 1, torch.bfloat16, 0),
    (33, 16, 14, 14, 31, 1, torch.float32, 0),
    (5, 16, 14, 14, 27, 1, torch.bfloat16, 0),
    (2, 8, 30, 23, 7, 1, torch.float32, 0),
    (2, 8, 30, 24, 5, 2, torch.bfloat16, 0),
    (1, 8, 14, 14, 7, 1, torch.float32, B.FLAG_FORCE_GENERIC),
]
sel = sys.argv[1] if len(sys.argv) > 1 else "all"  # all | generic | spec
for (N, C, H, W, K, st, dt, fl) in CASES:
    probe = B.Plan(N, C, H, W, K, B.direction_angles(8, C, "cycled"), stride=st, dtype=dt, flags=fl, device="cuda:0")
    fam = "spec" if probe.describe().startswith("spec") else "generic"
    del probe
    if sel != "all" and sel != fam:
        continue
    ang = B.direction_angles(8, C, "cycled")
    plan = B.Plan(N, C, H, W, K, ang, stride=st, dtype=dt, flags=fl, device="cuda:0")
    x = torch.randn(N, C, H, W, device="cuda").to(dt)
    dy = torch.randn(N, C, plan.P, plan.Q, device="cuda").to(dt)
    w = torch.randn(C, K, device="cuda")
    y = B.forward(plan, x, w)
    dx = B.backward_input(plan, dy, w)
    dW = B.backward_weight(plan, x, dy)
    fdx, fdW = B.backward(plan, x, dy, w)
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all() and torch.isfinite(dx.float()).all() and torch.isfinite(dW).all()
    print(f"ok {N}x{C}x{H}x{W} K={K} s={st} {dt} flags={fl}: {plan.describe()[:40]}", flush=True)
