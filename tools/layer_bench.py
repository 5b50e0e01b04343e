"""Time one oriented layer shape (forward, backward_input, backward_weight; back-to-back launches,
CUDA events) and report GB/s of algorithmic bytes and the kernel family the plan selected.
usage: python tools/layer_bench.py N C H W K stride angle|D dtype [flags]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_15812_b200 import binding as B

N, C, H, W, K, st = (int(v) for v in sys.argv[1:7])
ang = sys.argv[7]
dt = {"f32": torch.float32, "bf16": torch.bfloat16}[sys.argv[8]]
flags = int(sys.argv[9]) if len(sys.argv) > 9 else 0
angles = B.direction_angles(int(ang[1:]), C, "contiguous") if ang.startswith("D") else np.full(C, float(ang))
plan = B.Plan(N, C, H, W, K, angles, stride=st, dtype=dt, flags=flags, device="cuda:0")
x = torch.randn(N, C, H, W, device="cuda").to(dt)
dy = torch.randn(N, C, plan.P, plan.Q, device="cuda").to(dt)
w = torch.randn(C, K, device="cuda")
ws = B.workspace(plan)
y = torch.empty_like(dy); dx = torch.empty_like(x); dW = torch.empty_like(w)
es = x.element_size()
res = {}
for name, fn, byt in (("forward", lambda: B.forward(plan, x, w, y), (x.numel() + y.numel()) * es),
                      ("backward_input", lambda: B.backward_input(plan, dy, w, dx), (x.numel() + y.numel()) * es),
                      ("backward_weight", lambda: B.backward_weight(plan, x, dy, dW, ws), (x.numel() + y.numel()) * es)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    res[name] = (ms, byt / ms / 1e6)
print(f"N={N} C={C} {H}x{W} K={K} s={st} {ang} {sys.argv[8]}: " +
      ", ".join(f"{k} {v[0] * 1e3:.0f} us {v[1]:.0f} GB/s" for k, v in res.items()) + f" | {plan.describe()[:50]}")
