"""Run each pass of a specialised plan separately (debug helper).
usage: python tools/debug_spec.py N C H W K passes(0,1,2,3) dtype(f32|bf16|f16)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2309_15812_b200 import binding as B
N, C, H, W, K = [int(a) for a in sys.argv[1:6]] if len(sys.argv) > 5 else (2, 16, 56, 56, 31)
passes = sys.argv[6].split(",") if len(sys.argv) > 6 else ["0", "1", "2"]
dt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[sys.argv[7] if len(sys.argv) > 7 else "f32"]
ang = B.direction_angles(8, C, "cycled")
plan = B.Plan(N, C, H, W, K, ang, dtype=dt, device="cuda:0")
print(plan.describe(), flush=True)
x = torch.randn(N, C, H, W, device="cuda").to(dt)
w = torch.randn(C, K, device="cuda")
for p in passes:
    if p == "0":
        y = B.forward(plan, x, w)
    elif p == "1":
        dx = B.backward_input(plan, x, w)
    elif p == "2":
        dW = B.backward_weight(plan, x, x)
    else:
        B.backward(plan, x, x, w)
    torch.cuda.synchronize()
    print("pass", p, "ok", flush=True)
