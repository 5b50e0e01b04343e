"""Repeat-launch consistency check (diagnostics): many back-to-back steps without host syncs
must give bitwise the results of the first step (scheduler slots, counter resets, PDL)."""
import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2309_15812_b200 import binding as B, inputs
wl = inputs.S1
ang = B.direction_angles(wl.D, wl.C, wl.assign)
plan = B.Plan(wl.N, wl.C, wl.H, wl.W, wl.K, ang, device="cuda:0")
x = torch.randn(wl.N, wl.C, wl.H, wl.W, device="cuda"); dy = torch.randn_like(x)
w = torch.randn(wl.C, wl.K, device="cuda"); ws = B.workspace(plan)
y0 = B.forward(plan, x, w).clone(); dx0 = B.backward_input(plan, dy, w).clone(); dW0 = B.backward_weight(plan, x, dy, ws=ws).clone()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
ys = [torch.empty_like(y0) for _ in range(n)]
dxs = [torch.empty_like(dx0) for _ in range(4)]
dWs = [torch.empty_like(dW0) for _ in range(n)]
for i in range(n):
    B.forward(plan, x, w, ys[i]); B.backward_input(plan, dy, w, dxs[i % 4]); B.backward_weight(plan, x, dy, dWs[i], ws)
torch.cuda.synchronize()
bad = [i for i in range(n) if not (torch.equal(ys[i], y0) and torch.equal(dWs[i], dW0))]
print("steps", n, "mismatching steps:", len(bad), bad[:20])
