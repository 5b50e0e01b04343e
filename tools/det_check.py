"""Determinism / correctness check of backward_weight on one shape: launches vs an f64 torch reference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_15812_b200 import binding as B, inputs
from oracle import taps as T
N, C, H, W, K = (int(v) for v in sys.argv[1:6])
ang = B.direction_angles(8, C, "cycled")
plan = B.Plan(N, C, H, W, K, ang, device="cuda:0")
x = torch.from_numpy(inputs.activation((N, C, H, W), 0)).cuda()
dy = torch.from_numpy(inputs.activation((N, C, plan.P, plan.Q), 2)).cuda()
oh, ow = T.taps_table(K, K // 2, list(ang))
Wm = torch.zeros(C, 1, K, K, dtype=torch.float64, device="cuda", requires_grad=True)
y = torch.nn.functional.conv2d(x.double(), Wm, padding=K // 2, groups=C)
(y * dy.double()).sum().backward()
ref = torch.stack([torch.stack([Wm.grad[c, 0, K // 2 + oh[c][k], K // 2 + ow[c][k]] for k in range(K)]) for c in range(C)])
den = float(ref.abs().max())
ws = B.workspace(plan)
order = os.environ.get("DET_ORDER", "")
for i in range(int(os.environ.get("DET_RUNS", "8"))):
    if order == "nan":  # workspace pre-filled with NaN: any entry the kernel does not write shows up
        ws.fill_(float("nan"))
    d = B.backward_weight(plan, x, dy, ws=ws)
    torch.cuda.synchronize()
    err = float((d.double() - ref).abs().max()) / den
    if err > 1e-5 or i < 2:
        print("run", i, "normwise err", err, "worst channel", int((d.double() - ref).abs().max(1).values.argmax()))
print(plan.describe()[:60])
