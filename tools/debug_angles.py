"""Forward with a single angle on all channels, one process per angle (debug helper)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np, torch
    from paper_2309_15812_b200 import binding as B
    a, H, W = float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    plan = B.Plan(2, 8, H, W, 31, np.full(8, a), device="cuda:0")
    x = torch.randn(2, 8, H, W, device="cuda"); w = torch.randn(8, 31, device="cuda")
    B.forward(plan, x, w); torch.cuda.synchronize()
    print("ok", a, H, W, plan.describe()[:60])
else:
    for HW in [(56, 56)]:
        for i in range(8):
            r = subprocess.run([sys.executable, __file__, "child", str(i * 22.5), str(HW[0]), str(HW[1])],
                               capture_output=True, text=True, env={**os.environ, "O1D_TMA_DEBUG": "1"})
            print(i * 22.5, "rc", r.returncode, (r.stdout + r.stderr).strip().splitlines()[-3:])
