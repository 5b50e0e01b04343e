"""Share of the ConvNeXt-1D training step spent in the oriented-conv kernels (torch.profiler,
CUDA kernel time by name).  usage: python tools/model_profile.py [convnext_t_1d] [batch]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_15812_b200 import convnext1d

name = sys.argv[1] if len(sys.argv) > 1 else "convnext_t_1d"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dev = torch.device("cuda", 0)
torch.manual_seed(0)
model = convnext1d.ConvNeXt1D(name).to(dev).to(torch.bfloat16)
for m in convnext1d.oriented_layers(model):
    m.weight.data = m.weight.data.float()
opt = torch.optim.AdamW(model.parameters(), lr=1e-4)
x = torch.randn(B, 3, 224, 224, device=dev).to(torch.bfloat16)
lab = torch.randint(0, 1000, (B,), device=dev)


def step():
    opt.zero_grad(set_to_none=True)
    loss = torch.nn.functional.cross_entropy(model(x).float(), lab)
    loss.backward()
    opt.step()


for _ in range(3):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
tot = defaultdict(float)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
allt = sum(tot.values())
ours = {k: v for k, v in tot.items() if "o1d" in k or "generic" in k or "bwd_weight" in k or "bwd_input" in k}
print(f"total kernel time per step {allt / 3 / 1e3:.2f} ms; oriented-conv kernels {sum(ours.values()) / 3 / 1e3:.2f} ms "
      f"({100 * sum(ours.values()) / allt:.1f}%)")
for k, v in sorted(ours.items(), key=lambda t: -t[1]):
    print(f"  {v / 3 / 1e3:8.3f} ms  {k[:90]}")
print("top other kernels:")
for k, v in sorted(((k, v) for k, v in tot.items() if k not in ours), key=lambda t: -t[1])[:12]:
    print(f"  {v / 3 / 1e3:8.3f} ms  {k[:90]}")
for m in convnext1d.oriented_layers(model):
    for key, p in list(m._plans.items())[:1]:
        print(f"  layer C={m.C} K={m.K} stride={m.stride} x={key[:3]}: {p.describe()[:60]}")
