"""One-screen summary of a bench.py JSON line (tools/gpu_check.sh)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])


def brief(d, ind=""):
    pp = {k: round(v * 1000, 1) for k, v in d.get("per_pass_ms", {}).items()}
    pi = {k[:6]: round(v * 1000, 1) for k, v in d.get("per_pass_ms_isolated", {}).items()}
    r = d.get("roofline", {})
    print(f"{ind}value {d.get('value', 0):.0f} GB/s  step {d.get('ms_per_step', 0) * 1000:.1f} us  per-pass us {pp}  "
          f"roof {r.get('kernel')} {r.get('bound')} frac {r.get('frac', 0):.3f} (isolated {r.get('frac_isolated', 0):.3f} {pi})  plan {d.get('plan_create_ms', 0):.0f} ms")


brief(d)
for k in ("bf16", "bilinear"):
    if k in d and "error" not in d[k]:
        brief(d[k], f"  {k}: ")
    elif k in d:
        print(k, d[k])
if "convnext_t_1d_train" in d:
    m = d["convnext_t_1d_train"]
    print("  convnext:", m.get("value"), m.get("unit"), m.get("ms_per_step"), m.get("oriented_share", ""))
if "e2e" in d and d["e2e"]:
    print("  e2e:", round(d["e2e"]["value"], 1), "GB/s; clocks", d.get("clocks"))
