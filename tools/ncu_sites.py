"""Top stall sites of one kernel in an ncu report (per SASS instruction, with the dominant reasons)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iA, iS, iW, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
sc = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
I = lambda x: int(x) if x.strip().isdigit() else 0
tot = sum(I(r[iW]) for r in data)
agg = {}
for i, n in sc:
    agg[n] = sum(I(r[i]) for r in data)
print("total samples", tot, "by reason:", ", ".join(f"{n} {v}" for n, v in sorted(agg.items(), key=lambda t: -t[1])[:10]))
for idx, r in sorted(enumerate(data), key=lambda t: -I(t[1][iW]))[:top]:
    rs = sorted(((I(r[i]), n) for i, n in sc), reverse=True)[:3]
    print(f"{idx:6d} {r[iA]} {I(r[iW]):6d} ex={I(r[iE]):8d} {r[iS][:60]:60s}", ", ".join(f"{n}:{v}" for v, n in rs if v))
