"""Executed-instruction mix (per plane) and top stall sites of one kernel in an ncu report."""
import collections, csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
planes = float(sys.argv[3]) if len(sys.argv) > 3 else 6144.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if r and r[0].startswith("0x"):
        data.append(r)
    elif data:
        break
I = lambda x: int(x) if x.isdigit() else 0
c, w = collections.Counter(), collections.Counter()
for r in data:
    t = r[iS].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    c[op] += I(r[iE])
    w[op] += I(r[iW])
tot = sum(c.values())
print("instructions per plane", round(tot / planes, 1))
print("mix:", ", ".join(f"{k} {v / planes:.0f}" for k, v in c.most_common(16)))
print("stall samples by opcode:", ", ".join(f"{k} {v}" for k, v in w.most_common(10)))
