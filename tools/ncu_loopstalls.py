"""Stall breakdown of one kernel's tap loops (FFMA / FFMA2 / LDS / FADD / MOV sites) vs the rest."""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS, iW = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
sc = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
I = lambda x: int(x) if x.strip().isdigit() else 0
loop = collections.Counter(); rest = collections.Counter(); nl = nr = 0
for r in rows[2:]:
    if not r or not r[0].startswith("0x"): continue
    t = r[iS].split()
    if not t: continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    tgt = loop if op in ("FFMA2", "FFMA", "LDS", "FADD", "MOV", "IMAD") else rest
    for i, n in sc: tgt[n] += I(r[i])
for name, c in (("tap-loop sites", loop), ("other sites", rest)):
    tot = sum(c.values())
    print(f"{name}: {tot} samples;", ", ".join(f"{n} {100*v/tot:.1f}%" for n, v in c.most_common(9)))
