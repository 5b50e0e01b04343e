"""Write profiles/traffic.json: DRAM bytes per launch per pass, from an ncu --set full report
(the `traffic` field of bench.py's roofline object)."""
import csv, json, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = {}
order = []
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
    order.append((name, b))
# passes in launch order: stencil (fwd), stencil (bwd_in), wgrad + finalize (bwd_w)
res = {"source": rep, "note": "ncu --set full, one launch each; bytes = dram__bytes_read.sum + dram__bytes_write.sum"}
st = [b for n, b in order if n == "o1d_stencil"]
wg = [b for n, b in order if n == "o1d_wgrad"]
fi = [b for n, b in order if n == "o1d_wgrad_finalize"]
if len(st) >= 2:
    res["forward"], res["backward_input"] = st[0], st[1]
if wg:
    res["backward_weight"] = wg[0] + (fi[0] if fi else 0.0)
json.dump(res, open(out, "w"), indent=1)
print(res)
