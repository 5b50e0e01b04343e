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
l2w = []
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
    order.append((name, b))
    # bytes the SMs wrote into L2 (TMA stores included): the y / dx write-back of a launch can still
    # sit in L2 when the kernel ends, so DRAM writes inside the launch undercount it
    i = hdr.index("lts__t_sectors_srcunit_tex_op_write.sum")
    rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", "")) * scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
    l2w.append((name, rd + 32.0 * float(r[i].replace(",", ""))))
# passes in launch order: stencil (fwd), stencil (bwd_in), wgrad + finalize (bwd_w)
res = {"source": rep, "note": "ncu --set full, one launch each; bytes = dram__bytes_read.sum + dram__bytes_write.sum"}
st = [b for n, b in order if n == "o1d_stencil"]
wg = [b for n, b in order if n == "o1d_wgrad"]
fi = [b for n, b in order if n == "o1d_wgrad_finalize"]
if len(st) >= 2:
    res["forward"], res["backward_input"] = st[0], st[1]
if wg:
    res["backward_weight"] = wg[0] + (fi[0] if fi else 0.0)
st2 = [b for n, b in l2w if n == "o1d_stencil"]
wg2 = [b for n, b in l2w if n == "o1d_wgrad"]
res["dram_read_plus_l2_write"] = {}
if len(st2) >= 2:
    res["dram_read_plus_l2_write"]["forward"], res["dram_read_plus_l2_write"]["backward_input"] = st2[0], st2[1]
if wg2:
    res["dram_read_plus_l2_write"]["backward_weight"] = wg2[0]
json.dump(res, open(out, "w"), indent=1)
print(res)
