"""Measured RHS re-load factor alpha and DRAM traffic / B_min per config from an ncu launch list
(tools/kbench.py --once order: config x dtype x format).  Dev tool; writes a text table."""
import collections, csv, sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import inputs
import paper_1112_5588_b200 as pj
from paper_1112_5588_b200 import perfmodel as pm
src, out = sys.argv[1], sys.argv[2]
cfgs = sys.argv[3].split(","); dts = sys.argv[4].split(","); fmts = sys.argv[5].split(",")
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    d.setdefault(int(r[h.index("ID")]), {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
labels = [(c, t, f) for c in cfgs for t in dts for f in fmts]
lines = ["# Measured RHS re-load factor alpha (x elements read from DRAM per stored nonzero; ideal 1/N_nzr) and",
         "# DRAM traffic vs algorithmic bytes B_min, from one ncu launch per kernel (cold-ish, serialised).",
         f"# source: {os.path.basename(src)}", "",
         f"{'config':6s} {'prec':4s} {'format':9s} {'us':>9s} {'read GB':>8s} {'write GB':>8s} {'B_min GB':>8s} {'traffic/B_min':>13s} {'alpha':>7s} {'1/N_nzr':>7s} {'DRAM GB/s':>9s}"]
info = {}
for (c, t, f), (i, m) in zip(labels, d.items()):
    sv = 8 if t == "f64" else 4
    br = int(f[4:].rstrip("s")) if f.startswith("pjds") else 32
    if (c, t, br) not in info:
        n, rp, col, val = inputs.config_crs(c, dtype=np.float64 if sv == 8 else np.float32)
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, host_only=True)
        E = pj.EllrMatrix.from_crs(n, rp, col, val, host_only=True)
        info[(c, t, br)] = (n, len(col), A.info, E.info)
    n, nnz, ai, ei = info[(c, t, br)]
    rd, wr, tns = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"], m["gpu__time_duration.sum"]
    bmin = pm.min_bytes(nnz, n, sv)
    if f.startswith("pjds"):
        aux = ai["n_blocks"] * 4 + (ai["width"] + 1) * 8 + (0 if f.endswith("s") else n * 4)
        alpha = pm.measured_alpha(rd, ai["stored"], nnz, n, sv, aux)
    else:  # ELLPACK-R reads only the rows' own entries (rowmax-predicated) plus rowmax
        alpha = pm.measured_alpha(rd, nnz, nnz, n, sv, ei["n_pad"] * 4)
    lines.append(f"{c:6s} {t:4s} {f:9s} {tns/1e3:9.1f} {rd/1e9:8.3f} {wr/1e9:8.3f} {bmin/1e9:8.3f} {(rd+wr)/bmin:13.3f} {alpha:7.3f} {n/nnz:7.3f} {(rd+wr)/tns:9.1f}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
