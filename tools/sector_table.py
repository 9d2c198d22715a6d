"""RHS gather sector amplification and DRAM alpha per (format, b_r, sigma) from an ncu launch list
of `tools/kbench.py --once` (evaluate the sort scope and b_r by measured alpha
and sector amplification).  Dev tool; writes a text table.

  amplification = x-gather 32 B sectors requested at L1 / (nnz * s_v / 32)
  x-gather sectors = l1tex global-load sectors - val/col/aux sectors (stored * (s_v+4) / 32 + aux / 32;
                     ELLPACK-R: the rowmax-predicated entries, nnz * (s_v+4) / 32)
  L2 amplification = the same after L1 (lts sectors from the SM), alpha from DRAM reads (perfmodel).

usage: sector_table.py ncu.csv out.txt CONFIGS DTYPES FMTS SIGMAS
"""
import collections, csv, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs
import paper_1112_5588_b200 as pj
from paper_1112_5588_b200 import perfmodel as pm

src, out = sys.argv[1], sys.argv[2]
cfgs, dts, fmts, sigmas = (s.split(",") for s in sys.argv[3:7])
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    d.setdefault(int(r[h.index("ID")]), {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
labels = [(c, t, f, int(g)) for c in cfgs for t in dts for f in fmts
          for g in (sigmas if f.startswith("pjds") else ["0"])]
assert len(labels) == len(d), (len(labels), len(d))
lines = ["# x-gather sector amplification (32 B sectors per ideal nnz*s_v/32) at L1 and L2, DRAM alpha;",
         "# one ncu launch per kernel (serialised).  source: " + os.path.basename(src), "",
         f"{'config':6s} {'prec':4s} {'format':9s} {'sigma':>8s} {'us':>8s} {'stored':>11s} {'L1 x-sect M':>11s} "
         f"{'ampl L1':>7s} {'ampl L2':>7s} {'alpha':>6s} {'1/Nnzr':>6s} {'DRAM GB':>7s}"]
cache = {}
for (c, t, f, g), m in zip(labels, d.values()):
    sv = 8 if t == "f64" else 4
    if (c, t) not in cache:
        cache[(c, t)] = inputs.config_crs(c, dtype=np.float64 if sv == 8 else np.float32)
    n, rp, col, val = cache[(c, t)]
    nnz = len(col)
    if f.startswith("pjds"):
        br = int(f[4:].rstrip("s"))
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, symmetric=f.endswith("s"), sigma=g, host_only=True)
        i = A.info
        stored = i["stored"]
        aux = i["n_blocks"] * 4 + i["col_start_len"] * 8 + (0 if f.endswith("s") else n * 4)
        del A
    else:
        stored = nnz
        aux = (n + 31) // 32 * 32 * 4
    stream_sect = (stored * (sv + 4) + aux) / 32.0
    ideal = nnz * sv / 32.0
    l1 = m["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]
    l2 = m["lts__t_sectors_srcunit_tex_op_read.sum"]
    rd = m["dram__bytes_read.sum"]
    alpha = pm.measured_alpha(rd, stored, nnz, n, sv, aux)
    lines.append(f"{c:6s} {t:4s} {f:9s} {g:8d} {m['gpu__time_duration.sum'] / 1e3:8.1f} {stored:11d} "
                 f"{(l1 - stream_sect) / 1e6:11.2f} {(l1 - stream_sect) / ideal:7.3f} {(l2 - stream_sect) / ideal:7.3f} "
                 f"{alpha:6.3f} {n / nnz:6.3f} {rd / 1e9:7.3f}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
