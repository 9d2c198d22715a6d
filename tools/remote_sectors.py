"""Remote-read volume of the DIRECT transport (dev analysis, CPU only): for rank `r` of C5 at R
ranks, the 32-byte sectors of the owners' x windows its fused kernel gathers, counted once per CTA
(per-SM L1 reuse inside a CTA, none across CTAs: peer memory is not cached in the local L2), for
the owners' window layouts of the two bases: permuted (length-sorted local order) and original.
NVLink bytes = sectors x 32; ideal = halo entries x s_v."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
SEG = 142506
g = inputs.Generator.from_config("C5")
n = g.n
nb = n // SEG
offs = np.array([(nb * q // R) * SEG for q in range(R + 1)], np.int64)
offs[-1] = n
lens_all = g.rowlen()


def sort_perm(lens):  # stable descending by length (pJDS sort): perm[new] = old
    return np.argsort(-lens.astype(np.int64), kind="stable").astype(np.int64)


# window position of every global row in its owner's window, both bases
pos_perm = np.empty(n, np.int64)
for q in range(R):
    lo, hi = offs[q], offs[q + 1]
    p = sort_perm(lens_all[lo:hi])
    inv = np.empty(hi - lo, np.int64)
    inv[p] = np.arange(hi - lo)
    pos_perm[lo:hi] = inv
owner = np.repeat(np.arange(R), np.diff(offs))
lo, hi = offs[rank], offs[rank + 1]
rp, col, _ = g.crs(lo, hi)
m = hi - lo
perm = sort_perm(lens_all[lo:hi])
sorted_pos = np.empty(m, np.int64)
sorted_pos[perm] = np.arange(m)
rows_per_cta = 1024  # 256 threads x R=4 rows
row_of = np.repeat(np.arange(m), np.diff(rp))
remote = (col < lo) | (col >= hi)
c = col[remote].astype(np.int64)
cta = sorted_pos[row_of[remote]] // rows_per_cta
out = {"R": R, "rank": rank, "halo": int(len(np.unique(c))), "remote_gathers": int(len(c))}
sv = 8
for basis, pos in (("permuted", pos_perm[c]), ("original", c - offs[owner[c]])):
    sector = owner[c] * (1 << 30) + pos * sv // 32
    key = cta * (R << 30) + sector
    per_cta = len(np.unique(key))
    out[basis] = {"sectors_per_cta_sum": per_cta, "nvlink_bytes": per_cta * 32,
                  "amplification_vs_halo": round(per_cta * 32 / (out["halo"] * sv), 3),
                  "distinct_sectors": int(len(np.unique(sector)))}
print(json.dumps(out))
