"""Worker for tests/test_gpu_fake_nccl.py::test_direct_c5_sampled: one rank of the DIRECT transport on
the full C5 matrix (the bench workload; all ranks share cuda:0), permuted basis, x in the window;
2,000 sampled rows of y per rank compared bitwise with the oracle's FMA chain (the DIRECT result is
the unsplit chain).  Prints one JSON line per rank."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1112_5588_b200 as pj  # noqa: E402

rank, R = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
SEG = 142506
g = inputs.Generator.from_config("C5")
n = g.n
nb = n // SEG
offs = np.array([(nb * r // R) * SEG for r in range(R + 1)], np.int64)
offs[-1] = n
lo, hi = int(offs[rank]), int(offs[rank + 1])
rp, col, val = g.crs(lo, hi)
D = pj.DistPjds.create(n, offs, rp, col, val, permuted=True, transport="direct")
del col, val
w = D.x_window()
D.to_permuted(w, torch.from_numpy(inputs.vector(hi - lo, i0=lo)).cuda())
y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
for _ in range(3):
    D.spmv(y, w)
y0 = D.from_permuted(torch.empty_like(y), y).cpu().numpy()
timed_out = D.p2p_timed_out()
rows = np.unique(np.concatenate([np.random.default_rng(rank).integers(0, hi - lo, 2000), [0, hi - lo - 1]]))
x_full = inputs.vector(n)
srp = np.zeros(len(rows) + 1, np.int64)
sc, sv = [], []
for a, i in enumerate(rows):
    _, cc, vv = g.crs(lo + int(i), lo + int(i) + 1)
    sc.append(cc)
    sv.append(vv)
    srp[a + 1] = srp[a] + len(cc)
sc, sv = np.concatenate(sc), np.concatenate(sv)
chain = oracle.spmv_chain(len(rows), srp, sc, sv, x_full)
y_ref, bound = oracle.spmv_ld(len(rows), srp, sc, sv, x_full)
rec = {"rank": rank, "rows": int(len(rows)), "bitwise": bool(np.array_equal(y0[rows], chain)),
       "o2": bool(oracle.acceptance(y0[rows], y_ref, bound, np.diff(srp), np.float64).all()),
       "finite": bool(np.isfinite(y0).all()), "timed_out": bool(timed_out), "halo": D.info["halo"]}
os.write(1, (json.dumps(rec) + "\n").encode())
dist.barrier()
D.close()
dist.destroy_process_group()
