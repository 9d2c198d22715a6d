"""One-GPU emulation of the DIRECT transport at C5 scale (dev tool; a measurement of the product
kernels, NOT a multi-GPU bench number).  Launch with torchrun: R processes share cuda:0.

Every rank builds its PJDS_TRANSPORT_DIRECT handle (one pJDS matrix over its rows; nonlocal
columns address the owners' CUDA-IPC mapped x windows), then
  1. ranks take turns timing their fused kernel ALONE on the GPU (CUDA events, `reps` launches):
     remote gathers hit other processes' memory on the same GPU, so NVLink latency/bandwidth is
     not modelled -- the HBM bytes are (the per-rank HBM traffic of the design);
  2. all ranks run `calls` full pjds_dist_spmv calls concurrently (ready/done flags, window), the
     whole job on one GPU: total time vs the sum of the kernels = protocol overhead;
  (correctness of the same path is covered by tests/test_gpu_fake_nccl.py against the oracle; this
  tool only checks that y is finite -- dev tools do not import oracle/).
R = 1 also times the plain single-GPU kernel on the same matrix (the T_1 of the efficiency).
Prints one JSON line on rank 0.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import inputs  # noqa: E402
import paper_1112_5588_b200 as pj  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 10
BR = int(sys.argv[4]) if len(sys.argv) > 4 else 32  # block rows of the DIRECT matrix and of T_1
rank, R = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(0)
dist.init_process_group("gloo")
SEG = {"C1": 1024, "C3": 15504, "C5": 142506}[cfg]
g = inputs.Generator.from_config(cfg)
n = g.n
nb = n // SEG
offs = np.array([(nb * r // R) * SEG for r in range(R + 1)], np.int64)
offs[-1] = n
lo, hi = int(offs[rank]), int(offs[rank + 1])
rp, col, val = g.crs(lo, hi)
x_loc = inputs.vector(hi - lo, i0=lo)
D = pj.DistPjds.create(n, offs, rp, col, val, permuted=True, transport="direct", block_rows=BR)
del col, val
w = D.x_window()
D.to_permuted(w, torch.from_numpy(x_loc).cuda())
A = D.parts()[0]
y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")


def timeit(fn, k):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3  # us


t_kernel = None
for r in range(R):
    dist.barrier()
    if r == rank:
        t_kernel = timeit(lambda: A.spmv(y, w), reps)
    dist.barrier()
# whole job, all ranks concurrently on the one GPU
dist.barrier()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
D.spmv(y, w)
torch.cuda.synchronize()
dist.barrier()
e0.record()
for _ in range(calls):
    D.spmv(y, w)
e1.record()
torch.cuda.synchronize()
t_job = e0.elapsed_time(e1) / calls * 1e3
timed_out = D.p2p_timed_out()
finite = bool(torch.isfinite(y).all().item())
x_full = inputs.vector(n) if R == 1 else None
t_plain = None
if R == 1:
    rp1, col1, val1 = g.crs()
    P = pj.PjdsMatrix.from_crs(n, rp1, col1, val1, block_rows=BR, symmetric=True)
    del col1, val1
    xp = torch.empty(n, dtype=torch.float64, device="cuda")
    P.to_permuted(xp, torch.from_numpy(x_full).cuda())
    yp = torch.empty_like(xp)
    t_plain = timeit(lambda: P.spmv(yp, xp), reps)
info = D.info
rec = {"rank": rank, "t_kernel_us": round(t_kernel, 1), "t_job_us": round(t_job, 1), "finite": finite,
       "timed_out": timed_out, "halo": info["halo"], "nnz_nonlocal": info["nnz_nonlocal_part"],
       "n_loc": hi - lo, "t_plain_us": round(t_plain, 1) if t_plain else None}
recs = [None] * R
dist.all_gather_object(recs, rec)
if rank == 0:
    tk = [r_["t_kernel_us"] for r_ in recs]
    print(json.dumps({"config": cfg, "R": R, "block_rows": BR, "t_kernel_max_us": max(tk), "t_kernel_sum_us": round(sum(tk), 1),
                      "t_job_one_gpu_us": recs[0]["t_job_us"],
                      "protocol_overhead_per_call_us": round(recs[0]["t_job_us"] - sum(tk), 1),
                      "all_finite": all(r_["finite"] for r_ in recs),
                      "any_timeout": any(r_["timed_out"] for r_ in recs), "ranks": recs}), flush=True)
dist.barrier()
D.close()
dist.destroy_process_group()
