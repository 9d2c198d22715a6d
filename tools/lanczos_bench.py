"""Permuted-basis Lanczos driver timing (NEXT-1; dev tool): m steps on a symmetric-valued config,
wall time of the graph launch vs m x the bare pJDS kernel."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import inputs
import paper_1112_5588_b200 as pj
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 50
br = int(sys.argv[3]) if len(sys.argv) > 3 else 32
n, rp, col, val = inputs.config_crs(cfg, symmetric=True)
A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True, block_rows=br)
nnz = len(col)
del rp, col, val
v0 = torch.from_numpy(inputs.vector(n, seed=77)).cuda()
A.lanczos(v0, 2)
torch.cuda.synchronize()
t0 = time.perf_counter()
a, b, steps = A.lanczos(v0, m)
t = time.perf_counter() - t0
y = torch.empty_like(v0)
for _ in range(3): A.spmv(y, v0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(m): A.spmv(y, v0)
e1.record(); torch.cuda.synchronize()
ts = e0.elapsed_time(e1) * 1e-3
ev = pj.tridiag_eigenvalues(a[:steps], b[:steps])
# device span of the Lanczos graph (first kernel start to last kernel end, CUPTI via torch.profiler):
# the wall time above also counts the host setup (vector allocation, graph capture + instantiate)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    A.lanczos(v0, m)
    torch.cuda.synchronize()
kern = [e for e in prof.events() if e.device_type.name == "CUDA" and
        any(k in e.name for k in ("pjds_spmv", "lanczos_update", "reduce_alpha", "reduce_beta", "dot_partials", "init_c0"))]
span = (max(e.time_range.end for e in kern) - min(e.time_range.start for e in kern)) * 1e-6 if kern else float("nan")
busy = {}
for e in kern:
    key = next(k for k in ("pjds_spmv", "lanczos_update", "reduce_alpha", "reduce_beta", "dot_partials", "init_c0") if k in e.name)
    busy[key] = busy.get(key, 0.0) + (e.time_range.end - e.time_range.start) * 1e-6
print(json.dumps({"device_span_per_step_ms": round(span / m * 1e3, 4), "device_overhead_frac": round(span / ts - 1, 3),
                  "kernel_ms_per_step": {k: round(v / m * 1e3, 4) for k, v in busy.items()}, "n_kernels": len(kern)}))
print(json.dumps({"config": cfg, "block_rows": br, "m": m, "steps": steps, "lanczos_s": round(t, 4), "per_step_ms": round(t / m * 1e3, 3),
                  "spmv_only_per_step_ms": round(ts / m * 1e3, 3), "overhead_frac": round(t / ts - 1, 3),
                  "spmv_gflops_in_lanczos": round(2 * nnz * m / t / 1e9, 1), "ritz_min": ev[0], "ritz_max": ev[-1]}))
