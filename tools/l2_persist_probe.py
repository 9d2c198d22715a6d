"""Development probe (not the bench contract): does the L2 set-aside for persisting accesses change
how much of L2 the x gathers (createpolicy evict_last) keep on C5?  Times the default pJDS kernel
(permuted basis) with cudaLimitPersistingL2CacheSize = 0 (the default) and = the device maximum,
for the default tile order and the 2-D phonon-window keys.  --once: one launch per setting (ncu)."""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1112_5588_b200 as pj  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C5")
p.add_argument("--dtype", default="f64")
p.add_argument("--keys", default="none,w4096")
p.add_argument("--limits", default="0,max")
p.add_argument("--reps", type=int, default=30)
p.add_argument("--once", action="store_true")
a = p.parse_args()
SEG = {"C3": 15504, "C5": 142506}
rt = ctypes.CDLL("libcudart.so.12")
dev = 0
mx = ctypes.c_int()
rt.cudaDeviceGetAttribute(ctypes.byref(mx), 108, dev)  # cudaDevAttrMaxPersistingL2CacheSize
l2 = ctypes.c_int()
rt.cudaDeviceGetAttribute(ctypes.byref(l2), 38, dev)  # cudaDevAttrL2CacheSize
print(json.dumps({"l2_bytes": l2.value, "max_persisting_l2_bytes": mx.value}), flush=True)
npdt = np.float64 if a.dtype == "f64" else np.float32
sv = np.dtype(npdt).itemsize
n, rp, col, val = inputs.config_crs(a.config, dtype=npdt)
nnz = len(col)
A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
del col, val
x0 = torch.from_numpy(inputs.vector(n, npdt)).cuda()
x = A.to_permuted(torch.empty_like(x0), x0)
y = torch.empty_like(x)
bmin = nnz * (sv + 4) + 2 * n * sv
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
for kspec in a.keys.split(","):
    if kspec == "none":
        A.set_tile_keys(None)
    else:
        W, P = int(kspec[1:]), SEG[a.config]
        r = np.arange(n, dtype=np.int64)
        A.set_tile_keys(((r % P) // W) * n + r)
        del r
    for lim in a.limits.split(","):
        v = mx.value if lim == "max" else int(lim)
        st = rt.cudaDeviceSetLimit(0x06, ctypes.c_size_t(v))  # cudaLimitPersistingL2CacheSize
        got = ctypes.c_size_t()
        rt.cudaDeviceGetLimit(ctypes.byref(got), 0x06)
        if a.once:
            A.spmv(y, x)
            torch.cuda.synchronize()
            continue
        t_w = time.perf_counter()
        while time.perf_counter() - t_w < 0.2:
            for _ in range(5):
                A.spmv(y, x)
            torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            A.spmv(y, x)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / a.reps * 1e-3
        print(json.dumps({"cfg": a.config, "dtype": a.dtype, "keys": kspec, "persist_limit": got.value, "set_status": st,
                          "us": round(t * 1e6, 1), "frac": round(bmin / t / 1e9 / peak, 4)}), flush=True)
