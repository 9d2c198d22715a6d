"""Dev probe for the rows-only timing discrepancy (kbench 2.40 ms vs bench compare leg 2.19 ms on C5
DP): times one rows-only handle (a) alone, kbench-style, then (b) after a permuted-basis handle of
the same matrix was built and run (bench-style), with fresh and with reused x / y buffers."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import inputs
import paper_1112_5588_b200 as pj
from bench import ClockSampler

CLK = {}


def timed(fn, k=20, tag=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as c:
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
    if tag:
        CLK[tag] = c.summary()
    return e0.elapsed_time(e1) / k * 1e3


n, rp, col, val = inputs.config_crs("C5")
x = torch.from_numpy(inputs.vector(n)).cuda()
y = torch.empty_like(x)
pj.bw_probe(1 << 30, 20)
B = pj.PjdsMatrix.from_crs(n, rp, col, val)
out = {"alone_fresh": timed(lambda: B.spmv(y, x), tag="alone_fresh")}
y2 = torch.empty_like(x)
out["alone_other_y"] = timed(lambda: B.spmv(y2, x), tag="alone_other_y")
A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
xp = A.to_permuted(torch.empty_like(x), x)
out["permuted_after"] = timed(lambda: A.spmv(y, xp), 200, tag="permuted_after")
out["rows_after_permuted_run"] = timed(lambda: B.spmv(y, x), tag="rows_after_permuted_run")
del B
torch.cuda.synchronize()
B2 = pj.PjdsMatrix.from_crs(n, rp, col, val)
out["rows_rebuilt_after_permuted"] = timed(lambda: B2.spmv(y, x), tag="rows_rebuilt_after_permuted")
for order in (1, 3):
    pj.lib().pjds_set_tile_order(order)
    out[f"rows_order{order}"] = timed(lambda: B2.spmv(y, x), 40, tag=f"rows_order{order}")
    out[f"permuted_order{order}"] = timed(lambda: A.spmv(y, xp), 40, tag=f"permuted_order{order}")
pj.lib().pjds_set_tile_order(2)
print(json.dumps({k: {"us": round(v, 1), "sm_mhz": CLK.get(k, {}).get("sm_mhz"),
                       "reasons": CLK.get(k, {}).get("reasons")} for k, v in out.items()}), flush=True)
