import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch, torch.distributed as dist
import inputs, paper_1112_5588_b200 as pj
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29617")
dist.init_process_group("gloo", rank=0, world_size=1)
n, rp, col, val = inputs.config_crs("C3")
A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
D = pj.DistPjds.create(n, np.array([0, n]), rp, col, val, permuted=True)
Al, _ = D.parts()
x = torch.from_numpy(inputs.vector(n)).cuda(); y = torch.empty_like(x)
def t(fn, k=50):
    for _ in range(5): fn()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / k
print(json.dumps({"single": t(lambda: A.spmv(y, x)), "dist": t(lambda: D.spmv(y, x)), "dist_A_loc": t(lambda: Al.spmv(y, x)),
                  "single_info": {k: A.info[k] for k in ("stored", "n_blocks", "width")}, "loc_info": {k: Al.info[k] for k in ("stored", "n_blocks", "width", "flags")}}))
