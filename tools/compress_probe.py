"""Development probe (not product): does B200 L2 data compression shrink the DRAM traffic of the
pJDS matrix stream?  The jagged col (int32) and val arrays of C3 (permuted basis, b_r 128) are put
in device buffers three ways -- copy-engine H2D, then an SM copy kernel (torch), then read by an SM
reduction -- so that ncu (`--metrics dram__bytes_read.sum,dram__bytes_write.sum,
lts__average_gcomp_input_sector_success_rate.pct -k regex:reduce`) shows whether SM-written data
comes back from DRAM in fewer bytes.  One marker line per launch on stdout."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import inputs
import paper_1112_5588_b200 as pj

n, rp, col, val = inputs.config_crs(os.environ.get("CFG", "C3"))
A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=128, symmetric=True)
e = A.export()
del A, rp, col, val
for name, arr in (("col", e["col"]), ("val", e["val"]), ("zeros", np.zeros(len(e["col"]), np.int32)),
                  ("col_delta", np.diff(e["col"], prepend=0).astype(np.int32))):
    t_ce = torch.from_numpy(arr).cuda()              # written by the copy engine
    t_sm = torch.empty_like(t_ce)
    t_sm.copy_(t_ce)                                 # written by SMs (elementwise copy kernel)
    torch.cuda.synchronize()
    for tag, t in (("ce", t_ce), ("sm", t_sm)):
        print(f"{name} {tag} {t.numel() * t.element_size()} bytes", flush=True)
        s = t.view(torch.int32).sum(dtype=torch.int64)   # SM read of every byte
        torch.cuda.synchronize()
    del t_ce, t_sm
    torch.cuda.empty_cache()
