"""Dev tool for the ncu traffic pass: one launch of every kernel the bench line reports (the N=1
headline C5 DP permuted and rows-only, and the per_config table's pJDS (permuted basis) and
ELLPACK-R kernels), each preceded by an NVTX-free marker line on stdout, so that
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:spmv`
yields one row per (config, dtype, format) in this order (tools/make_traffic_json.py)."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import inputs
import paper_1112_5588_b200 as pj

ORDER = [("C5", "f64", "permuted"), ("C5", "f64", "permuted/br128"), ("C5", "f64", "rows"),
         ("C5", "f64", "rows/br128"), ("C5", "f64", "ellr"), ("C5", "f32", "permuted/br128"),
         ("C5", "f32", "ellr")] + [(c, d, f) for c in ("C2", "C3", "C4") for d in ("f64", "f32")
                                   for f in ("permuted", "permuted/br128", "ellr")]
if __name__ == "__main__":
    cache = {}
    for cfg, dt, fmt in ORDER:
        npdt = np.float64 if dt == "f64" else np.float32
        key = (cfg, dt)
        if key not in cache:
            cache.clear()
            cache[key] = inputs.config_crs(cfg, dtype=npdt)
        n, rp, col, val = cache[key]
        x = torch.from_numpy(inputs.vector(n, npdt)).cuda()
        y = torch.empty_like(x)
        if fmt == "ellr":
            M = pj.EllrMatrix.from_crs(n, rp, col, val)
        else:
            base, _, br = fmt.partition("/br")
            M = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=int(br or 32), symmetric=(base == "permuted"))
        M.spmv(y, x)
        torch.cuda.synchronize()
        print(json.dumps({"cfg": cfg, "dtype": dt, "fmt": fmt}), flush=True)
        del M, x, y
        torch.cuda.synchronize()
