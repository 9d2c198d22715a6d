"""cuSPARSE CSR SpMV (torch.sparse CSR, torch.mv) on a config matrix, for an ncu capture beside the
pJDS kernel (dev tool; the timed comparison is bench.py's `compare.cusparse_csr`)."""
import argparse
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402

warnings.filterwarnings("ignore", message="Sparse CSR tensor support is in beta")
p = argparse.ArgumentParser()
p.add_argument("--config", default="C5")
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
n, rp, col, val = inputs.config_crs(a.config)
C = torch.sparse_csr_tensor(torch.from_numpy(rp.astype(np.int32)).cuda(), torch.from_numpy(col).cuda(),
                            torch.from_numpy(val).cuda(), size=(n, n), check_invariants=False)
x = torch.from_numpy(inputs.vector(n)).cuda()
for _ in range(a.reps):
    y = torch.mv(C, x)
torch.cuda.synchronize()
print("ok", a.config, n, len(col))
