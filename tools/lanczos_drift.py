"""Dev probe: per-step deviation |alpha_j - alpha_j(oracle)|, |beta_j - beta_j(oracle)| of the GPU
Lanczos driver on the tests' matrices, to set evidence-based tolerances in tests/test_lanczos.py."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1112_5588_b200 as pj  # noqa: E402
from oracle import lanczos as olz  # noqa: E402
from test_lanczos import sym_matrix  # noqa: E402

for dtype in (np.float64, np.float32):
    for name, src in (("rand", sym_matrix(3000, 5)), ("C1", inputs.config_crs("C1", symmetric=True))):
        n, rp, col, val = src
        val = val.astype(dtype)
        v0 = inputs.vector(n, dtype, seed=77)
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
        perm = A.export()["perm"]
        m = 40
        a, b, steps = A.lanczos(torch.from_numpy(v0[perm].copy()).cuda(), m)
        ra, rb = olz.lanczos(n, rp, col, val.astype(np.float64), v0.astype(np.float64), m)
        scale = max(np.abs(ra).max(), np.abs(rb).max())
        print(json.dumps({"dtype": np.dtype(dtype).name, "matrix": name, "steps": int(steps),
                          "da_over_scale": (np.abs(a - ra) / scale).tolist(),
                          "db_over_scale": (np.abs(b - rb) / scale).tolist()}), flush=True)
