"""Property-based (hypothesis) GPU parity: random CRS matrices (empty rows, very long rows,
duplicates, explicit zeros, ragged n) through the default pJDS and ELLPACK-R kernels, both bases,
every b_r step, SP and DP — y equal to the oracle's FMA chain (O3) and within O2."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

import oracle
from test_property_convert import crs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(m=crs(), br=st.sampled_from([32, 64, 96, 128]), sym=st.booleans(), sigma_k=st.sampled_from([0, 1]))
def test_gpu_kernels_match_chain(m, br, sym, sigma_k):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_1112_5588_b200 as pj
    n, rp, col, val = m
    if n == 0:
        return
    x = np.random.default_rng(n).uniform(-1, 1, n).astype(val.dtype)
    tdt = torch.float64 if val.dtype == np.float64 else torch.float32
    sigma = 0 if sigma_k == 0 else int(np.lcm(1024, br))
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, symmetric=sym, sigma=sigma)
    perm = A.export()["perm"]
    y = torch.full((n,), float("nan"), dtype=tdt, device="cuda")
    A.spmv(y, torch.from_numpy(x[perm] if sym else x).cuda())
    yh = y.cpu().numpy()
    if sym:
        yo = np.empty_like(yh)
        yo[perm] = yh
        yh = yo
    chain = oracle.spmv_chain(n, rp, col, val, x)
    assert np.array_equal(yh, chain)
    yl, b = oracle.spmv_ld(n, rp, col, val, x)
    assert oracle.acceptance(yh, yl, b, np.diff(rp), val.dtype).all()
    E = pj.EllrMatrix.from_crs(n, rp, col, val)
    y2 = torch.full((n,), float("nan"), dtype=tdt, device="cuda")
    E.spmv(y2, torch.from_numpy(x).cuda())
    assert np.array_equal(y2.cpu().numpy(), chain)
