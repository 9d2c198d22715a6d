"""NEXT-4 workloads: DLR2-shaped (108,396 points, N = 5.4e5,
N_nzr ~ 315, dense 5x5 blocks, Table 1 data reduction 48.0 %) and UHBR-shaped (L129-138: N = 4.5e6,
N_nzr ~ 123).  CPU: the generator reproduces those numbers; GPU: parity of pJDS / ELLPACK-R on them."""
import numpy as np
import pytest

import inputs
import oracle


def test_w4_dlr2_shape():
    g = inputs.Generator.from_config("W4")
    lens = g.rowlen()
    assert g.n == 108396 * 5
    assert 310 < lens.mean() < 320 and lens.max() == 605 and np.all(lens % 5 == 0)
    n_pad = -(-g.n // 32) * 32
    s = np.zeros(n_pad, np.int64)
    s[:g.n] = np.sort(lens)[::-1]
    red = 1 - 32 * s.reshape(-1, 32).max(axis=1).sum() / (n_pad * lens.max())
    assert abs(red - 0.480) < 0.01  # Table 1: 48.0 %


def test_w5_uhbr_shape():
    g = inputs.Generator.from_config("W5")
    assert g.n == 4500000
    lens = g.rowlen(0, 500000)
    assert 118 < lens.mean() < 128 and np.all(lens % 5 == 0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["W4", "W5"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gpu_parity_long_rows(name, dtype):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_1112_5588_b200 as pj
    n, rp, col, val = inputs.config_crs(name, dtype=dtype)
    x = inputs.vector(n, dtype)
    y_ref, bound = oracle.spmv_ld(n, rp, col, val, x)
    chain = oracle.spmv_chain(n, rp, col, val, x)
    for mk in (lambda: pj.PjdsMatrix.from_crs(n, rp, col, val), lambda: pj.EllrMatrix.from_crs(n, rp, col, val)):
        A = mk()
        y = np.empty(n, dtype=dtype)
        yt = torch.empty(n, dtype=torch.float64 if dtype == np.float64 else torch.float32, device="cuda")
        A.spmv(yt, torch.from_numpy(x).cuda())
        y = yt.cpu().numpy()
        assert oracle.acceptance(y, y_ref, bound, np.diff(rp), dtype).all()
        assert np.array_equal(y, chain)
        del A
