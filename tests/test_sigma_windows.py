"""NEXT-2: sort scope sigma -- rows sorted only within windows of sigma rows, each
window a pJDS matrix of its own (the sliced-ELLPACK idea).  Oracle pins:
sigma >= n reproduces the paper's global pJDS; every window keeps its rows; the stored slots
reproduce the CRS entry multiset; padding only grows as sigma shrinks.  Library: bit-exact against
the oracle on the host; GPU: parity (O2 + FMA chain) for both bases and all variants."""
from collections import Counter

import numpy as np
import pytest

import inputs
import oracle
from oracle import convert


def entries_from_windows(P, n, rp):
    """Independent reconstruction: walk every real row's slots through its window's jagged columns.
    Returns (entry multiset, mask of the slots that hold real entries)."""
    got = Counter()
    used = np.zeros(P["stored"], bool)
    sigma = P.get("sigma", P["n_pad"])
    for k in range(n):
        w = k // sigma
        cs = P["col_start"][P["wcs_off"][w]:P["wcs_off"][w + 1]]
        kk = P["wstart"][w] + (k - w * sigma)
        r = int(P["perm"][k])
        for j in range(int(rp[r + 1] - rp[r])):
            off = int(cs[j] + kk)
            assert not used[off]
            used[off] = True
            got[(r, int(P["col"][off]), float(P["val"][off]))] += 1
    return got, used


@pytest.mark.parametrize("kind,n", [("random", 5000), ("empty_rows", 3100), ("clustered", 4096)])
def test_oracle_windows_pins(kind, n):
    _, rp, col, val = inputs.small(kind, n, seed=3)
    G = convert.pjds_reference(n, rp, col, val, b_r=32)
    W0 = convert.pjds_windows_reference(n, rp, col, val, b_r=32, sigma=1 << 20)
    for k in ("perm", "block_len", "col_start", "val", "col"):
        assert np.array_equal(G[k], W0[k]), k
    prev = None
    for sigma in (4096, 2048, 1024):
        P = convert.pjds_windows_reference(n, rp, col, val, b_r=32, sigma=sigma)
        # rows never leave their window
        for w0 in range(0, n, sigma):
            assert sorted(P["perm"][w0:w0 + sigma].tolist()) == list(range(w0, min(n, w0 + sigma)))
        # block lengths non-increasing inside each window
        bpw = sigma // 32
        for b0 in range(0, P["n_blocks"], bpw):
            bl = P["block_len"][b0:b0 + bpw]
            assert np.all(bl[:-1] >= bl[1:])
        # entries reproduced exactly; every other slot is padding (+0.0, column 0)
        real = Counter((i, int(col[k]), float(val[k])) for i in range(n) for k in range(rp[i], rp[i + 1]))
        got, used = entries_from_windows(P, n, rp)
        assert got == real
        assert np.all(P["val"][~used] == 0) and np.all(P["col"][~used] == 0)
        assert not np.signbit(P["val"][~used]).any()
        # padding grows as the sort scope shrinks (never below the global sort)
        assert P["stored"] >= G["stored"]
        if prev is not None:
            assert P["stored"] >= prev
        prev = P["stored"]


@pytest.fixture(scope="module")
def pj():
    import build_native
    build_native.build_pjds()
    import paper_1112_5588_b200 as pj
    return pj


@pytest.mark.parametrize("sigma", [1024, 2048, 4096, 0])
@pytest.mark.parametrize("br", [32, 64])
@pytest.mark.parametrize("symmetric", [False, True])
def test_library_windows_bit_exact(pj, sigma, br, symmetric):
    n = 5123
    _, rp, col, val = inputs.small("random", n, seed=sigma + br, max=50)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, host_only=True, sigma=sigma, symmetric=symmetric)
    P = convert.pjds_windows_reference(n, rp, col, val, b_r=br, sigma=sigma, symmetric=symmetric)
    got = A.export()
    for k in ("perm", "block_len", "col_start", "col", "wstart", "wcs_off"):
        assert np.array_equal(got[k], P[k]), k
    assert got["val"].tobytes() == P["val"].tobytes()
    assert A.info["stored"] == P["stored"]


def test_library_rejects_bad_sigma(pj):
    n, rp, col, val = inputs.config_crs("C1")
    with pytest.raises(pj.PjdsError):
        pj.PjdsMatrix.from_crs(n, rp, col, val, host_only=True, sigma=1000)


@pytest.mark.gpu
@pytest.mark.parametrize("sigma", [1024, 8192])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gpu_windows_parity(pj, sigma, dtype):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    for name, src in (("rand", inputs.small("random", 20000, seed=1, max=40, dtype=dtype)),
                      ("C1", inputs.config_crs("C1", dtype=dtype)), ("C4", inputs.config_crs("C4", dtype=dtype))):
        n, rp, col, val = src
        x = inputs.vector(n, dtype)
        y_ref, bound = oracle.spmv_ld(n, rp, col, val, x)
        chain = oracle.spmv_chain(n, rp, col, val, x)
        for sym in (False, True):
            A = pj.PjdsMatrix.from_crs(n, rp, col, val, sigma=sigma, symmetric=sym)
            xt = torch.from_numpy(x).cuda()
            if sym:
                xt = A.to_permuted(torch.empty_like(xt), xt)
            y = torch.empty_like(xt)
            A.spmv(y, xt)
            if sym:
                y = A.from_permuted(torch.empty_like(y), y)
            yh = y.cpu().numpy()
            assert oracle.acceptance(yh, y_ref, bound, np.diff(rp), dtype).all(), (name, sym)
            assert np.array_equal(yh, chain), (name, sym)
