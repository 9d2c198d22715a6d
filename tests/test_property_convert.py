"""Property-based (hypothesis) check of the library's host conversion (PJDS_HOST_ONLY, no GPU)
against the independent oracle converters on random CRS matrices: random n (incl. 0 and ragged
tails), row-length distributions with empty and very long rows, duplicates, explicit zeros,
block_rows, sort scope sigma, both bases and both precisions.  Bit-exact arrays."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from oracle import convert

pj = pytest.importorskip("paper_1112_5588_b200")


@st.composite
def crs(draw):
    n = draw(st.integers(0, 2600))
    seed = draw(st.integers(0, 2 ** 31 - 1))
    mode = draw(st.sampled_from(["uniform", "skewed", "sparse", "one_long"]))
    rng = np.random.default_rng(seed)
    if n == 0:
        lens = np.zeros(0, np.int64)
    elif mode == "uniform":
        lens = rng.integers(0, 12, n)
    elif mode == "skewed":
        lens = np.minimum(rng.geometric(0.15, n) - 1, n)
    elif mode == "sparse":
        lens = (rng.random(n) < 0.1) * rng.integers(1, 5, n)
    else:
        lens = rng.integers(0, 3, n)
        lens[rng.integers(0, n)] = min(n, 1500)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    col = rng.integers(0, max(n, 1), int(rp[-1])).astype(np.int32)  # duplicates allowed
    dtype = draw(st.sampled_from([np.float64, np.float32]))
    val = rng.uniform(-1, 1, int(rp[-1])).astype(dtype)
    val[rng.random(len(val)) < 0.05] = 0.0  # explicit zeros are stored entries
    return n, rp, col, val


@settings(max_examples=120, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(m=crs(), br=st.sampled_from([32, 64, 96, 128]), sym=st.booleans(),
       sigma_k=st.sampled_from([0, 1, 2, 3]))
def test_host_conversion_matches_oracle(m, br, sym, sigma_k):
    n, rp, col, val = m
    # sigma: 0 = global sort, else a multiple of 1024 and of b_r
    sigma = 0 if sigma_k == 0 else int(np.lcm(1024, br)) * sigma_k
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, symmetric=sym, sigma=sigma, host_only=True)
    got = A.export()
    if sigma == 0:
        ref = convert.pjds_reference(n, rp, col, val, b_r=br, symmetric=sym)
    else:
        ref = convert.pjds_windows_reference(n, rp, col, val, b_r=br, sigma=sigma, symmetric=sym)
    assert np.array_equal(got["perm"], ref["perm"])
    assert np.array_equal(got["block_len"], ref["block_len"])
    assert np.array_equal(got["col_start"], ref["col_start"])
    assert np.array_equal(got["col"], ref["col"])
    assert got["val"].tobytes() == ref["val"].tobytes()
    assert A.info["stored"] == ref["stored"]
    E = pj.EllrMatrix.from_crs(n, rp, col, val, host_only=True)
    R = convert.ellr_reference(n, rp, col, val)
    ge = E.export()
    assert np.array_equal(ge["rowmax"], R["rowmax"]) and np.array_equal(ge["col"], R["col"])
    assert ge["val"].tobytes() == R["val"].tobytes()
