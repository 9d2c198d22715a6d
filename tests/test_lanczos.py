"""NEXT-1: permuted-basis Lanczos driver.  CPU: the oracle recurrence is pinned against dense
eigenvalues (extreme Ritz values converge to numpy.linalg.eigvalsh of A) and the library's
tridiagonal eigen-solver against LAPACK.  GPU: the library driver (pJDS kernel in the permuted basis,
CUDA-graph captured) reproduces the oracle's alpha/beta and extreme Ritz values."""
import numpy as np
import pytest

import inputs
from oracle import lanczos as olz


def sym_matrix(n, seed):
    """Structurally symmetric random sparse matrix with symmetric values."""
    rng = np.random.default_rng(seed)
    rows = [set([i]) for i in range(n)]
    for _ in range(4 * n):
        a, b = rng.integers(0, n, 2)
        rows[a].add(int(b))
        rows[b].add(int(a))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    col = np.concatenate([np.array(sorted(r), np.int32) for r in rows])
    val = np.empty(len(col))
    k = 0
    for i in range(n):
        for c in sorted(rows[i]):
            lo, hi = min(i, c), max(i, c)
            val[k] = np.sin(1.0 + 0.37 * lo + 0.61 * hi + 0.013 * lo * hi)
            k += 1
    return n, rp, col, val


def test_oracle_lanczos_extreme_ritz_values():
    n, rp, col, val = sym_matrix(400, 1)
    A = np.zeros((n, n))
    for i in range(n):
        A[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    assert np.allclose(A, A.T)
    ev = np.linalg.eigvalsh(A)
    a, b = olz.lanczos(n, rp, col, val, np.random.default_rng(0).uniform(-1, 1, n), 150)
    rv = olz.ritz_values(a, b)
    assert abs(rv[0] - ev[0]) < 1e-9 * abs(ev).max()
    assert abs(rv[-1] - ev[-1]) < 1e-9 * abs(ev).max()
    # interlacing: Ritz values lie inside the spectrum
    assert rv[0] >= ev[0] - 1e-9 and rv[-1] <= ev[-1] + 1e-9


def test_oracle_lanczos_first_step_by_hand():
    """m = 1: alpha_0 = v.Av / v.v (Rayleigh quotient), beta_0 = ||Av - alpha v|| / ||v||."""
    n, rp, col, val = sym_matrix(50, 2)
    import scipy.sparse as sp
    A = sp.csr_matrix((val, col, rp), shape=(n, n))
    v = np.linspace(-1, 1, n) + 0.1
    a, b = olz.lanczos(n, rp, col, val, v, 1)
    u = v / np.linalg.norm(v)
    w = A @ u
    assert a[0] == pytest.approx(w @ u, rel=1e-14)
    assert b[0] == pytest.approx(np.linalg.norm(w - (w @ u) * u), rel=1e-13)


def test_tridiag_eigenvalues_vs_lapack():
    import build_native
    build_native.build_pjds()
    import paper_1112_5588_b200 as pj
    rng = np.random.default_rng(3)
    for m in (1, 2, 7, 60):
        a = rng.normal(size=m)
        b = rng.uniform(0.1, 2.0, size=m)
        got = pj.tridiag_eigenvalues(a, b)
        want = olz.ritz_values(a, b)
        assert np.allclose(got, want, rtol=0, atol=1e-12 * max(1.0, np.abs(want).max()))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gpu_lanczos_matches_oracle(dtype):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_1112_5588_b200 as pj
    for name, src in (("rand", sym_matrix(3000, 5)), ("C1", inputs.config_crs("C1", symmetric=True))):
        n, rp, col, val = src
        val = val.astype(dtype)
        v0 = inputs.vector(n, dtype, seed=77)
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
        perm = A.export()["perm"]
        m = 40
        a, b, steps = A.lanczos(torch.from_numpy(v0[perm].copy()).cuda(), m)
        assert steps == m
        ra, rb = olz.lanczos(n, rp, col, val.astype(np.float64), v0.astype(np.float64), m)
        # every coefficient of the m = 40 steps, not only the first ones: the GPU products are
        # bitwise the oracle's FMA chains, so the recurrences differ only by the rounding of the
        # dot products / vector updates.  Measured on B200 (tools/lanczos_drift.py,
        # profiles/r02_lanczos_drift.jsonl): max |da|, |db| / scale = 6.2e-16 (DP), 6.6e-8 (SP)
        # over all 40 steps; the bounds below leave ~100x (DP) / ~30x (SP) of headroom and are still
        # 1e3-1e4 x tighter than a single wrong term or a dropped step would produce.
        tol = 1e-13 if dtype == np.float64 else 2e-6
        scale = max(np.abs(ra).max(), np.abs(rb).max())
        assert np.abs(a - ra).max() <= tol * scale, name
        assert np.abs(b - rb).max() <= tol * scale, name
        assert (b > 0).all(), name  # no breakdown on these matrices
        ev, rv = pj.tridiag_eigenvalues(a, b), olz.ritz_values(ra, rb)
        assert np.abs(ev - rv).max() <= 10 * tol * scale, name  # all 40 Ritz values


@pytest.mark.gpu
def test_gpu_lanczos_many_product_partials():
    """n_pad = 40,032 runs the one-row-per-thread kernel: 157 CTAs x 8 warps = 1,256 per-warp dot
    partials, more than the update pass's 1,184 and than n_pad / 32 + 1 (the partial buffer and the
    two-level alpha reduce must hold them all)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_1112_5588_b200 as pj
    n, rp, col, val = sym_matrix(40001, 11)
    v0 = inputs.vector(n, np.float64, seed=78)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
    perm = A.export()["perm"]
    m = 12
    a, b, steps = A.lanczos(torch.from_numpy(v0[perm].copy()).cuda(), m)
    assert steps == m
    ra, rb = olz.lanczos(n, rp, col, val, v0, m)
    scale = max(np.abs(ra).max(), np.abs(rb).max())
    assert np.abs(a - ra).max() <= 1e-10 * scale
    assert np.abs(b - rb).max() <= 1e-10 * scale


@pytest.mark.gpu
def test_gpu_lanczos_breakdown_and_zero_start():
    """A = 2 I with v0 = e_0: alpha_0 = 2 and w = 0 exactly, so the recurrence stops after one step
    (steps_done = 1), as the oracle does; a zero start vector is rejected."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_1112_5588_b200 as pj
    n = 500
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    val = np.full(n, 2.0)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
    perm = A.export()["perm"]
    e0 = np.zeros(n)
    e0[0] = 1.0
    a, b, steps = A.lanczos(torch.from_numpy(e0[perm].copy()).cuda(), 10)
    ra, rb = olz.lanczos(n, rp, col, val, e0, 10)
    assert steps == 1 == len(ra)
    assert a[0] == ra[0] == 2.0 and b[0] == rb[0] == 0.0
    with pytest.raises(pj.PjdsError):
        A.lanczos(torch.zeros(n, dtype=torch.float64, device="cuda"), 5)


@pytest.mark.gpu
def test_gpu_lanczos_split_variant():
    """The fused alpha epilogue of the long-row split-j kernel (knob 16 + S) in the Lanczos driver."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_1112_5588_b200 as pj
    n, rp, col, val = sym_matrix(3000, 6)
    v0 = inputs.vector(n, seed=78)
    ra, rb = olz.lanczos(n, rp, col, val, v0, 30)
    L = pj.lib()
    try:
        for S in (2, 4, 8):
            assert L.pjds_set_kernel_variant(16 + S, 4) == 0
            A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
            perm = A.export()["perm"]
            a, b, steps = A.lanczos(torch.from_numpy(v0[perm].copy()).cuda(), 30)
            scale = max(np.abs(ra).max(), np.abs(rb).max())
            assert steps == 30
            assert np.abs(a[:10] - ra[:10]).max() <= 1e-10 * scale, S
            assert np.abs(b[:10] - rb[:10]).max() <= 1e-10 * scale, S
    finally:
        L.pjds_set_kernel_variant(0, 0)


@pytest.mark.gpu
def test_gpu_lanczos_c3_br128_lane_interleaved():
    """C3-sized symmetric HMEp matrix at b_r = 128 in DP: the Lanczos product runs the
    lane-interleaved kernel with the fused alpha partials (R = 4, rows 32 apart per thread); its
    coefficients follow the oracle recurrence (scipy CSR products) over 12 steps."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_1112_5588_b200 as pj
    n, rp, col, val = inputs.config_crs("C3", symmetric=True)
    v0 = inputs.vector(n, np.float64, seed=79)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=128, symmetric=True)
    perm = A.export()["perm"]
    m = 12
    a, b, steps = A.lanczos(torch.from_numpy(v0[perm].copy()).cuda(), m)
    assert steps == m
    ra, rb = olz.lanczos(n, rp, col, val, v0, m)
    scale = max(np.abs(ra).max(), np.abs(rb).max())
    assert np.abs(a - ra).max() <= 1e-12 * scale
    assert np.abs(b - rb).max() <= 1e-12 * scale
