"""Pins for oracle O1 (long-double CRS spMVM + bound), O2 (acceptance), O3 (FMA chain) and the
plain CRS baseline against things other than the oracle itself: exact rational brute force on
dense matrices, scipy.sparse, closed-form special cases, the G1 hand-computed example, and a
constructed case whose result differs between fused and unfused arithmetic."""
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp

import inputs
import oracle
from conftest import g1_crs

FAMILIES = [("constant", dict(k=3)), ("constant", dict(k=7)), ("uniform", dict(lo=1, hi=9)),
            ("clustered", dict(max=12)), ("adversarial", {}), ("banded", {}), ("empty_rows", {}),
            ("duplicates", {}), ("random", dict(max=20)), ("identity", {}), ("zero", {})]


def dense_exact(n, rowptr, col, val, x):
    """Brute force: materialise A densely with exact rationals (duplicates summed) and form A x."""
    A = [[Fraction(0)] * n for _ in range(n)]
    for i in range(n):
        for k in range(rowptr[i], rowptr[i + 1]):
            A[i][int(col[k])] += Fraction(float(val[k]))
    xs = [Fraction(float(v)) for v in x]
    return [sum((A[i][j] * xs[j] for j in range(n)), Fraction(0)) for i in range(n)]


def ld_frac(v):
    return Fraction(*np.longdouble(v).as_integer_ratio())


@pytest.mark.parametrize("kind,kw", FAMILIES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_spmv_ld_vs_exact_dense(kind, kw, dtype):
    n = 37
    for seed in range(3):
        n_, rp, col, val, = inputs.small(kind, n, seed=seed, dtype=dtype, **kw)
        x = np.random.default_rng(100 + seed).uniform(-1, 1, n).astype(dtype)
        y, b = oracle.spmv_ld(n, rp, col, val, x)
        ex = dense_exact(n, rp, col, val, x)
        for i in range(n):
            nnz = int(rp[i + 1] - rp[i])
            # long-double rounding of each product and partial sum: |err| <= 2*nnz*2^-64*bound
            tol = Fraction(2 * nnz) * Fraction(1, 2 ** 64) * ld_frac(b[i])
            if dtype == np.float32:
                tol = Fraction(nnz) * Fraction(1, 2 ** 64) * ld_frac(b[i])  # products exact
            assert abs(ld_frac(y[i]) - ex[i]) <= tol, (kind, i)
            # the bound is sum |a x| over stored entries
            bb = sum((abs(Fraction(float(val[k])) * Fraction(float(x[col[k]]))) for k in range(rp[i], rp[i + 1])),
                     Fraction(0))
            assert abs(ld_frac(b[i]) - bb) <= Fraction(2 * nnz, 2 ** 64) * bb


def test_g1_golden():
    n, rp, col, val, g = g1_crs()
    x = np.array(g["x"], dtype=np.float64)
    y, _ = oracle.spmv_ld(n, rp, col, val, x)
    assert [float(v) for v in y] == g["y"]
    assert list(oracle.spmv_chain(n, rp, col, val, x)) == g["y"]
    assert list(oracle.spmv_crs(n, rp, col, val, x)) == g["y"]
    y32 = oracle.spmv_chain(n, rp, col, val.astype(np.float32), x.astype(np.float32))
    assert list(y32) == g["y"]


def test_special_cases():
    rng = np.random.default_rng(5)
    n = 200
    x = rng.uniform(-1, 1, n)
    # identity -> x
    _, rp, col, val = inputs.small("identity", n)
    for f in (lambda: oracle.spmv_ld(n, rp, col, val, x)[0], lambda: oracle.spmv_chain(n, rp, col, val, x),
              lambda: oracle.spmv_crs(n, rp, col, val, x)):
        assert np.array_equal(np.asarray(f(), dtype=np.float64), x)
    # zero -> 0
    _, rp, col, val = inputs.small("zero", n)
    assert np.all(oracle.spmv_ld(n, rp, col, val, x)[0] == 0)
    assert np.all(oracle.spmv_chain(n, rp, col, val, x) == 0)
    # ones -> row sums of the values
    _, rp, col, val = inputs.small("uniform", n, seed=3, lo=1, hi=9)
    y, _ = oracle.spmv_ld(n, rp, col, val, np.ones(n))
    rs = [sum(Fraction(float(v)) for v in val[rp[i]:rp[i + 1]]) for i in range(n)]
    for i in range(n):
        assert abs(ld_frac(y[i]) - rs[i]) <= Fraction(16, 2 ** 64)


def test_chain_is_fused_and_in_stored_order():
    """a = 1+2^-30, x0 = 1-2^-30: a*x0 = 1-2^-60 exactly.  Row [(1,-1), (0,a)] with x1 = 1:
    fused chain: fma(-1,1,0) = -1; fma(a,x0,-1) = -2^-60 exactly.  Unfused: round(a*x0) = 1 -> 0.
    Reversed stored order gives fma(a,x0,0) = 1.0 then fma(-1,1,1) = 0."""
    a = 1 + 2.0 ** -30
    x = np.array([1 - 2.0 ** -30, 1.0])
    rp = np.array([0, 2])
    y = oracle.spmv_chain(1, rp, np.array([1, 0], np.int32), np.array([-1.0, a]), x)
    assert y[0] == -(2.0 ** -60)
    y_rev = oracle.spmv_chain(1, rp, np.array([0, 1], np.int32), np.array([a, -1.0]), x)
    assert y_rev[0] == 0.0
    y_plain = oracle.spmv_crs(1, rp, np.array([1, 0], np.int32), np.array([-1.0, a]), x)
    assert y_plain[0] == 0.0  # -ffp-contract=off: mul then add
    yl, _ = oracle.spmv_ld(1, rp, np.array([1, 0], np.int32), np.array([-1.0, a]), x)
    assert yl[0] == -np.longdouble(2.0) ** -60


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_scipy_and_bound(dtype):
    """O1 vs scipy.sparse (library routine) and O2: a double/float FMA chain and the plain CRS loop
    both satisfy the 4*nnz*eps*bound acceptance rule against O1 (textbook gamma_n bound)."""
    g = inputs.Generator.from_config("C1")
    rp, col, val = g.crs(dtype=dtype)
    n = g.n
    x = inputs.vector(n, dtype)
    y, b = oracle.spmv_ld(n, rp, col, val, x)
    A = sp.csr_matrix((val.astype(np.float64), col, rp), shape=(n, n))
    ys = A @ x.astype(np.float64)
    nnz = np.diff(rp)
    assert oracle.acceptance(ys, y, b, nnz, np.float64).all()
    for yt in (oracle.spmv_chain(n, rp, col, val, x), oracle.spmv_crs(n, rp, col, val, x)):
        ok = oracle.acceptance(yt, y, b, nnz, dtype)
        assert ok.all()
    # a perturbation of one ulp-scale multiple beyond the bound must fail (the check is not vacuous)
    yt = oracle.spmv_chain(n, rp, col, val, x).astype(np.longdouble)
    eps = oracle.EPS[np.dtype(dtype)]
    yt[7] += 5 * nnz[7] * eps * b[7]
    assert not oracle.acceptance(yt, y, b, nnz, dtype)[7]


def test_acceptance_edge_rules():
    y_ref = np.array([0, 0, 1], dtype=np.longdouble)
    b = np.array([0, 1, 1], dtype=np.longdouble)
    nnz = np.array([0, 2, 2])
    assert list(oracle.acceptance(np.array([0.0, 0.0, 1.0]), y_ref, b, nnz, np.float64)) == [True, True, True]
    assert list(oracle.acceptance(np.array([-0.0, 0.0, 1.0]), y_ref, b, nnz, np.float64)) == [True, True, True]
    assert not oracle.acceptance(np.array([1e-300, 0.0, 1.0]), y_ref, b, nnz, np.float64)[0]
    assert not oracle.acceptance(np.array([0.0, 0.0, np.nan]), y_ref, b, nnz, np.float64)[2]


def test_crs_baseline_threads_identical():
    g = inputs.Generator.from_config("C1")
    rp, col, val = g.crs()
    x = inputs.vector(g.n)
    y1 = oracle.spmv_crs(g.n, rp, col, val, x, nthreads=1)
    y4 = oracle.spmv_crs(g.n, rp, col, val, x, nthreads=4)
    assert np.array_equal(y1, y4)


def test_split_chain_order_by_hand():
    """oracle_spmv_split_chain (the long-row kernel's arithmetic): interleaved sub-chains and the
    pairwise tree, on exactly representable cases (x = 1) where each order gives a different value.
      row0 = [2^53, 1, -2^53, 1]: single chain 1 (the first +1 is absorbed); S=2 interleaved:
             p0 = 2^53-2^53 = 0, p1 = 1+1 = 2 -> 2 (a contiguous split would give 1);
             S=4: (2^53+1 -> 2^53) + (-2^53+1) = 1.
      row1 = [2^53, 1, 1, -2^53]: single chain 0; S=2: 2^53 + -(2^53-1) = 1; S=4 tree 1
             (a left-to-right sum of the four partials would give 0).
      row2 = [(col1,-1), (col0, 0), (col0, a)] with x0 = 1-2^-30, x1 = 1, a = 1+2^-30, S=2:
             p0 = fma(a, x0, fma(-1, 1, 0)) = -2^-60 exactly (fused), p1 = 0 -> -2^-60."""
    a = 1 + 2.0 ** -30
    B = 2.0 ** 53
    rp = np.array([0, 4, 8, 11])
    col = np.array([0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0], np.int32)
    val = np.array([B, 1, -B, 1, B, 1, 1, -B, -1, 0, a])
    x = np.array([1.0, 1.0])
    assert oracle.spmv_split_chain(2, rp[:3], col[:8], val[:8], x, 1).tolist() == [1.0, 0.0]
    assert oracle.spmv_split_chain(2, rp[:3], col[:8], val[:8], x, 2).tolist() == [2.0, 1.0]
    assert oracle.spmv_split_chain(2, rp[:3], col[:8], val[:8], x, 4).tolist() == [1.0, 1.0]
    x2 = np.array([1 - 2.0 ** -30, 1.0])
    y = oracle.spmv_split_chain(3, rp, col, val, x2, 2)
    assert y[2] == -(2.0 ** -60)
    # S = 1 is the single chain (O3)
    _, rp3, col3, val3 = inputs.small("random", 500, seed=3, max=60)
    xv = inputs.vector(500)
    assert np.array_equal(oracle.spmv_split_chain(500, rp3, col3, val3, xv, 1),
                          oracle.spmv_chain(500, rp3, col3, val3, xv))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("S", [2, 4, 8])
def test_split_chain_within_bound(dtype, S):
    """Any summation order obeys the O2 bound (gamma_n holds for every evaluation tree)."""
    _, rp, col, val = inputs.small("random", 800, seed=S, max=300, dtype=dtype)
    x = inputs.vector(800, dtype)
    y = oracle.spmv_split_chain(800, rp, col, val, x, S)
    yl, b = oracle.spmv_ld(800, rp, col, val, x)
    assert oracle.acceptance(y, yl, b, np.diff(rp), dtype).all()
