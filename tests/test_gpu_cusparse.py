"""An independent GPU witness: cuSPARSE CSR SpMV, reached through torch.sparse CSR (`torch.mv`).

SURVEY §8(c), "What pins each part", O1 pin (ii): "on the GPU box, cuSPARSE CSR SpMV as an
independent GPU result under the same bound".  cuSPARSE shares nothing with the oracle (plain C,
long double) or with libpjds (pJDS / ELLPACK-R kernels): its own format (CRS as given), its own
summation order.  Any summation order of a row's products has |error| <= gamma_nnz * sum|a x|
(Higham), inside the north-star bound 4 nnz_i eps sum|a x|, so:

  1. at the full paper-shaped sizes (C1-C4, SP and DP; beyond scipy's reach in the CPU suite) the
     oracle and cuSPARSE must agree within O2 -- a dropped term, a wrong sign or a mis-indexed
     column in the oracle fails this on essentially every row;
  2. on C5, the bench workload (942 M nonzeros, the bench's launch configuration), EVERY row of the
     pJDS product is checked against cuSPARSE with the triangle-inequality bound
     |y_pjds - y_cus| <= 8 nnz_i eps (|A| |x|)_i, |A||x| also computed by cuSPARSE in DP (its own
     relative rounding, <= nnz_i eps, is covered by a 1e-6 relative slack on the tolerance).

Test infrastructure only: cuSPARSE never appears on the product path.
"""
import numpy as np
import pytest

import inputs
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.filterwarnings("ignore:Sparse CSR tensor support is in beta"),
              pytest.mark.filterwarnings("ignore:Sparse invariant checks are implicitly disabled")]

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pj():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1112_5588_b200 as pj
    pj.lib()
    return pj


def csr_gpu(n, rp, col, val):
    """torch sparse CSR on cuda:0 (int32 indices: every config has nnz < 2^31)."""
    assert rp[-1] < 2**31
    return torch.sparse_csr_tensor(torch.from_numpy(rp.astype(np.int32)).cuda(),
                                   torch.from_numpy(np.ascontiguousarray(col)).cuda(),
                                   torch.from_numpy(np.ascontiguousarray(val)).cuda(), size=(n, n),
                                   check_invariants=False)


@pytest.mark.parametrize("name", ["C1", "C4", "C2", "C3"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cusparse_pins_oracle(pj, name, dtype):
    n, rp, col, val = inputs.config_crs(name, dtype=dtype)
    x = inputs.vector(n, dtype)
    A = csr_gpu(n, rp, col, val)
    y = torch.mv(A, torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    y_cus = y.cpu().numpy()
    y_ref, bound = oracle.spmv_ld(n, rp, col, val, x)
    ok = oracle.acceptance(y_cus, y_ref, bound, np.diff(rp), dtype)
    assert ok.all(), f"{name}: {(~ok).sum()} rows where cuSPARSE and the oracle disagree beyond O2"
    # the comparison is not vacuous: the bound is tight against a real perturbation of one term
    if n > 0 and bound.max() > 0:
        i = int(np.argmax(np.diff(rp)))
        k = int(rp[i])
        bad = y_ref.copy()
        bad[i] -= 2 * np.longdouble(val[k]) * np.longdouble(x[col[k]])  # one sign flipped
        if abs(val[k] * x[col[k]]) > 4 * (rp[i + 1] - rp[i]) * np.finfo(dtype).eps * bound[i]:
            assert not oracle.acceptance(y_cus[i:i + 1], bad[i:i + 1], bound[i:i + 1],
                                         np.diff(rp)[i:i + 1], dtype).all()


def test_c5_every_row_vs_cusparse(pj):
    """C5 DP at full size, the bench's launch configuration (b_r = 32, permuted basis, tile order)."""
    g = inputs.Generator.from_config("C5")
    n = g.n
    rp, col, val = g.crs()
    lens = torch.from_numpy(np.diff(rp)).cuda()
    x = inputs.vector(n)
    xt = torch.from_numpy(x).cuda()
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=32, symmetric=True)
    xp = torch.empty_like(xt)
    yp = torch.empty_like(xt)
    y = torch.empty_like(xt)
    A.to_permuted(xp, xt)
    A.spmv(yp, xp)
    A.from_permuted(y, yp)
    del A
    C = csr_gpu(n, rp, col, val)
    del col
    y_cus = torch.mv(C, xt)
    absC = torch.sparse_csr_tensor(C.crow_indices(), C.col_indices(), C.values().abs(), size=(n, n),
                                   check_invariants=False)
    del C
    bound = torch.mv(absC, xt.abs())
    del absC
    torch.cuda.synchronize()
    eps = np.finfo(np.float64).eps
    tol = 8 * lens.double() * eps * bound * (1 + 1e-6)
    diff = (y - y_cus).abs()
    bad = ~(diff <= tol) | ~torch.isfinite(y)
    assert int(bad.sum()) == 0, f"{int(bad.sum())} rows of the C5 pJDS product outside the bound vs cuSPARSE"
