"""Pins of the §2.2 performance model (paper_1112_5588_b200/perfmodel.py) against the values the
paper and SPEC print: Eq. 1 limits, Eq. 3/4 worked thresholds (PAPER.md
L373-390: "N_nzr <= 25", "<= 7", ">~ 80", ">~ 266"; exact algebra 24.67 / 7.2 / 79.2 / 264.67,
reading 20: +-2), the split-kernel penalty (L445-447) and Eq. 2 / Eq. 3 consistency."""
import pytest

from paper_1112_5588_b200 import perfmodel as pm


def test_eq1_code_balance():
    assert pm.code_balance(1.0, 1e12) == pytest.approx(10.0)                 # alpha=1, N -> inf
    assert pm.code_balance(1.0, 8) == 11.0                                   # 6 + 4 + 1
    assert pm.code_balance(1 / 4, 4) == 9.0                                  # 6 + 12/N at N = 4
    assert pm.code_balance(1 / 4, 4) == 6 + 4 * 0.25 + 8 / 4                  # printed right-hand side
    # split kernel adds exactly 8/N_nzr
    assert pm.code_balance(0.3, 16, split=True) - pm.code_balance(0.3, 16) == pytest.approx(8 / 16)
    # write-only LHS (reading 11): 6 + 4 alpha + 4/N ; SP: 4 + 2 alpha + 2/N
    assert pm.code_balance(0.5, 10, lhs="w") == pytest.approx(6 + 2 + 0.4)
    assert pm.code_balance(0.5, 10, precision="sp", lhs="w") == pytest.approx(4 + 1 + 0.2)
    # SP < DP, monotone in alpha and N_nzr
    assert pm.code_balance(0.5, 10, "sp") < pm.code_balance(0.5, 10, "dp")
    assert pm.code_balance(0.6, 10) > pm.code_balance(0.5, 10)
    assert pm.code_balance(0.5, 11) < pm.code_balance(0.5, 10)


def test_eq3_eq4_paper_worked_values():
    assert pm.n_nzr_upper(20, pm.RECIPROCAL) == pytest.approx(37 / 1.5)      # 24.67
    assert abs(pm.n_nzr_upper(20, pm.RECIPROCAL) - 25) <= 2                   # paper: "N_nzr <= 25"
    assert pm.n_nzr_upper(10, 1.0) == pytest.approx(7.2)                      # paper: "N_nzr <= 7"
    assert pm.n_nzr_lower(10, 1.0) == pytest.approx(79.2)                     # paper: ">~ 80"
    assert pm.n_nzr_lower(20, pm.RECIPROCAL) == pytest.approx(397 / 1.5)      # 264.67
    assert abs(pm.n_nzr_lower(20, pm.RECIPROCAL) - 266) <= 2                  # paper: ">~ 266"


def test_eq2_eq3_consistency():
    """At the Eq. 3 threshold T_MVM == T_PCI exactly (fixed alpha)."""
    bg, bp = 91e9, 6e9
    for alpha in (0.1, 0.5, 1.0):
        nz = pm.n_nzr_upper(bg / bp, alpha)
        assert pm.t_mvm(1e6, nz, alpha, bg) == pytest.approx(pm.t_pci(1e6, bp), rel=1e-12)
        nz = pm.n_nzr_lower(bg / bp, alpha)
        assert pm.t_mvm(1e6, nz, alpha, bg) == pytest.approx(10 * pm.t_pci(1e6, bp), rel=1e-12)
    # SPEC.md L311 worked value: 8e6/91e9 * 252 = 22.15 ms
    assert pm.t_mvm(1e6, 100, 1.0, 91e9) == pytest.approx(22.15e-3, rel=1e-3)


def test_min_bytes_and_alpha():
    # min bytes = Eq. 1 (write-only LHS) at alpha = 1/N_nzr times 2 nnz flops
    n, nnz = 1000, 15000
    assert pm.min_bytes(nnz, n, 8) == pytest.approx(pm.code_balance(n / nnz, nnz / n, lhs="w") * 2 * nnz)
    # a DRAM count equal to matrix + one x read gives alpha = 1/N_nzr
    assert pm.measured_alpha(nnz * 12 + n * 8, nnz, nnz, n, 8) == pytest.approx(n / nnz)
