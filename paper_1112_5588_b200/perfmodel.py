"""The paper's performance model (§2.2), host-side arithmetic.

  Eq. 1 (L333-339)  code balance  B_W^DP = (8 + 4 + 8 alpha + 16/N_nzr) / 2  bytes/flop
                    (Listing semantics c += : the LHS is read and written).  With y = A x written
                    only (reading 11) the LHS term is 8/N_nzr; SP halves value bytes
                    (reading 12).  The split local/nonlocal kernel adds 8/N_nzr (L445-447).
  Eq. 2 (L356-364)  T_MVM = 8N/B_GPU [N_nzr (alpha + 3/2) + 2],  T_PCI = 16N/B_PCI   (DP)
  Eq. 3 (L365-372)  T_MVM <= T_PCI  <=>  N_nzr <= 2 (B_GPU/B_PCI - 1) / (alpha + 3/2)
  Eq. 4 (L380-390)  T_MVM >= 10 T_PCI  <=>  N_nzr >= (20 B_GPU/B_PCI - 2) / (alpha + 3/2)
  alpha (L340-351)  RHS re-load factor, 1/N_nzr (each x element loaded once) .. 1 (no cache).
With alpha = 1/N_nzr ("reciprocal") Eq. 3/4 are solved exactly for N_nzr:
  N_nzr (1/N_nzr + 3/2) <= 2(r - 1)  =>  N_nzr <= (2(r - 1) - 1) / (3/2)
  N_nzr (1/N_nzr + 3/2) >= 20 r - 2  =>  N_nzr >= (20 r - 3) / (3/2)
"""
from __future__ import annotations

RECIPROCAL = "reciprocal"


def code_balance(alpha: float, n_nzr: float, precision: str = "dp", lhs: str = "rw", split: bool = False) -> float:
    """Bytes per flop of the ELLPACK(-R)/pJDS kernels (Eq. 1).  lhs: "rw" as printed (c +=),
    "w" for y = A x (write only).  split: local/nonlocal two-pass kernel (+8/N_nzr DP)."""
    sv = 8 if precision == "dp" else 4
    lhs_bytes = (2 if lhs == "rw" else 1) * sv
    b = (sv + 4 + sv * alpha + lhs_bytes / n_nzr) / 2.0
    if split:
        b += sv / n_nzr
    return b


def t_mvm(n: float, n_nzr: float, alpha: float, b_gpu: float) -> float:
    """Eq. 2, DP spMVM time on the device (seconds for bandwidth in bytes/s)."""
    return 8.0 * n / b_gpu * (n_nzr * (alpha + 1.5) + 2.0)


def t_pci(n: float, b_pci: float) -> float:
    """Eq. 2, DP RHS down + LHS up over PCIe (16 N bytes)."""
    return 16.0 * n / b_pci


def n_nzr_upper(ratio: float, alpha) -> float:
    """Eq. 3: largest N_nzr for which PCIe costs more than the spMVM (> 50 % penalty)."""
    if alpha == RECIPROCAL:
        return (2.0 * (ratio - 1.0) - 1.0) / 1.5
    return 2.0 * (ratio - 1.0) / (alpha + 1.5)


def n_nzr_lower(ratio: float, alpha) -> float:
    """Eq. 4: smallest N_nzr with less than 10 % PCIe penalty."""
    if alpha == RECIPROCAL:
        return (20.0 * ratio - 3.0) / 1.5
    return (20.0 * ratio - 2.0) / (alpha + 1.5)


def measured_alpha(dram_read_bytes: float, stored: int, nnz: int, n: int, value_bytes: int,
                   aux_bytes: float = 0.0) -> float:
    """RHS re-load factor from a DRAM byte count: x bytes actually read per
    stored nonzero, in units of one x element: (read - matrix - aux) / (nnz * s_v)."""
    x_bytes = dram_read_bytes - stored * (value_bytes + 4) - aux_bytes
    return x_bytes / (nnz * value_bytes)


def min_bytes(nnz: int, n: int, value_bytes: int) -> int:
    """Algorithmic bytes of one y = A x: values + indices once, x once, y written once
    (Eq. 1 at alpha = 1/N_nzr with a write-only LHS, times 2 nnz flops)."""
    return nnz * (value_bytes + 4) + 2 * n * value_bytes
