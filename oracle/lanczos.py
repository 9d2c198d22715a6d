"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Symmetric Lanczos recurrence written out as in the textbook (no re-orthogonalisation), fp64,
using a plain CRS product (scipy.sparse as the matrix-vector primitive) — the reference for the
library's permuted-basis Lanczos driver ("application of our
results to a production-grade eigensolver", L241-246 permuted basis):

    v_0 = v0 / ||v0||, beta_{-1} = 0, v_{-1} = 0
    for j = 0 .. m-1:
        w = A v_j
        alpha_j = w . v_j
        w = w - alpha_j v_j - beta_{j-1} v_{j-1}
        beta_j = ||w||
        v_{j+1} = w / beta_j

and the eigenvalues of the resulting tridiagonal matrix via numpy (LAPACK) as the Ritz values.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def lanczos(n, rowptr, col, val, v0, m):
    A = sp.csr_matrix((np.asarray(val, dtype=np.float64), np.asarray(col), np.asarray(rowptr)), shape=(n, n))
    v = np.asarray(v0, dtype=np.float64)
    v = v / np.linalg.norm(v)
    v_prev = np.zeros(n)
    beta_prev = 0.0
    alpha = np.zeros(m)
    beta = np.zeros(m)
    for j in range(m):
        w = A @ v
        alpha[j] = w @ v
        w = w - alpha[j] * v - beta_prev * v_prev
        beta[j] = np.linalg.norm(w)
        if beta[j] == 0.0:
            return alpha[: j + 1], beta[: j + 1]
        v_prev, v = v, w / beta[j]
        beta_prev = beta[j]
    return alpha, beta


def ritz_values(alpha, beta):
    m = len(alpha)
    T = np.diag(alpha) + np.diag(beta[: m - 1], 1) + np.diag(beta[: m - 1], -1)
    return np.linalg.eigvalsh(T)
