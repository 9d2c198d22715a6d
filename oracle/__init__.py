"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously correct CPU reference for the pJDS hot path of Kreutzer et al.,
arXiv 1112.5588.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import, call, link or execute anything here.
It shares no code, header, table or constant generator with ``paper_1112_5588_b200`` (the CUDA
path) and never imports it; the only thing both consume is ``inputs/`` (seeded generators).

Modules
  oracle.c / this file  O1 long-double CRS spMVM + per-row bound, O2 acceptance check,
                        O3 FMA-chain emulation, plain CRS baseline
  convert.py            O4 reference CRS->pJDS / CRS->ELLPACK-R converters, Listing 1/2
                        emulations, footprint & utilisation counters
  dist.py               O5 row-partition / halo-schedule / local+nonlocal split emulator
                                                                          
Every function is pinned by tests/test_oracle_*.py against something other than itself (exact
rational brute force, scipy, the paper's closed forms, SPEC worked examples, invariants);
see DESIGN.md §"Oracle and its pins".
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: build with build_native.build_oracle()")
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        lib.oracle_spmv_ld.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_int, P, P]
        lib.oracle_spmv_chain.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_int, P]
        lib.oracle_spmv_split_chain.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_spmv_crs.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_int, P, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _prep(n, rowptr, col, val, x):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val)
    if val.dtype not in (np.float32, np.float64):
        raise TypeError("val must be float32 or float64")
    x = np.ascontiguousarray(x, dtype=val.dtype)
    assert rowptr.shape == (n + 1,) and col.shape == val.shape and x.ndim == 1
    return rowptr, col, val, x, (1 if val.dtype == np.float64 else 0)


def spmv_ld(n, rowptr, col, val, x):
    """O1: y_i = sum_k val[k]*x[col[k]] accumulated in long double, and bound_i = sum_k |val[k]*x[col[k]]|.

    PAPER.md L37-39 (y = A x), Table 1 L296 (CRS).  Returns (y, bound) as np.longdouble arrays.
    """
    rowptr, col, val, x, dt = _prep(n, rowptr, col, val, x)
    y = np.empty(n, dtype=np.longdouble)
    b = np.empty(n, dtype=np.longdouble)
    _load().oracle_spmv_ld(n, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data, x.ctypes.data, dt,
                           y.ctypes.data, b.ctypes.data)
    return y, b


def spmv_chain(n, rowptr, col, val, x):
    """O3: per row, acc = +0.0; acc = fma(val[k], x[col[k]], acc) in stored CRS order (matrix precision)."""
    rowptr, col, val, x, dt = _prep(n, rowptr, col, val, x)
    y = np.empty(n, dtype=val.dtype)
    _load().oracle_spmv_chain(n, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data, x.ctypes.data, dt,
                              y.ctypes.data)
    return y


def spmv_split_chain(n, rowptr, col, val, x, S: int):
    """Split-j arithmetic: S interleaved FMA chains per row (entries j = s mod S, CRS order, from +0)
    combined by the pairwise tree ((p0+p1)+(p2+p3))+...; S = 1 is spmv_chain (see oracle.c)."""
    assert S >= 1 and S & (S - 1) == 0 and S <= 64
    rowptr, col, val, x, dt = _prep(n, rowptr, col, val, x)
    y = np.empty(n, dtype=val.dtype)
    _load().oracle_spmv_split_chain(n, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data, x.ctypes.data, dt,
                                    int(S), y.ctypes.data)
    return y


def spmv_crs(n, rowptr, col, val, x, nthreads: int = 0):
    """Plain CRS loop in the matrix precision (s += a*x, no FMA contraction), OpenMP over rows.

    The CPU baseline timed by bench.py (Table 1 "CRS (DP)").
    """
    rowptr, col, val, x, dt = _prep(n, rowptr, col, val, x)
    y = np.empty(n, dtype=val.dtype)
    _load().oracle_spmv_crs(n, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data, x.ctypes.data, dt,
                            y.ctypes.data, int(nthreads))
    return y


def max_threads() -> int:
    return int(_load().oracle_max_threads())


EPS = {np.dtype(np.float64): np.longdouble(2.0) ** -52, np.dtype(np.float32): np.longdouble(2.0) ** -23}


def acceptance(y, y_ref, bound, row_nnz, dtype):
    """O2 (north star): per row |y_i - y_ref_i| <= 4 * nnz_i * eps_T * bound_i.

    nnz_i = stored CRS entries of row i; nnz_i = 0 or bound_i = 0 requires y_i == 0 (+-0 equal);
    NaN/Inf always fails.  Returns a boolean mask of rows that PASS.
    """
    eps = EPS[np.dtype(dtype)]
    y = np.asarray(y).astype(np.longdouble)
    y_ref = np.asarray(y_ref, dtype=np.longdouble)
    bound = np.asarray(bound, dtype=np.longdouble)
    nnz = np.asarray(row_nnz).astype(np.longdouble)
    tol = 4 * nnz * eps * bound
    ok = np.abs(y - y_ref) <= tol
    ok &= np.isfinite(y)
    return ok
