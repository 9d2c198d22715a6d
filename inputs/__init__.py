"""Seeded synthetic inputs for the pJDS hot path (shared by oracle tests, GPU tests, bench).

Holds none of the method's arithmetic: it only produces CRS matrices (int64 rowptr, int32 col,
float64/float32 val) and dense x vectors.  Large, paper-shaped families come from the C++
generator ``inputs/gen.cpp`` (counter-based, any row range); small test families are numpy.

Configs (BASELINE.json ``configs``):
  C1  tiny HMEp-shaped banded, N = 16,384
  C2  sAMG-shaped 7-point Poisson, 150x150x151, N = 3,397,500
  C3  HMEp physical, M = 15, N = 6,201,600
  C4  DLR1-shaped, 46,417 points x 6, N = 278,502
  C5  HMEp physical scaled, M = 25, N = 57,002,400, nested spin-grid ordering
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

BASE_SEED = 0x11125588
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpjdsgen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(_LIB_PATH)
        lib.pjdsgen_create.restype = ctypes.c_void_p
        lib.pjdsgen_create.argtypes = [ctypes.c_int] * 4 + [ctypes.c_uint64]
        lib.pjdsgen_destroy.argtypes = [ctypes.c_void_p]
        lib.pjdsgen_n.restype = ctypes.c_int64
        lib.pjdsgen_n.argtypes = [ctypes.c_void_p]
        lib.pjdsgen_rowlen.restype = ctypes.c_int64
        lib.pjdsgen_rowlen.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        lib.pjdsgen_fill.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.pjdsgen_vector.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
        lib.pjdsgen_value.restype = ctypes.c_double
        lib.pjdsgen_value.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64]
        _lib = lib
    return _lib


HMEP, HMEP_BANDED, SAMG, DLR1, DLR2, UHBR = 0, 1, 2, 3, 4, 5


@dataclass(frozen=True)
class Config:
    name: str
    family: int
    p0: int = 0
    p1: int = 0
    p2: int = 0
    desc: str = ""


CONFIGS = {
    "C1": Config("C1", HMEP_BANDED, desc="tiny HMEp-shaped banded, N=16384"),
    "C2": Config("C2", SAMG, 150, 150, 151, desc="sAMG-shaped Poisson, N=3,397,500"),
    "C3": Config("C3", HMEP, 15, 0, desc="HMEp physical M=15, N=6,201,600"),
    "C4": Config("C4", DLR1, desc="DLR1-shaped, N=278,502"),
    "C5": Config("C5", HMEP, 25, 1, desc="HMEp physical M=25 nested spin-grid, N=57,002,400"),
    # NEXT-4 workloads: long rows, dense 5x5 blocks
    "W4": Config("W4", DLR2, desc="DLR2-shaped 108,396 points x 5, N=541,980, N_nzr~315 (PAPER.md L121-127)"),
    "W5": Config("W5", UHBR, desc="UHBR-shaped 900,000 points x 5, N=4,500,000, N_nzr~123 (PAPER.md L129-138)"),
}


class Generator:
    """Handle on one C++ matrix family; rows can be generated per range (per rank)."""

    def __init__(self, family: int, p0: int = 0, p1: int = 0, p2: int = 0, seed: int = BASE_SEED):
        lib = _load()
        self._h = lib.pjdsgen_create(family, p0, p1, p2, seed)
        if not self._h:
            raise ValueError(f"bad generator spec family={family} p=({p0},{p1},{p2})")
        self.n = int(lib.pjdsgen_n(self._h))
        self.seed = seed

    @classmethod
    def from_config(cls, name: str, seed: int = BASE_SEED) -> "Generator":
        c = CONFIGS[name]
        return cls(c.family, c.p0, c.p1, c.p2, seed)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.pjdsgen_destroy(self._h)
            self._h = None

    def rowlen(self, r0: int = 0, r1: int | None = None) -> np.ndarray:
        r1 = self.n if r1 is None else r1
        out = np.empty(r1 - r0, dtype=np.int32)
        _load().pjdsgen_rowlen(self._h, r0, r1, out.ctypes.data)
        return out

    def crs(self, r0: int = 0, r1: int | None = None, dtype=np.float64, symmetric: bool = False):
        """Rows [r0, r1) as CRS: (rowptr int64 [m+1], col int32 (global ids), val dtype).
        symmetric: a(r,c) = a(c,r) (structurally symmetric families: HMEp, banded, sAMG)."""
        r1 = self.n if r1 is None else r1
        lens = self.rowlen(r0, r1)
        rowptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
        np.cumsum(lens, out=rowptr[1:])
        nnz = int(rowptr[-1])
        col = np.empty(nnz, dtype=np.int32)
        dt = np.dtype(dtype)
        val = np.empty(nnz, dtype=dt)
        _load().pjdsgen_fill(self._h, r0, r1, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data,
                             (1 if dt == np.float64 else 0) | (2 if symmetric else 0))
        return rowptr, col, val


def vector(n: int, dtype=np.float64, seed: int = BASE_SEED + 1, i0: int = 0) -> np.ndarray:
    """x entries [i0, i0+n): uniform in [-1, 1) from splitmix64(seed, i)."""
    dt = np.dtype(dtype)
    out = np.empty(n, dtype=dt)
    _load().pjdsgen_vector(seed, i0, i0 + n, out.ctypes.data, 1 if dt == np.float64 else 0)
    return out


def value(row: int, col: int, seed: int = BASE_SEED) -> float:
    return float(_load().pjdsgen_value(seed, row, col))


def config_crs(name: str, dtype=np.float64, seed: int = BASE_SEED, symmetric: bool = False):
    g = Generator.from_config(name, seed)
    rowptr, col, val = g.crs(dtype=dtype, symmetric=symmetric)
    return g.n, rowptr, col, val


# ---------------------------------------------------------------- small numpy families
def _from_rows(n, rows, rng, dtype, values=None):
    """rows: list of column arrays (CRS order kept as given)."""
    lens = np.array([len(r) for r in rows], dtype=np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rowptr[1:])
    col = np.concatenate([np.asarray(r, dtype=np.int32) for r in rows]) if rows else np.zeros(0, np.int32)
    if values is None:
        val = rng.uniform(-1.0, 1.0, size=int(rowptr[-1]))
    else:
        val = np.asarray(values, dtype=np.float64)
    return n, rowptr, col.astype(np.int32), val.astype(dtype)


def small(kind: str, n: int, seed: int = 0, dtype=np.float64, **kw):
    """Small test matrices (SPEC.md L39 families plus edge cases).

    kinds: constant(k), uniform(lo,hi), clustered, adversarial, banded(offsets), empty_rows,
           duplicates, random (uniform lengths 0..maxlen, unsorted columns), identity, zero.
    Returns (n, rowptr, col, val).
    """
    rng = np.random.default_rng(seed)
    rows = []
    if kind == "constant":
        k = min(kw.get("k", 3), n)
        rows = [np.sort(rng.choice(n, k, replace=False)) for _ in range(n)]
    elif kind == "uniform":
        lo, hi = kw.get("lo", 1), min(kw.get("hi", 8), n)
        rows = [np.sort(rng.choice(n, rng.integers(lo, hi + 1), replace=False)) for _ in range(n)]
    elif kind == "clustered":
        mx = min(kw.get("max", 20), n)
        frac = kw.get("frac", 0.8)
        rows = []
        for _ in range(n):
            k = rng.integers(int(0.8 * mx), mx + 1) if rng.random() < frac else rng.integers(1, max(2, int(0.8 * mx)))
            rows.append(np.sort(rng.choice(n, int(k), replace=False)))
    elif kind == "adversarial":  # one full row, all others one entry
        rows = [np.arange(n)] + [np.array([rng.integers(0, n)]) for _ in range(n - 1)]
    elif kind == "banded":
        offs = kw.get("offsets", [-3, -1, 0, 1, 3])
        rows = [np.array([i + o for o in sorted(offs) if 0 <= i + o < n]) for i in range(n)]
    elif kind == "empty_rows":
        mx = min(kw.get("max", 10), n)
        rows = [np.sort(rng.choice(n, rng.integers(0, mx + 1), replace=False)) if rng.random() > 0.3 else np.array([], np.int64)
                for _ in range(n)]
    elif kind == "duplicates":
        mx = kw.get("max", 10)
        rows = [rng.integers(0, n, size=rng.integers(0, mx + 1)) for _ in range(n)]  # repeats, unsorted
    elif kind == "random":
        mx = kw.get("max", 40)
        rows = [rng.permutation(rng.choice(n, min(n, rng.integers(0, mx + 1)), replace=False)) for _ in range(n)]
    elif kind == "identity":
        return _from_rows(n, [np.array([i]) for i in range(n)], rng, dtype, values=np.ones(n))
    elif kind == "zero":
        return _from_rows(n, [np.array([], np.int64) for _ in range(n)], rng, dtype)
    else:
        raise ValueError(kind)
    return _from_rows(n, rows, rng, dtype)
