"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

O4: reference CRS -> pJDS and CRS -> ELLPACK-R converters, written step by step from PAPER.md
§2.1 (L144-266) in the paper's order and notation, plus literal emulations of Listing 1 and
Listing 2 and the footprint / Fig. 2 utilisation counters.  Readings of silent or ambiguous
points are SURVEY §8(c) / DESIGN.md readings 1-17; each is cited where used.
"""
from __future__ import annotations

import numpy as np


def _lens(rowptr):
    # reading 2: "number of non-zeros" = stored CRS entries per row (explicit zeros count)
    return np.diff(np.asarray(rowptr, dtype=np.int64))


def pjds_reference(n, rowptr, col, val, b_r: int = 32, symmetric: bool = False):
    """CRS -> pJDS, PAPER.md L213-229 ("sort" and "pad" steps, col_start[]) and Listing 2 L231-237.

    Returns dict with perm (perm[new] = old, reading 10), invperm, block_len, col_start
    (width+1 int64 entries, reading 5), val, col (jagged column-major), n_pad, n_blocks, width, stored.
    b_r >= 1 is any positive block size here (the library restricts it to multiples of 32).
    """
    if b_r < 1:
        raise ValueError("b_r >= 1")
    rowptr = np.asarray(rowptr, dtype=np.int64)
    col = np.asarray(col)
    val = np.asarray(val)
    lens = _lens(rowptr)
    # "sort": rows sorted by number of non-zeros, starting with the longest row (L216-219);
    # ties by ascending original index (reading 1: stable sort).
    perm = np.argsort(-lens, kind="stable").astype(np.int32)
    invperm = np.empty(n, dtype=np.int32)
    invperm[perm] = np.arange(n, dtype=np.int32)
    # "pad": blocks of b_r consecutive (sorted) rows padded to the longest row within the block
    # (L219-222); N padded to a multiple of b_r with zero-length virtual rows (reading 3, L153-155).
    n_blocks = -(-n // b_r)
    n_pad = n_blocks * b_r
    sorted_len = np.zeros(n_pad, dtype=np.int64)
    sorted_len[:n] = lens[perm]
    block_len = sorted_len.reshape(n_blocks, b_r).max(axis=1) if n_blocks else np.zeros(0, np.int64)
    width = int(block_len.max()) if n_blocks else 0
    # col_start[]: starting offset of each jagged column (L225-228); column j holds one slot for
    # every row of every block whose padded length exceeds j.
    col_start = np.zeros(width + 1, dtype=np.int64)
    for j in range(width):
        col_start[j + 1] = col_start[j] + b_r * int(np.count_nonzero(block_len > j))
    stored = int(col_start[width])
    # fill (Listing 2 indexing): val[col_start[j] + k] = j-th stored entry of sorted row k;
    # CRS order kept within a row (reading 8); padding = (+0.0, col 0) (reading 7).
    out_val = np.zeros(stored, dtype=val.dtype)
    out_col = np.zeros(stored, dtype=np.int32)
    cols_mapped = invperm[col] if symmetric and len(col) else col  # reading 9 (symmetric: P A P^T)
    for j in range(width):
        m = int(col_start[j + 1] - col_start[j])  # rows k = 0 .. m-1 have a slot in column j
        k = np.arange(min(m, n))
        r = perm[k]
        has = lens[r] > j
        src = rowptr[r[has]] + j
        dst = col_start[j] + k[has]
        out_val[dst] = val[src]
        out_col[dst] = cols_mapped[src]
    return dict(perm=perm, invperm=invperm, block_len=block_len.astype(np.int32), col_start=col_start,
                val=out_val, col=out_col, n=n, n_pad=n_pad, n_blocks=n_blocks, width=width, stored=stored,
                b_r=b_r, row_len_sorted=sorted_len)


def pjds_windows_reference(n, rowptr, col, val, b_r: int = 32, sigma: int = 1024, symmetric: bool = False):
    """Sort scope sigma (the sliced-ELLPACK idea of PAPER.md L527-531): every
    window of sigma consecutive rows is an independent pJDS matrix (pjds_reference on its rows),
    stored one after the other.  Returns the concatenation plus wstart (first stored slot of each
    window) and wcs_off (start of each window's col_start in the concatenated col_start)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    col = np.asarray(col)
    val = np.asarray(val)
    n_blocks = -(-n // b_r)
    n_pad = n_blocks * b_r
    if sigma <= 0 or sigma >= n_pad:
        P = pjds_reference(n, rowptr, col, val, b_r=b_r, symmetric=symmetric)
        P.update(wstart=np.array([0, P["stored"]], np.int64), wcs_off=np.array([0, P["width"] + 1], np.int64))
        return P
    parts = []
    for r0 in range(0, n_pad, sigma):
        r1 = min(n, r0 + sigma)
        m = max(r1 - r0, 0)
        sub_rp = rowptr[r0:r0 + m + 1] - rowptr[r0]
        W = pjds_reference(m, sub_rp, col[rowptr[r0]:rowptr[r0 + m]], val[rowptr[r0]:rowptr[r0 + m]], b_r=b_r)
        # the window's own padded row count (the last window may hold fewer blocks)
        nb_w = (min(n_pad, r0 + sigma) - r0) // b_r
        bl = np.zeros(nb_w, np.int32)
        bl[:W["n_blocks"]] = W["block_len"]
        W["block_len"] = bl
        W["perm"] = W["perm"] + r0
        parts.append(W)
    perm = np.concatenate([W["perm"] for W in parts]).astype(np.int32)
    invperm = np.empty(n, np.int32)
    invperm[perm] = np.arange(n, dtype=np.int32)
    out_col = np.concatenate([W["col"] for W in parts]).astype(np.int32)
    if symmetric and len(out_col):
        # padded slots keep column 0; real slots map through the global inverse permutation
        is_real = np.concatenate([_real_slots(W) for W in parts])
        out_col[is_real] = invperm[out_col[is_real]]
    stored = [W["stored"] for W in parts]
    wstart = np.zeros(len(parts) + 1, np.int64)
    np.cumsum(stored, out=wstart[1:])
    wcs_off = np.zeros(len(parts) + 1, np.int64)
    np.cumsum([W["width"] + 1 for W in parts], out=wcs_off[1:])
    return dict(perm=perm, invperm=invperm, block_len=np.concatenate([W["block_len"] for W in parts]),
                col_start=np.concatenate([W["col_start"] for W in parts]), val=np.concatenate([W["val"] for W in parts]),
                col=out_col, n=n, n_pad=n_pad, n_blocks=n_blocks, width=max(W["width"] for W in parts),
                stored=int(wstart[-1]), b_r=b_r, wstart=wstart, wcs_off=wcs_off, sigma=sigma)


def _real_slots(W):
    """Boolean mask over a pJDS matrix's slots: True where the slot holds a stored CRS entry."""
    mask = np.zeros(W["stored"], bool)
    lens = W["row_len_sorted"]
    for j in range(W["width"]):
        m = int(W["col_start"][j + 1] - W["col_start"][j])
        k = np.arange(m)
        mask[W["col_start"][j] + k] = lens[k] > j
    return mask


def ellr_reference(n, rowptr, col, val, warp: int = 32):
    """CRS -> ELLPACK-R, PAPER.md L146-159 (shift left, N x N^max rectangle, column-major,
    N padded to a multiple of the warp size, footnote L153-155) and L187-191 (rowmax[]).
    Padding = (+0.0, col 0) (reading 7); rowmax = 0 for pad rows (reading 16)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    val = np.asarray(val)
    col = np.asarray(col)
    lens = _lens(rowptr)
    n_pad = -(-n // warp) * warp
    width = int(lens.max()) if n else 0
    out_val = np.zeros(n_pad * width, dtype=val.dtype)
    out_col = np.zeros(n_pad * width, dtype=np.int32)
    rowmax = np.zeros(n_pad, dtype=np.int32)
    rowmax[:n] = lens
    for j in range(width):
        i = np.nonzero(lens > j)[0]
        out_val[j * n_pad + i] = val[rowptr[i] + j]
        out_col[j * n_pad + i] = col[rowptr[i] + j]
    return dict(rowmax=rowmax, val=out_val, col=out_col, n=n, n_pad=n_pad, width=width, stored=n_pad * width,
                warp=warp)


def listing1_spmv(E, x):
    """Literal Listing 1: c[i] += val[j*N + i] * rhs[col_idx[j*N + i]], j < rowmax[i].
    Pure-Python loops: small inputs only.  FMA-free, float64/32 as the arrays."""
    N = E["n_pad"]
    c = np.zeros(N, dtype=E["val"].dtype)
    for i in range(N):
        for j in range(int(E["rowmax"][i])):
            c[i] += E["val"][j * N + i] * x[E["col"][j * N + i]]
    return c[: E["n"]]


def listing2_spmv(P, x):
    """Literal Listing 2 in the permuted basis: for each (sorted) row i,
    c[i] += val[col_start[j] + i] * rhs[col_idx[col_start[j] + i]] for j < rowmax[i]
    (rowmax[i] = the row's own length; reading 6), then y[perm[i]] = c[i] (row-only basis, reading 9).
    Pure-Python loops: small inputs only."""
    n = P["n"]
    c = np.zeros(P["n_pad"], dtype=P["val"].dtype)
    rowmax = P["row_len_sorted"]
    for i in range(P["n_pad"]):
        for j in range(int(rowmax[i])):
            off = int(P["col_start"][j])
            c[i] += P["val"][off + i] * x[P["col"][off + i]]
    y = np.zeros(n, dtype=c.dtype)
    y[P["perm"]] = c[:n]
    return y


def footprint(P=None, E=None, value_bytes: int = 8):
    """Storage accounting (Table 1 "data reduction", L284-286 overhead).

    pJDS bytes: values + int32 indices + col_start (int64, width+1) + block_len (int32) + perm (int32).
    ELLPACK-R bytes: values + int32 indices + rowmax (int32, n_pad).
    data_reduction = 1 - stored_pJDS / (N_pad * N^max)   (entries basis, reading 17).
    """
    out = {}
    if P is not None:
        S = P["stored"]
        out["pjds"] = dict(stored=S, bytes_values=S * value_bytes, bytes_indices=S * 4,
                           bytes_aux=(P["width"] + 1) * 8 + P["n_blocks"] * 4 + P["n"] * 4)
        out["pjds"]["bytes_total"] = sum(v for k, v in out["pjds"].items() if k.startswith("bytes_"))
        ell_entries = (-(-P["n"] // 32) * 32) * P["width"]
        out["pjds"]["data_reduction_vs_ellpack"] = (1.0 - S / ell_entries) if ell_entries else 0.0
    if E is not None:
        S = E["stored"]
        out["ellr"] = dict(stored=S, bytes_values=S * value_bytes, bytes_indices=S * 4, bytes_aux=E["n_pad"] * 4)
        out["ellr"]["bytes_total"] = sum(v for k, v in out["ellr"].items() if k.startswith("bytes_"))
    return out


def utilisation(P=None, E=None, nnz: int = 0):
    """Fig. 2 counters, in lane-slots (one per row per j step).

    pJDS (our kernel loops to block_len, reading 6): useful = nnz, padded = stored - nnz, idle = 0.
    ELLPACK-R (warp of `warp` consecutive rows, loops to rowmax[i]): useful = nnz, padded = 0,
    idle = sum_warps sum_lanes (warp max rowmax - rowmax[i]).
    """
    out = {}
    if P is not None:
        out["pjds"] = dict(useful=nnz, padded=P["stored"] - nnz, idle=0)
    if E is not None:
        w = E["warp"]
        rm = E["rowmax"].astype(np.int64).reshape(-1, w) if E["n_pad"] else np.zeros((0, w), np.int64)
        idle = int((rm.max(axis=1, keepdims=True) - rm).sum()) if len(rm) else 0
        out["ellr"] = dict(useful=nnz, padded=0, idle=idle)
    return out
