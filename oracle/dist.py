"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

O5: CPU emulation of the row-partitioned distributed spMVM of PAPER.md §3 (L428-461):
contiguous row partition, split of each rank's rows into a local and a nonlocal part
("The spMVM must be split into a local and a nonlocal part", L442-444), the halo schedule
("local gather ... collection of data to be sent to other processes into a contiguous buffer",
Fig. 4 caption L401-402), and the two-pass result ("the result vector must be written twice",
L445).  Schedule conventions (readings 22-23):

  * rank r owns rows and x entries [off[r], off[r+1]) (square matrix);
  * recv list from owner q = sorted unique global columns owned by q referenced by r's rows;
  * halo slot = position in the concatenation of the recv lists ordered by owner rank;
  * send list r -> q = q's recv list from r, as r-local indices;
  * A_loc: all n_loc rows, only local entries (local column ids), CRS order kept;
  * A_nl : only the rows with >= 1 nonlocal entry, ascending local row order, halo-slot columns;
  * combine: y_i = chain(A_loc row i) then y_i = y_i + chain(A_nl row i) (one rounding add),
    rows without nonlocal entries untouched.
"""
from __future__ import annotations

import numpy as np

from . import spmv_chain


def split(n, rowptr, col, val, offsets):
    """Partition + halo schedule + local/nonlocal CRS parts for every rank (list of dicts)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    R = len(offsets) - 1
    assert offsets[0] == 0 and offsets[-1] == n and np.all(np.diff(offsets) >= 0)
    rowptr = np.asarray(rowptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    val = np.asarray(val)
    owner_of = np.searchsorted(offsets, np.arange(n), side="right") - 1 if n else np.zeros(0, np.int64)
    ranks = []
    for r in range(R):
        lo, hi = int(offsets[r]), int(offsets[r + 1])
        nl = hi - lo
        rp = rowptr[lo:hi + 1] - rowptr[lo]
        c = col[rowptr[lo]:rowptr[hi]]
        v = val[rowptr[lo]:rowptr[hi]]
        row_of = np.repeat(np.arange(nl), np.diff(rp))
        is_loc = (c >= lo) & (c < hi)
        # recv lists per owner (sorted unique global ids), halo slot numbering by owner rank
        remote = np.unique(c[~is_loc])
        rem_owner = owner_of[remote] if len(remote) else np.zeros(0, np.int64)
        recv = [remote[rem_owner == q] for q in range(R)]
        halo_cols = np.concatenate(recv) if R else np.zeros(0, np.int64)  # already owner-ordered
        slot_of = {int(g): s for s, g in enumerate(halo_cols)}
        # A_loc: every row, local entries only, CRS order kept
        loc_len = np.bincount(row_of[is_loc], minlength=nl) if nl else np.zeros(0, np.int64)
        loc_rp = np.zeros(nl + 1, dtype=np.int64)
        np.cumsum(loc_len, out=loc_rp[1:])
        loc_col = (c[is_loc] - lo).astype(np.int32)
        loc_val = v[is_loc]
        # A_nl: rows with >= 1 nonlocal entry, ascending local row order
        nl_len_all = np.bincount(row_of[~is_loc], minlength=nl) if nl else np.zeros(0, np.int64)
        rows_nl = np.nonzero(nl_len_all)[0].astype(np.int32)
        nl_rp = np.zeros(len(rows_nl) + 1, dtype=np.int64)
        np.cumsum(nl_len_all[rows_nl], out=nl_rp[1:])
        nl_col = np.array([slot_of[int(g)] for g in c[~is_loc]], dtype=np.int32)
        nl_val = v[~is_loc]
        ranks.append(dict(rank=r, lo=lo, hi=hi, n_loc=nl, recv=recv, halo_cols=halo_cols,
                          loc=(nl, loc_rp, loc_col, loc_val), rows_nl=rows_nl,
                          nl=(len(rows_nl), nl_rp, nl_col, nl_val)))
    # send lists: r -> q is q's recv list from r, as r-local ids
    for r in range(R):
        ranks[r]["send"] = [(ranks[q]["recv"][r] - ranks[r]["lo"]).astype(np.int32) for q in range(R)]
    return ranks


def spmv(ranks, x):
    """Two-pass split spMVM over all ranks (FMA chains, SURVEY §8(c) O3 combine); gathered y."""
    x = np.asarray(x)
    n = ranks[-1]["hi"] if ranks else 0
    y = np.zeros(n, dtype=x.dtype)
    for rk in ranks:
        lo, hi = rk["lo"], rk["hi"]
        x_loc = x[lo:hi]
        halo = x[rk["halo_cols"]]
        nl, rp, c, v = rk["loc"]
        y_loc = spmv_chain(nl, rp, c, v, x_loc) if nl else np.zeros(0, x.dtype)
        m, rp2, c2, v2 = rk["nl"]
        if m:
            y_nl = spmv_chain(m, rp2, c2, v2, halo)
            y_loc[rk["rows_nl"]] = y_loc[rk["rows_nl"]] + y_nl
        y[lo:hi] = y_loc
    return y


def reassemble(ranks, n):
    """Rebuild the global (row, col, val) triples from the split parts (pin: split loses nothing)."""
    trip = []
    for rk in ranks:
        lo = rk["lo"]
        nl, rp, c, v = rk["loc"]
        for i in range(nl):
            for k in range(rp[i], rp[i + 1]):
                trip.append((lo + i, lo + int(c[k]), float(v[k])))
        m, rp2, c2, v2 = rk["nl"]
        for a in range(m):
            i = int(rk["rows_nl"][a])
            for k in range(rp2[a], rp2[a + 1]):
                trip.append((lo + i, int(rk["halo_cols"][c2[k]]), float(v2[k])))
    return sorted(trip)
