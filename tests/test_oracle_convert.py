"""Pins for oracle O4 (reference pJDS / ELLPACK-R converters, Listing 1/2 emulations, footprint,
utilisation counters): the hand-derived G1 example, the paper's closed forms
(PAPER.md L256-266), SPEC acceptance 1/2, and invariants checked by independent
recounts."""
from collections import Counter

import numpy as np
import pytest

import inputs
from conftest import g1_crs
from oracle import convert


def test_g1_pjds_br2_br4():
    n, rp, col, val, g = g1_crs()
    for key, br in (("pjds_br2", 2), ("pjds_br4", 4)):
        P = convert.pjds_reference(n, rp, col, val, b_r=br)
        exp = g[key]
        assert P["perm"].tolist() == exp["perm"]
        assert P["block_len"].tolist() == exp["block_len"]
        assert P["col_start"].tolist() == exp["col_start"]
        assert P["val"].tolist() == exp["val"]
        assert P["col"].tolist() == exp["col"]
        assert P["stored"] == exp["stored"]
        E = convert.ellr_reference(n, rp, col, val, warp=br)
        assert E["stored"] == exp["ellpack_stored"]
        x = np.array(g["x"], dtype=np.float64)
        assert convert.listing2_spmv(P, x).tolist() == g["y"]


def test_g1_ellr_warp2():
    n, rp, col, val, g = g1_crs()
    E = convert.ellr_reference(n, rp, col, val, warp=2)
    exp = g["ellr_warp2"]
    assert E["rowmax"].tolist() == exp["rowmax"]
    assert E["val"].tolist() == exp["val"]
    assert E["col"].tolist() == exp["col"]
    assert E["width"] == exp["width"] and E["stored"] == exp["stored"]
    assert convert.listing1_spmv(E, np.array(g["x"], dtype=np.float64)).tolist() == g["y"]
    # library convention N_pad = 32: same arrays, each jagged column zero-extended
    E32 = convert.ellr_reference(n, rp, col, val, warp=32)
    for j in range(3):
        assert E32["val"][32 * j:32 * j + 6].tolist() == exp["val"][6 * j:6 * j + 6]
        assert not E32["val"][32 * j + 6:32 * (j + 1)].any()


def test_adversarial_closed_form():
    """one full row + single entries -> ELLPACK N x N, pJDS (b_r+1) N - b_r.
    SPEC.md L471 acceptance 1: N = 1024, b_r = 32 -> 33760; L160 reduction ~ 0.9678."""
    n = 1024
    _, rp, col, val = inputs.small("adversarial", n, seed=1)
    P = convert.pjds_reference(n, rp, col, val, b_r=32)
    E = convert.ellr_reference(n, rp, col, val, warp=32)
    assert P["stored"] == 33 * 1024 - 32 == 33760
    assert E["stored"] == 1024 * 1024
    fp = convert.footprint(P, E)
    assert fp["pjds"]["data_reduction_vs_ellpack"] == pytest.approx(1 - 33760 / 1024 ** 2, abs=0)
    assert round(fp["pjds"]["data_reduction_vs_ellpack"], 4) == 0.9678
    for br in (1, 2, 4, 8, 64):
        assert convert.pjds_reference(n, rp, col, val, b_r=br)["stored"] == (br + 1) * n - br


@pytest.mark.parametrize("k", [1, 7, 15, 144])
def test_constant_zero_overhead(k):
    """constant row length -> no storage overhead."""
    n = 320
    _, rp, col, val = inputs.small("constant", n, seed=k, k=k)
    for br in (1, 3, 32, 64):
        P = convert.pjds_reference(n, rp, col, val, b_r=br)
        n_pad = -(-n // br) * br
        assert P["stored"] == n_pad * k
        if n % br == 0:
            assert P["stored"] == n * k  # nothing but the non-zeros
    E = convert.ellr_reference(n, rp, col, val)
    assert E["stored"] == n * k


def _check_invariants(n, rp, col, val, br):
    P = convert.pjds_reference(n, rp, col, val, b_r=br)
    lens = np.diff(rp)
    perm = P["perm"]
    # perm is a bijection on [0, n)
    assert sorted(perm.tolist()) == list(range(n))
    # sorted lengths non-increasing; ties in ascending original index (stable)
    sl = lens[perm]
    assert np.all(sl[:-1] >= sl[1:])
    for a in range(n - 1):
        if sl[a] == sl[a + 1]:
            assert perm[a] < perm[a + 1]
    # block_len: max of its block, non-increasing
    bl = P["block_len"]
    for b in range(P["n_blocks"]):
        rows = [int(lens[perm[k]]) for k in range(b * br, min(n, (b + 1) * br))]
        assert bl[b] == (max(rows) if rows else 0)
    assert np.all(bl[:-1] >= bl[1:])
    # col_start recount: slots in column j = rows whose block is padded beyond j
    for j in range(P["width"]):
        cnt = sum(br for b in range(P["n_blocks"]) if bl[b] > j)
        assert P["col_start"][j + 1] - P["col_start"][j] == cnt
    assert P["col_start"][-1] == P["stored"] == br * int(bl.sum())
    # entry multiset preserved; padding is (+0.0, 0) and only in padded slots
    got = Counter()
    pad = 0
    for k in range(P["n_pad"]):
        b = k // br
        for j in range(int(bl[b])):
            off = int(P["col_start"][j]) + k
            if k < n and j < lens[perm[k]]:
                got[(int(perm[k]), int(P["col"][off]), float(P["val"][off]))] += 1
            else:
                assert P["col"][off] == 0 and P["val"][off] == 0 and not np.signbit(P["val"][off])
                pad += 1
    want = Counter((i, int(col[k]), float(val[k])) for i in range(n) for k in range(rp[i], rp[i + 1]))
    assert got == want
    assert pad == P["stored"] - len(col)
    # row order kept (CRS order within a row, reading 8)
    for k in range(n):
        r = perm[k]
        seq = [int(P["col"][int(P["col_start"][j]) + k]) for j in range(lens[r])]
        assert seq == col[rp[r]:rp[r + 1]].tolist()
    # determinism
    P2 = convert.pjds_reference(n, rp, col, val, b_r=br)
    assert all(np.array_equal(P[k], P2[k]) for k in ("perm", "block_len", "col_start", "val", "col"))
    # storage ordering: pJDS <= ELLPACK-R at warp = b_r
    assert P["stored"] <= convert.ellr_reference(n, rp, col, val, warp=br)["stored"]
    return P


@pytest.mark.parametrize("kind", ["uniform", "clustered", "empty_rows", "duplicates", "random", "banded"])
@pytest.mark.parametrize("br", [1, 2, 4, 32])
def test_pjds_invariants(kind, br):
    for seed in range(3):
        n = [1, 31, 70][seed]
        _, rp, col, val = inputs.small(kind, n, seed=seed)
        _check_invariants(n, rp, col, val, br)


def test_empty_matrix():
    P = convert.pjds_reference(0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0), b_r=32)
    assert P["stored"] == 0 and P["n_blocks"] == 0 and P["col_start"].tolist() == [0]
    E = convert.ellr_reference(0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    assert E["stored"] == 0


@pytest.mark.parametrize("kind", ["uniform", "empty_rows", "duplicates", "random"])
def test_listings_reproduce_dense_product(kind):
    """Listing 1 / Listing 2 applied to the converted arrays equal the exact dense product
    (integer-valued entries keep every operation exact)."""
    n = 45
    _, rp, col, _ = inputs.small(kind, n, seed=9)
    rng = np.random.default_rng(1)
    val = rng.integers(-20, 21, size=len(col)).astype(np.float64)
    x = rng.integers(-20, 21, size=n).astype(np.float64)
    ex = [0] * n
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            ex[i] += int(val[k]) * int(x[col[k]])
    for br in (1, 4, 32):
        assert convert.listing2_spmv(convert.pjds_reference(n, rp, col, val, b_r=br), x).tolist() == ex
    assert convert.listing1_spmv(convert.ellr_reference(n, rp, col, val, warp=4), x).tolist() == ex


def test_symmetric_mode_is_PAPt():
    n = 40
    _, rp, col, val = inputs.small("uniform", n, seed=4)
    P = convert.pjds_reference(n, rp, col, val, b_r=4, symmetric=True)
    rng = np.random.default_rng(2)
    val_i = rng.integers(-9, 10, size=len(col)).astype(np.float64)
    P = convert.pjds_reference(n, rp, col, val_i, b_r=4, symmetric=True)
    x = rng.integers(-9, 10, size=n).astype(np.float64)
    # (P A P^T)(P x) = P (A x): in the permuted basis x_perm[k] = x[perm[k]]
    x_perm = x[P["perm"]]
    c = np.zeros(P["n_pad"])
    for k in range(P["n_pad"]):
        for j in range(int(P["row_len_sorted"][k])):
            off = int(P["col_start"][j]) + k
            c[k] += P["val"][off] * x_perm[P["col"][off]]
    ex = np.zeros(n)
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            ex[i] += val_i[k] * x[col[k]]
    assert c[:n].tolist() == ex[P["perm"]].tolist()


def test_utilisation_counters():
    """Fig. 2: ELLPACK-R idle lane slots = sum over warps of (warp max - len),
    recounted directly; pJDS padded slots = stored - nnz."""
    n, rp, col, val, _ = g1_crs()
    E = convert.ellr_reference(n, rp, col, val, warp=2)
    u = convert.utilisation(convert.pjds_reference(n, rp, col, val, b_r=2), E, nnz=len(col))
    # warps (rows 0,1): max 3 -> idle 2+0; (2,3): max 3 -> 1+0; (4,5): max 2 -> 0+1
    assert u["ellr"] == dict(useful=12, padded=0, idle=4)
    assert u["pjds"] == dict(useful=12, padded=0, idle=0)
    P4 = convert.pjds_reference(n, rp, col, val, b_r=4)
    assert convert.utilisation(P4, None, nnz=12)["pjds"]["padded"] == 4


def test_footprint_bytes():
    n, rp, col, val, _ = g1_crs()
    P = convert.pjds_reference(n, rp, col, val, b_r=2)
    fp = convert.footprint(P, convert.ellr_reference(n, rp, col, val), value_bytes=8)
    assert fp["pjds"]["bytes_values"] == 96 and fp["pjds"]["bytes_indices"] == 48
    assert fp["pjds"]["bytes_aux"] == 4 * 8 + 3 * 4 + 6 * 4
    assert fp["ellr"]["stored"] == 32 * 3 and fp["ellr"]["bytes_aux"] == 32 * 4


def test_paper_shaped_reductions():
    """Table 1 data reductions pin only the generator shapes; recorded here so a
    generator change is noticed: C1 17.8 %, C2 ~68.3 %, C3 31.7 %, C4 ~17.2 %."""
    for name, lo, hi in (("C1", 0.177, 0.178), ("C3", 0.317, 0.318), ("C4", 0.170, 0.175)):
        g = inputs.Generator.from_config(name)
        lens = g.rowlen()
        n = g.n
        s = np.zeros(-(-n // 32) * 32, np.int64)
        s[:n] = np.sort(lens)[::-1]
        stored = 32 * int(s.reshape(-1, 32).max(axis=1).sum())
        red = 1 - stored / (len(s) * lens.max())
        assert lo <= red <= hi, (name, red)
