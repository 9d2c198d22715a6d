"""Pins for oracle O5 (row partition, halo schedule, local/nonlocal split):
SPEC.md dist examples (L386-406): one rank == unsplit, block-diagonal split -> empty halos,
reassembly reproduces A, send/recv lengths pairwise symmetric; split result within the O2 bound of
the unsplit long-double result, and equal to a hand-computed split on G1."""
import numpy as np
import pytest

import inputs
import oracle
from conftest import g1_crs
from oracle import dist


def offsets_even(n, R):
    return np.array([n * r // R for r in range(R + 1)], dtype=np.int64)


def triples(n, rp, col, val):
    return sorted((i, int(col[k]), float(val[k])) for i in range(n) for k in range(rp[i], rp[i + 1]))


def test_one_rank_is_unsplit():
    n, rp, col, val, g = g1_crs()
    ranks = dist.split(n, rp, col, val, [0, n])
    assert len(ranks[0]["halo_cols"]) == 0 and ranks[0]["nl"][0] == 0
    nl, rp2, c2, v2 = ranks[0]["loc"]
    assert np.array_equal(rp2, rp) and np.array_equal(c2, col) and np.array_equal(v2, val)
    x = np.array(g["x"], dtype=np.float64)
    assert dist.spmv(ranks, x).tolist() == g["y"]


def test_g1_two_ranks_by_hand():
    """G1 split at row 3: rank 0 rows 0-2 (cols 0-2 local), rank 1 rows 3-5.
    rank 0: row1 has col 5 (owner 1) -> recv from 1 = [5]; row2 has col 3 -> recv [3,5].
    rank 1: row3 has col 1 (owner 0); row4 has col 2 -> recv from 0 = [1, 2]."""
    n, rp, col, val, g = g1_crs()
    r0, r1 = dist.split(n, rp, col, val, [0, 3, 6])
    assert [a.tolist() for a in r0["recv"]] == [[], [3, 5]]
    assert [a.tolist() for a in r1["recv"]] == [[1, 2], []]
    assert r0["send"][1].tolist() == [1, 2] and r1["send"][0].tolist() == [0, 2]
    assert r0["rows_nl"].tolist() == [1, 2] and r1["rows_nl"].tolist() == [0, 1]
    # rank 0 nonlocal part: row1 -> (slot of 5 = 1, val 4); row2 -> (slot of 3 = 0, val 6)
    m, rpn, cn, vn = r0["nl"]
    assert rpn.tolist() == [0, 1, 2] and cn.tolist() == [1, 0] and vn.tolist() == [4, 6]
    x = np.array(g["x"], dtype=np.float64)
    assert dist.spmv([r0, r1], x).tolist() == g["y"]


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
def test_random_split_invariants(R):
    n = 200
    _, rp, col, val = inputs.small("random", n, seed=R, max=25)
    offs = offsets_even(n, R)
    ranks = dist.split(n, rp, col, val, offs)
    # reassembly reproduces A entry for entry
    assert dist.reassemble(ranks, n) == triples(n, rp, col, val)
    # send/recv pairwise symmetric and duplicate-free
    for a in range(R):
        for b in range(R):
            assert len(ranks[a]["send"][b]) == len(ranks[b]["recv"][a])
            assert len(set(ranks[b]["recv"][a].tolist())) == len(ranks[b]["recv"][a])
            assert np.all((ranks[b]["recv"][a] >= offs[a]) & (ranks[b]["recv"][a] < offs[a + 1]))
        assert len(ranks[a]["recv"][a]) == 0
    # total halo = distinct nonlocal columns per rank
    for rk in ranks:
        c = col[rp[rk["lo"]]:rp[rk["hi"]]]
        assert len(rk["halo_cols"]) == len(set(int(v) for v in c if not rk["lo"] <= v < rk["hi"]))
    # split result within the O2 bound of the unsplit long-double result
    x = np.random.default_rng(R).uniform(-1, 1, n)
    y = dist.spmv(ranks, x)
    yl, b = oracle.spmv_ld(n, rp, col, val, x)
    assert oracle.acceptance(y, yl, b, np.diff(rp), np.float64).all()
    if R == 1:
        assert np.array_equal(y, oracle.spmv_chain(n, rp, col, val, x))


def test_block_diagonal_has_empty_halo():
    """SPEC.md L388/L395/L405: block-diagonal matrix split on block boundaries -> empty halos,
    nonlocal parts empty, result bitwise equal to the unsplit chain."""
    rng = np.random.default_rng(0)
    n, B = 96, 4
    rows = []
    for i in range(n):
        b = i // (n // B)
        rows.append(np.sort(rng.choice(np.arange(b * n // B, (b + 1) * n // B), 5, replace=False)))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    col = np.concatenate(rows).astype(np.int32)
    val = rng.uniform(-1, 1, len(col))
    ranks = dist.split(n, rp, col, val, offsets_even(n, B))
    for rk in ranks:
        assert len(rk["halo_cols"]) == 0 and rk["nl"][0] == 0
        assert all(len(s) == 0 for s in rk["send"])
    x = rng.uniform(-1, 1, n)
    assert np.array_equal(dist.spmv(ranks, x), oracle.spmv_chain(n, rp, col, val, x))


def test_hmep_banded_split():
    g = inputs.Generator.from_config("C1")
    rp, col, val = g.crs()
    n = g.n
    x = inputs.vector(n)
    for R in (2, 4):
        ranks = dist.split(n, rp, col, val, offsets_even(n, R))
        y = dist.spmv(ranks, x)
        yl, b = oracle.spmv_ld(n, rp, col, val, x)
        assert oracle.acceptance(y, yl, b, np.diff(rp), np.float64).all()
        # block hops cross ranks as whole length-1024 segments
        for rk in ranks:
            assert len(rk["halo_cols"]) % 1024 == 0
