"""Input recipe checks: the synthetic generators reproduce the paper's workload numbers
(SURVEY §8(d) sizes) and are deterministic and row-range consistent."""
import numpy as np

import inputs


def test_config_sizes():
    exp = {"C1": (16384, 256000, 12, 19), "C3": (6201600, 97365120, 6, 23), "C4": (278502, None, 90, 174)}
    for name, (n, nnz, lo, hi) in exp.items():
        g = inputs.Generator.from_config(name)
        lens = g.rowlen()
        assert g.n == n
        if nnz is not None:
            assert int(lens.sum()) == nnz
        assert lens.min() == lo and lens.max() == hi
    g = inputs.Generator.from_config("C2")
    lens = g.rowlen()
    assert g.n == 3397500 and lens.min() == 4 and lens.max() == 22
    assert 6.9 < lens.mean() < 7.0                       # N_nzr ~ 7
    g = inputs.Generator.from_config("C4")
    lens = g.rowlen()
    assert 143.5 < lens.mean() < 144.5                   # N_nzr ~ 144
    assert np.mean(lens >= 0.8 * lens.max()) > 0.75      # "80% of the rows ... 0.8 N^max" (L272-274)


def test_c5_size():
    g = inputs.Generator.from_config("C5")
    assert g.n == 57002400
    lens = g.rowlen(0, 2_000_000)
    assert lens.min() >= 6 and lens.max() <= 23


def test_hmep_contiguous_offdiagonals():
    """contiguous off-diagonals of length ~15,000 (here P = 15,504)."""
    g = inputs.Generator(inputs.HMEP, 3, 0)  # M = 3: P = C(8,5) = 56
    rp, col, val = g.crs()
    P = 56
    assert g.n == 400 * P
    rows = np.repeat(np.arange(g.n), np.diff(rp))
    off = col.astype(np.int64) - rows
    # every inter-block offset (a multiple of P) appears on a whole block of P consecutive rows
    for d in np.unique(off[np.abs(off) >= P]):
        assert d % P == 0
        r = rows[off == d]
        assert len(r) % P == 0


def test_determinism_and_ranges():
    g = inputs.Generator.from_config("C1")
    a = g.crs()
    b = g.crs()
    assert all(np.array_equal(u, v) for u, v in zip(a, b))
    rp, col, val = a
    rp2, col2, val2 = g.crs(5000, 9000)
    assert np.array_equal(col2, col[rp[5000]:rp[9000]])
    assert np.array_equal(val2, val[rp[5000]:rp[9000]])
    x = inputs.vector(1000)
    assert np.array_equal(inputs.vector(100, i0=300), x[300:400])
    assert np.all((x >= -1) & (x < 1))
    f = g.crs(dtype=np.float32)[2]
    assert np.array_equal(f, val.astype(np.float32))
    # sorted, in-range, duplicate-free columns per row
    for i in range(0, g.n, 997):
        c = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < g.n
