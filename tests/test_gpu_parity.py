"""GPU parity of the CUDA path (through the C ABI) against the oracle, on the same seeded inputs.

Bars:
  * conversion / permutation: bit-exact (device export == oracle/convert.py);
  * y: every row within the north-star bound |y - y_ref| <= 4 nnz_i eps sum|a_ij x_j| of the
    long-double oracle (O2), AND equal to the oracle's FMA-chain emulation (O3) — the kernels keep
    one fused chain per row in CRS order, so equality is exact (+-0 compare equal);
  * dist (local+nonlocal split, LOCAL transport on one GPU): equal to oracle/dist.py and within O2.
"""
import numpy as np
import pytest

import inputs
import oracle
from oracle import convert, dist as odist

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pj():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1112_5588_b200 as pj
    pj.lib()
    return pj


def tdev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check_y(y_gpu, n, rp, col, val, x, exact=True):
    y_gpu = np.asarray(y_gpu)
    y_ref, bound = oracle.spmv_ld(n, rp, col, val, x)
    ok = oracle.acceptance(y_gpu, y_ref, bound, np.diff(rp), val.dtype)
    assert ok.all(), f"{(~ok).sum()} rows outside the O2 bound, first {np.nonzero(~ok)[0][:5]}"
    if exact:
        chain = oracle.spmv_chain(n, rp, col, val, x)
        bad = np.nonzero(y_gpu != chain)[0]
        assert len(bad) == 0, f"{len(bad)} rows differ from the FMA-chain emulation, first {bad[:5]}"


SMALL = [("uniform", 1000, {}), ("clustered", 777, {}), ("empty_rows", 513, {}), ("duplicates", 300, {}),
         ("random", 1500, dict(max=90)), ("adversarial", 1024, {}), ("constant", 96, dict(k=7)), ("zero", 70, {}),
         ("identity", 31, {}), ("banded", 2049, {}),
         ("adversarial", 3000, {})]  # width 3000 > the 1024 col_start entries staged in shared memory


@pytest.mark.parametrize("kind,n,kw", SMALL)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("br", [32, 64, 96, 128, 160])
def test_pjds_small(pj, kind, n, kw, dtype, br):
    _, rp, col, val = inputs.small(kind, n, seed=br + n, dtype=dtype, **kw)
    x = inputs.vector(n, dtype)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br)
    y = torch.full((n,), float("nan"), dtype=torch.float64 if dtype == np.float64 else torch.float32, device="cuda")
    A.spmv(y, tdev(x))
    torch.cuda.synchronize()
    check_y(y.cpu().numpy(), n, rp, col, val, x)
    # uploaded arrays are the oracle's, bit for bit
    got = A.export()
    P = convert.pjds_reference(n, rp, col, val, b_r=br)
    assert np.array_equal(got["col"], P["col"]) and got["val"].tobytes() == P["val"].tobytes()


@pytest.mark.parametrize("kind,n,kw", SMALL)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_ellr_small(pj, kind, n, kw, dtype):
    _, rp, col, val = inputs.small(kind, n, seed=n, dtype=dtype, **kw)
    x = inputs.vector(n, dtype)
    E = pj.EllrMatrix.from_crs(n, rp, col, val)
    y = torch.full((n,), float("nan"), dtype=torch.float64 if dtype == np.float64 else torch.float32, device="cuda")
    E.spmv(y, tdev(x))
    torch.cuda.synchronize()
    check_y(y.cpu().numpy(), n, rp, col, val, x)


def test_g1_golden_on_gpu(pj):
    from conftest import g1_crs
    n, rp, col, val, g = g1_crs()
    x = np.array(g["x"], dtype=np.float64)
    for br in (32, 64):
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br)
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        A.spmv(y, tdev(x))
        assert y.cpu().tolist() == g["y"]
    E = pj.EllrMatrix.from_crs(n, rp, col, val)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    E.spmv(y, tdev(x))
    assert y.cpu().tolist() == g["y"]


@pytest.mark.parametrize("name", ["C1", "C4", "C2", "C3"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_configs_full(pj, name, dtype):
    """Full-size paper-shaped configs, every row checked (oracle in C, OpenMP over rows)."""
    n, rp, col, val = inputs.config_crs(name, dtype=dtype)
    x = inputs.vector(n, dtype)
    xt = tdev(x)
    for br in (32, 64):
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br)
        y = torch.empty(n, dtype=xt.dtype, device="cuda")
        A.spmv(y, xt)
        torch.cuda.synchronize()
        check_y(y.cpu().numpy(), n, rp, col, val, x)
        del A
    # the bench's basis: x permuted once, y in the permuted basis, direct
    # vector store; automatic variant and tile order as bench.py / per_config launch them
    for br in (32, 128):
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, symmetric=True)
        xp = A.to_permuted(torch.empty_like(xt), xt)
        yp = torch.full((n,), float("nan"), dtype=xt.dtype, device="cuda")
        A.spmv(yp, xp)
        y = A.from_permuted(torch.empty_like(yp), yp)
        torch.cuda.synchronize()
        check_y(y.cpu().numpy(), n, rp, col, val, x)
        del A
    E = pj.EllrMatrix.from_crs(n, rp, col, val)
    y = torch.empty(n, dtype=xt.dtype, device="cuda")
    E.spmv(y, xt)
    torch.cuda.synchronize()
    check_y(y.cpu().numpy(), n, rp, col, val, x)


def c5_sampled_rows(g, n, rp):
    """>= 100 K sampled C5 rows: 100 random chunks of 1000 consecutive rows (all length classes of a
    region, i.e. whole CTA tiles of several lengths) + 20 K uniformly random rows + first/last."""
    rng = np.random.default_rng(5)
    starts = rng.integers(0, n - 1000, 100)
    rows = np.unique(np.concatenate([(starts[:, None] + np.arange(1000)[None, :]).ravel(),
                                     rng.integers(0, n, 20000), [0, n - 1]]))
    return rows


def oracle_of_rows(g, rows, rp, dtype):
    """The sampled rows regenerated from inputs/ as one CRS (the oracle's own copy)."""
    lens = np.diff(rp)
    srp = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lens[rows], out=srp[1:])
    sc = np.empty(srp[-1], np.int32)
    sv = np.empty(srp[-1], dtype)
    # contiguous runs of sampled rows are generated in one call each
    brk = np.nonzero(np.diff(rows) != 1)[0] + 1
    for run in np.split(np.arange(len(rows)), brk):
        r0, r1 = int(rows[run[0]]), int(rows[run[-1]]) + 1
        _, cc, vv = g.crs(r0, r1, dtype=dtype)
        sc[srp[run[0]]:srp[run[-1] + 1]] = cc
        sv[srp[run[0]]:srp[run[-1] + 1]] = vv
    return srp, sc, sv


def test_c5_sampled(pj):
    """C5 (bench workload, 942 M nnz) in the ORIGINAL basis (row-only permutation, y stored through
    perm: the §8 default basis, bench compare leg `pjds_rows_only`): sampled rows vs the oracle."""
    g = inputs.Generator.from_config("C5")
    rp, col, val = g.crs()
    n = g.n
    x = inputs.vector(n)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=32)
    del col, val
    xt = tdev(x)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    A.spmv(y, xt)
    torch.cuda.synchronize()
    yh = y.cpu().numpy()
    rows = np.unique(np.concatenate([np.random.default_rng(0).integers(0, n, 20000), [0, n - 1]]))
    lens = np.diff(rp)
    srp = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lens[rows], out=srp[1:])
    sc = np.empty(srp[-1], np.int32)
    sv = np.empty(srp[-1])
    rp2, col2, val2 = None, None, None
    for a, r in enumerate(rows):
        rr, cc, vv = g.crs(int(r), int(r) + 1)
        sc[srp[a]:srp[a + 1]] = cc
        sv[srp[a]:srp[a + 1]] = vv
    y_ref, bound = oracle.spmv_ld(len(rows), srp, sc, sv, x)
    assert oracle.acceptance(yh[rows], y_ref, bound, lens[rows], np.float64).all()
    assert np.array_equal(yh[rows], oracle.spmv_chain(len(rows), srp, sc, sv, x))
    # property at full size: y is finite everywhere
    assert np.isfinite(yh).all()


@pytest.mark.parametrize("dtype,br", [(np.float64, 128), (np.float32, 128), (np.float64, 32)])
def test_c5_permuted_bench_instance(pj, dtype, br):
    """The exact headline instance of bench.py: C5, permuted basis (PJDS_PERM_SYMMETRIC), b_r = 128
    (the bench default since round 2; 32 = the library default, also checked),
    automatic variant (R = 4, U = 2), automatic tile order (original-row order: x > 64 MB), vector
    y store.  >= 100 K sampled rows against O1 at the O2 bound AND bitwise against the O3 chain (one
    FMA chain per row in CRS order, Listing 2); all rows finite."""
    g = inputs.Generator.from_config("C5")
    rp, col, val = g.crs(dtype=dtype)
    n = g.n
    x = inputs.vector(n, dtype)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, symmetric=True)
    del col, val
    assert A.symmetric
    xt = tdev(x)
    xp = A.to_permuted(torch.empty_like(xt), xt)
    yp = torch.full((n,), float("nan"), dtype=xt.dtype, device="cuda")
    for _ in range(2):  # the bench times back-to-back launches on the same x / y
        A.spmv(yp, xp)
    y = A.from_permuted(torch.empty_like(yp), yp)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(y).all())
    rows = c5_sampled_rows(g, n, rp)
    assert len(rows) >= 100_000
    yh = y.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    srp, sc, sv = oracle_of_rows(g, rows, rp, dtype)
    y_ref, bound = oracle.spmv_ld(len(rows), srp, sc, sv, x)
    ok = oracle.acceptance(yh, y_ref, bound, np.diff(srp), dtype)
    assert ok.all(), f"{(~ok).sum()} sampled rows outside O2"
    chain = oracle.spmv_chain(len(rows), srp, sc, sv, x)
    bad = np.nonzero(yh != chain)[0]
    assert len(bad) == 0, f"{len(bad)} sampled rows differ from the O3 chain, first {rows[bad[:5]]}"


def test_spmv_host_e2e(pj):
    n, rp, col, val = inputs.config_crs("C1")
    x = inputs.vector(n)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val)
    y = np.empty(n)
    A.spmv_host(y, x)
    check_y(y, n, rp, col, val, x)


def test_symmetric_mode(pj):
    n = 3000
    _, rp, col, val = inputs.small("random", n, seed=11, max=40)
    x = inputs.vector(n)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
    perm = A.export()["perm"]
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    A.spmv(y, tdev(x[perm]))  # x in the permuted basis
    yp = y.cpu().numpy()
    y_orig = np.empty(n)
    y_orig[perm] = yp
    check_y(y_orig, n, rp, col, val, x)


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("permuted", [False, True])
@pytest.mark.parametrize("nl_sigma,br", [(1024, 32), (0, 32), (2048, 128)])
def test_dist_group_random(pj, R, permuted, nl_sigma, br):
    """The split path against the O5 emulator, bitwise: A_nl in y-target order with 1024 / 2048-row
    sort windows (the default, reading 27) or globally sorted, b_r 32 and 128."""
    n = 4000
    _, rp, col, val = inputs.small("random", n, seed=R, max=50)
    x = inputs.vector(n)
    offs = np.array([n * r // R for r in range(R + 1)], np.int64)
    L = pj.lib()
    assert L.pjds_set_dist_nl_sigma(nl_sigma) == 0
    try:
        hs = pj.DistPjds.create_group(n, rp, col, val, offs, permuted=permuted, block_rows=br)
    finally:
        L.pjds_set_dist_nl_sigma(1024)
    xs = [tdev(x[offs[r]:offs[r + 1]]) for r in range(R)]
    if permuted:
        xs = [h.to_permuted(torch.empty_like(v), v) for h, v in zip(hs, xs)]
    ys = [torch.full((offs[r + 1] - offs[r],), float("nan"), dtype=torch.float64, device="cuda") for r in range(R)]
    pj.DistPjds.group_spmv(hs, ys, xs)
    if permuted:
        ys = [h.from_permuted(torch.empty_like(v), v) for h, v in zip(hs, ys)]
    torch.cuda.synchronize()
    y = np.concatenate([t.cpu().numpy() for t in ys])
    parts = odist.split(n, rp, col, val, offs)
    ref = odist.spmv(parts, x)
    assert np.array_equal(y, ref)
    check_y(y, n, rp, col, val, x, exact=(R == 1))
    # pjds_dist_stats: per-peer halo sizes equal the emulator's recv / send lists
    for r, h in enumerate(hs):
        st = h.stats()
        assert st["recv_per_peer"] == [len(v) for v in parts[r]["recv"]]
        assert st["send_per_peer"] == [len(v) for v in parts[r]["send"]]
        assert sum(st["recv_per_peer"]) == st["halo"] and sum(st["send_per_peer"]) == st["send_total"]


@pytest.mark.parametrize("permuted", [False, True])
def test_dist_group_empty_ranks(pj, permuted):
    """Ranks owning no rows (repeated offsets) take part with empty local/nonlocal parts."""
    n = 2000
    _, rp, col, val = inputs.small("random", n, seed=8, max=40)
    x = inputs.vector(n)
    offs = np.array([0, 0, 700, 700, 2000, 2000], np.int64)
    R = len(offs) - 1
    hs = pj.DistPjds.create_group(n, rp, col, val, offs, permuted=permuted)
    xs = [tdev(x[offs[r]:offs[r + 1]]) for r in range(R)]
    if permuted:
        xs = [h.to_permuted(torch.empty_like(v), v) for h, v in zip(hs, xs)]
    ys = [torch.full((int(offs[r + 1] - offs[r]),), float("nan"), dtype=torch.float64, device="cuda") for r in range(R)]
    pj.DistPjds.group_spmv(hs, ys, xs)
    if permuted:
        ys = [h.from_permuted(torch.empty_like(v), v) for h, v in zip(hs, ys)]
    torch.cuda.synchronize()
    y = np.concatenate([t.cpu().numpy() for t in ys])
    assert np.array_equal(y, odist.spmv(odist.split(n, rp, col, val, offs), x))


@pytest.mark.parametrize("name,R,permuted", [("C1", 4, False), ("C1", 4, True), ("C3", 4, False), ("C3", 8, True)])
def test_dist_group_configs(pj, name, R, permuted):
    n, rp, col, val = inputs.config_crs(name)
    x = inputs.vector(n)
    blk = 1024 if name == "C1" else 15504
    nb = n // blk
    offs = np.array([(nb * r // R) * blk for r in range(R + 1)], np.int64)
    hs = pj.DistPjds.create_group(n, rp, col, val, offs, permuted=permuted)
    for h in hs:
        if not permuted:
            assert h.info["packed_send"] == 0  # HMEp halos are whole segments: sent straight from x
    xs = [tdev(x[offs[r]:offs[r + 1]]) for r in range(R)]
    if permuted:
        xs = [h.to_permuted(torch.empty_like(v), v) for h, v in zip(hs, xs)]
    ys = [torch.empty(int(offs[r + 1] - offs[r]), dtype=torch.float64, device="cuda") for r in range(R)]
    pj.DistPjds.group_spmv(hs, ys, xs)
    if permuted:
        ys = [h.from_permuted(torch.empty_like(v), v) for h, v in zip(hs, ys)]
    torch.cuda.synchronize()
    y = np.concatenate([t.cpu().numpy() for t in ys])
    check_y(y, n, rp, col, val, x, exact=False)
    ref = odist.spmv(odist.split(n, rp, col, val, offs), x) if name == "C1" else None
    if ref is not None:
        assert np.array_equal(y, ref)


def test_bw_probe_and_launch_count(pj):
    c0 = pj.launch_count()
    copy, read = pj.bw_probe(1 << 30, 3)
    assert 1000 < copy < 10000 and 1000 < read < 10000
    assert pj.launch_count() > c0


def test_empty_matrix(pj):
    """n = 0 (n = 0 accepted): create, spmv with empty (possibly NULL) vectors, info."""
    rp = np.zeros(1, np.int64)
    col = np.zeros(0, np.int32)
    for dt in (np.float64, np.float32):
        val = np.zeros(0, dt)
        tdt = torch.float64 if dt == np.float64 else torch.float32
        x = torch.empty(0, dtype=tdt, device="cuda")
        y = torch.empty(0, dtype=tdt, device="cuda")
        A = pj.PjdsMatrix.from_crs(0, rp, col, val)
        assert A.info["n"] == 0 and A.info["stored"] == 0
        A.spmv(y, x)
        E = pj.EllrMatrix.from_crs(0, rp, col, val)
        E.spmv(y, x)
        S = pj.PjdsMatrix.from_crs(0, rp, col, val, symmetric=True)
        S.spmv(y, x)
        torch.cuda.synchronize()


def test_misuse_errors(pj):
    n, rp, col, val = inputs.config_crs("C1")
    A = pj.PjdsMatrix.from_crs(n, rp, col, val)
    x = tdev(inputs.vector(n))
    with pytest.raises(pj.PjdsError):
        A.spmv(x, x)  # aliasing
    with pytest.raises(ValueError):
        A.spmv(torch.empty(n, dtype=torch.float32, device="cuda"), x)


@pytest.mark.parametrize("variant", [(1, 8), (2, 4), (2, 8), (4, 2), (4, 4), (9, 8), (10, 4), (12, 2), (4, 18),
                                     (4, 34), (2, 36), (4, 36), (12, 34)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_kernel_variants_bitwise(pj, variant, dtype):
    """Every (rows per thread, unroll) variant gives the same per-row FMA chain (R+8: 64-bit offsets,
    U+16: software-pipelined, U+32: lane-interleaved rows, active where b_r % 32R == 0)."""
    L = pj.lib()
    try:
        assert L.pjds_set_kernel_variant(*variant) == 0
        for kind, n, br in (("random", 3001, 32), ("empty_rows", 999, 64), ("clustered", 4100, 128)):
            _, rp, col, val = inputs.small(kind, n, seed=5, dtype=dtype)
            x = inputs.vector(n, dtype)
            for sym in (False, True):
                A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, symmetric=sym)
                y = torch.full((n,), float("nan"), dtype=torch.float64 if dtype == np.float64 else torch.float32,
                               device="cuda")
                perm = A.export()["perm"]
                A.spmv(y, tdev(x[perm] if sym else x))
                yh = y.cpu().numpy()
                if sym:
                    yo = np.empty(n, dtype=yh.dtype)
                    yo[perm] = yh
                    yh = yo
                check_y(yh, n, rp, col, val, x)
            E = pj.EllrMatrix.from_crs(n, rp, col, val)  # the variant knob also picks ELLPACK-R's R
            y = torch.full((n,), float("nan"), dtype=torch.float64 if dtype == np.float64 else torch.float32,
                           device="cuda")
            E.spmv(y, tdev(x))
            check_y(y.cpu().numpy(), n, rp, col, val, x)
    finally:
        L.pjds_set_kernel_variant(0, 0)


@pytest.mark.parametrize("variant", [(18, 4), (18, 8), (20, 4), (20, 8), (24, 4)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_split_variant_bitwise(pj, variant, dtype):
    """Long-row split-j kernel (knob 16 + S threads per row): equal to the oracle's split-chain
    arithmetic (S interleaved FMA chains + pairwise tree) bit for bit, and within O2; both bases,
    ragged lengths, a row wider than the staged col_start, and the dist (y +=) store path."""
    L = pj.lib()
    S = variant[0] - 16
    try:
        assert L.pjds_set_kernel_variant(*variant) == 0
        for kind, n, br, kw in (("random", 3001, 32, dict(max=300)), ("empty_rows", 999, 64, {}),
                                ("clustered", 4100, 128, {}), ("adversarial", 3000, 32, {})):
            _, rp, col, val = inputs.small(kind, n, seed=7, dtype=dtype, **kw)
            x = inputs.vector(n, dtype)
            want = oracle.spmv_split_chain(n, rp, col, val, x, S)
            for sym in (False, True):
                A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, symmetric=sym)
                y = torch.full((n,), float("nan"), dtype=torch.float64 if dtype == np.float64 else torch.float32,
                               device="cuda")
                perm = A.export()["perm"]
                A.spmv(y, tdev(x[perm] if sym else x))
                yh = y.cpu().numpy()
                if sym:
                    yo = np.empty(n, dtype=yh.dtype)
                    yo[perm] = yh
                    yh = yo
                check_y(yh, n, rp, col, val, x, exact=False)
                assert np.array_equal(yh, want), (kind, sym)
        n = 3000
        _, rp, col, val = inputs.small("random", n, seed=9, max=200, dtype=dtype)
        x = inputs.vector(n, dtype)
        offs = np.array([0, 1000, 2000, 3000], np.int64)
        hs = pj.DistPjds.create_group(n, rp, col, val, offs)
        xs = [tdev(x[offs[r]:offs[r + 1]]) for r in range(3)]
        ys = [torch.empty(1000, dtype=xs[0].dtype, device="cuda") for _ in range(3)]
        pj.DistPjds.group_spmv(hs, ys, xs)
        torch.cuda.synchronize()
        check_y(np.concatenate([t.cpu().numpy() for t in ys]), n, rp, col, val, x, exact=False)
    finally:
        L.pjds_set_kernel_variant(0, 0)


def test_permute_and_symmetric_host_e2e(pj):
    """Basis change kernels and the e2e host path of the permuted-basis mode."""
    n, rp, col, val = inputs.config_crs("C1")
    x = inputs.vector(n)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
    perm = A.export()["perm"]
    xt = tdev(x)
    xp = torch.empty_like(xt)
    A.to_permuted(xp, xt)
    assert np.array_equal(xp.cpu().numpy(), x[perm])
    back = torch.empty_like(xt)
    A.from_permuted(back, xp)
    assert np.array_equal(back.cpu().numpy(), x)
    y = np.empty(n)
    A.spmv_host(y, x)
    check_y(y, n, rp, col, val, x)


@pytest.mark.parametrize("order", [0, 1, 2, 3])
def test_tile_order_bitwise(pj, order):
    """CTA (or, mode 3, warp-tile) execution order does not change any row's chain."""
    L = pj.lib()
    try:
        assert L.pjds_set_tile_order(order) == 0
        for name in ("C1", "C4"):
            n, rp, col, val = inputs.config_crs(name)
            x = inputs.vector(n)
            for sym in (False, True):
                A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=sym)
                y = np.empty(n)
                A.spmv_host(y, x)
                check_y(y, n, rp, col, val, x)
    finally:
        L.pjds_set_tile_order(2)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_warp_tile_order_variants_bitwise(pj, dtype):
    """Mode 3 (warp tiles by original row) with every rows-per-thread variant, b_r 32/128, ragged
    and empty-row inputs, both bases, the Lanczos-style fused dot kernel excluded (sigma = 0 only)."""
    L = pj.lib()
    try:
        assert L.pjds_set_tile_order(3) == 0
        cases = [("C3", None), ("random", 2500), ("empty_rows", 777), ("adversarial", 1100)]
        for name, m in cases:
            if m is None:
                n, rp, col, val = inputs.config_crs(name, dtype=dtype)
            else:
                n, rp, col, val = inputs.small(name, m, seed=m, dtype=dtype, **({"max": 70} if name == "random" else {}))
            x = inputs.vector(n, dtype)
            xt = tdev(x)
            for br in (32, 128):
                for sym in (False, True):
                    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, symmetric=sym)
                    xin = A.to_permuted(torch.empty_like(xt), xt) if sym else xt
                    # (4, 34) / (2, 36): lane-interleaved rows inside the warp tiles (b_r 128 only)
                    for variant in ((0, 0), (1, 8), (2, 4), (4, 2), (4, 4), (4, 34), (2, 36)):
                        assert L.pjds_set_kernel_variant(*variant) == 0
                        y = torch.full_like(xt, float("nan"))
                        A.spmv(y, xin)
                        yo = A.from_permuted(torch.empty_like(y), y) if sym else y
                        torch.cuda.synchronize()
                        check_y(yo.cpu().numpy(), n, rp, col, val, x)
                        if not sym:  # y += A x through the warp tiles as well
                            y0 = inputs.vector(n, dtype, seed=93)
                            ya = tdev(y0)
                            A.spmv_accum(ya, xin)
                            torch.cuda.synchronize()
                            want = (y0 + oracle.spmv_chain(n, rp, col, val, x)).astype(dtype)
                            assert np.array_equal(ya.cpu().numpy(), want), (name, br, variant)
                    del A
    finally:
        L.pjds_set_kernel_variant(0, 0)
        L.pjds_set_tile_order(2)


@pytest.mark.parametrize("y_kind", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("variant", [(0, 0), (4, 2), (2, 4), (1, 8)])
def test_y_store_bitwise(pj, y_kind, variant):
    """The permuted-basis y store (plain scalar stores, or one R-wide vector store with each L2
    policy; pjds_set_cache_policy bits 8-15) writes the same chains, ragged last thread included."""
    L = pj.lib()
    try:
        assert L.pjds_set_cache_policy(1 | (y_kind << 8), 2) == 0
        assert L.pjds_set_kernel_variant(*variant) == 0
        for dtype in (np.float64, np.float32):
            for n, rp, col, val in (inputs.config_crs("C1"), inputs.small("random", 1501, seed=7, dtype=dtype, max=40)):
                val = val.astype(dtype)
                x = inputs.vector(n, dtype)
                A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
                y = np.empty(n, dtype)
                A.spmv_host(y, x)
                check_y(y, n, rp, col, val, x)
                # the per-handle override (pjds_set_y_store) with every kind, on top of the global one
                for ys in (-1, 0, 1, 2, 3, 4):
                    assert L.pjds_set_y_store(A._h, ys) == 0
                    y = np.empty(n, dtype)
                    A.spmv_host(y, x)
                    check_y(y, n, rp, col, val, x)
    finally:
        L.pjds_set_cache_policy(1 | (2 << 8), 2)
        L.pjds_set_kernel_variant(0, 0)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_y_store_unaligned_output(pj, dtype):
    """A caller's y needs only element alignment: a tensor view one element into its storage takes
    the plain-store path instead of faulting on the R-wide vector store."""
    L = pj.lib()
    try:
        assert L.pjds_set_kernel_variant(4, 2) == 0
        n, rp, col, val = inputs.small("random", 1501, seed=8, dtype=dtype, max=40)
        x = inputs.vector(n, dtype)
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=True)
        tdt = torch.float64 if dtype == np.float64 else torch.float32
        for shift in (0, 1, 2, 3):
            buf = torch.full((n + 4,), float("nan"), dtype=tdt, device="cuda")
            y = buf[shift:shift + n]
            A.spmv(y, tdev(x[A.export()["perm"]]))
            torch.cuda.synchronize()
            yo = np.empty(n, dtype)
            yo[A.export()["perm"]] = y.cpu().numpy()
            check_y(yo, n, rp, col, val, x)
    finally:
        L.pjds_set_kernel_variant(0, 0)


def test_tile_keys_bitwise(pj):
    """pjds_set_tile_keys (user execution order: a random key, the HMEp 2-D window key, and back to
    the default) never changes a row's chain; a wrong-length key is rejected."""
    L = pj.lib()
    n, rp, col, val = inputs.config_crs("C1")
    x = inputs.vector(n)
    rng = np.random.default_rng(3)
    r = np.arange(n, dtype=np.int64)
    try:
        assert L.pjds_set_tile_order(1) == 0
        for sym in (False, True):
            A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=sym)
            for keys in (rng.permutation(n).astype(np.int64), ((r % 1024) // 256) * n + r, None):
                A.set_tile_keys(keys)
                y = np.empty(n)
                A.spmv_host(y, x)
                check_y(y, n, rp, col, val, x)
            with pytest.raises(pj.PjdsError):
                A.set_tile_keys(np.zeros(n - 1, np.int64))
    finally:
        L.pjds_set_tile_order(2)


@pytest.mark.parametrize("symmetric", [False, True])
def test_spmv_host_batch_pipelined(pj, symmetric):
    """Pipelined host-buffer products (double-buffered staging, copy streams) equal the oracle."""
    n, rp, col, val = inputs.config_crs("C1")
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=symmetric)
    xs = [torch.from_numpy(inputs.vector(n, seed=100 + i)).pin_memory().numpy() for i in range(5)]
    ys = [torch.full((n,), float("nan"), dtype=torch.float64).pin_memory().numpy() for _ in range(5)]
    A.spmv_host_batch(ys, xs)
    for x, y in zip(xs, ys):
        check_y(y, n, rp, col, val, x)


@pytest.mark.parametrize("sched", [0, 1])
def test_schedule_bitwise(pj, sched):
    """pjds_set_schedule: the dynamic warp-tile kernel runs the same row chains as the static grid
    (bitwise = the FMA chain), for every rows-per-thread variant, the pipelined variant, both
    bases, both tile orders, ragged warp tiles, and repeated launches (its counter resets itself)."""
    L = pj.lib()
    try:
        assert L.pjds_set_schedule(sched) == 0
        cases = [("C4", None), ("C1", None), ("random", 1500), ("adversarial", 1000), ("empty_rows", 513)]
        for name, m in cases:
            for dtype in (np.float64, np.float32):
                if m is None:
                    n, rp, col, val = inputs.config_crs(name, dtype=dtype)
                else:
                    n, rp, col, val = inputs.small(name, m, seed=m, dtype=dtype, **({"max": 90} if name == "random" else {}))
                x = inputs.vector(n, dtype)
                xt = tdev(x)
                for sym in (False, True):
                    A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=sym)
                    xin = A.to_permuted(torch.empty_like(xt), xt) if sym else xt
                    for variant in ((0, 0), (1, 8), (2, 4), (4, 2), (2, 20)):
                        assert L.pjds_set_kernel_variant(*variant) == 0
                        for order in (0, 1):
                            assert L.pjds_set_tile_order(order) == 0
                            y = torch.full_like(xt, float("nan"))
                            for _ in range(3):
                                A.spmv(y, xin)
                            yo = A.from_permuted(torch.empty_like(y), y) if sym else y
                            torch.cuda.synchronize()
                            check_y(yo.cpu().numpy(), n, rp, col, val, x)
                            if not sym:  # y += A x: one rounding add onto the previous y
                                y0 = inputs.vector(n, dtype, seed=91)
                                ya = tdev(y0)
                                A.spmv_accum(ya, xin)
                                torch.cuda.synchronize()
                                want = (y0 + oracle.spmv_chain(n, rp, col, val, x)).astype(dtype)
                                assert np.array_equal(ya.cpu().numpy(), want), (name, variant, order)
                    del A
    finally:
        L.pjds_set_schedule(0)
        L.pjds_set_kernel_variant(0, 0)
        L.pjds_set_tile_order(2)


@pytest.mark.parametrize("overlap", [(1, 0), (1, 4), (1, 64), (2, 2), (3, 0)])
def test_launch_overlap_dependent_chain(pj, overlap):
    """pjds_set_launch_overlap: a product launched as a programmatic dependent of the previous one
    starts in its tail but reads x and writes y only after griddepcontrol.wait, so a chain of
    dependent products x_{k+1} = A x_k over two ping-pong buffers (product k+1 overwrites the x that
    product k reads: RAW and WAR on every step) gives, bitwise, the oracle's chain of FMA chains --
    for the pJDS kernel (row-only and permuted basis, tile orders 0/1/3, every rows-per-thread
    variant, widths past the 1024 staged col_start entries), y += A x, and ELLPACK-R."""
    L = pj.lib()
    try:
        assert L.pjds_set_launch_overlap(*overlap) == 0
        cases = [("C1", None), ("C4", None), ("random", 1500), ("adversarial", 3000), ("empty_rows", 513)]
        for name, m in cases:
            for dtype in (np.float64, np.float32):
                if m is None:
                    n, rp, col, val = inputs.config_crs(name, dtype=dtype)
                else:
                    n, rp, col, val = inputs.small(name, m, seed=m, dtype=dtype, **({"max": 90} if name == "random" else {}))
                # scale the values so that 6 products stay O(1) (exact: a power of two)
                val = (val * dtype(2.0 ** -4)).astype(dtype)
                x0 = inputs.vector(n, dtype)
                want = [x0]
                for _ in range(6):
                    want.append(oracle.spmv_chain(n, rp, col, val, want[-1]))
                for sym in (False, True):
                    A = pj.PjdsMatrix.from_crs(n, rp, col, val, symmetric=sym, block_rows=128 if n > 2000 else 32)
                    for variant in ((0, 0), (1, 8), (2, 4), (4, 2)):
                        assert L.pjds_set_kernel_variant(*variant) == 0
                        for order in (0, 1, 3):
                            assert L.pjds_set_tile_order(order) == 0
                            b = [tdev(x0), torch.full_like(tdev(x0), float("nan"))]
                            if sym:
                                b[0] = A.to_permuted(torch.empty_like(b[0]), b[0])
                            for k in range(6):
                                A.spmv(b[(k + 1) % 2], b[k % 2])
                            out = b[0]
                            if sym:
                                out = A.from_permuted(torch.empty_like(out), out)
                            torch.cuda.synchronize()
                            assert np.array_equal(out.cpu().numpy(), want[6]), (name, dtype, sym, variant, order)
                    if not sym:  # y += A x, three times onto the same y (each depends on the previous)
                        assert L.pjds_set_kernel_variant(0, 0) == 0
                        ya = tdev(x0)
                        xt = tdev(want[1])
                        acc = x0.copy()
                        for _ in range(3):
                            A.spmv_accum(ya, xt)
                            acc = (acc + want[2]).astype(dtype)
                        torch.cuda.synchronize()
                        assert np.array_equal(ya.cpu().numpy(), acc), (name, dtype, "accum")
                    del A
                E = pj.EllrMatrix.from_crs(n, rp, col, val)
                b = [tdev(x0), torch.full_like(tdev(x0), float("nan"))]
                for k in range(6):
                    E.spmv(b[(k + 1) % 2], b[k % 2])
                torch.cuda.synchronize()
                assert np.array_equal(b[0].cpu().numpy(), want[6]), (name, dtype, "ellr")
    finally:
        L.pjds_set_launch_overlap(2, 2)
        L.pjds_set_kernel_variant(0, 0)
        L.pjds_set_tile_order(2)


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_compressible_col_bitwise(pj, name):
    """pjds_set_compression: the column indices in generic compressible memory are the same array
    (device export == the oracle converter's), the product is bitwise the same as with plain memory
    and the FMA chain, for pJDS (both bases) and ELLPACK-R; info reports where col lives."""
    L = pj.lib()
    granted = 1
    try:  # a device without generic compression falls back to plain memory (col_compressible 0)
        from cuda.bindings import driver as cu
        cu.cuInit(0)
        err, dev = cu.cuDeviceGet(torch.cuda.current_device())
        err2, sup = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, dev)
        if err == cu.CUresult.CUDA_SUCCESS and err2 == cu.CUresult.CUDA_SUCCESS:
            granted = int(sup != 0)
    except ImportError:
        pass
    try:
        for dtype in (np.float64, np.float32):
            n, rp, col, val = inputs.config_crs(name, dtype=dtype)
            x = inputs.vector(n, dtype)
            xt = tdev(x)
            chain = oracle.spmv_chain(n, rp, col, val, x)
            ref = convert.pjds_reference(n, rp, col, val, 128, symmetric=True)
            for mode in (0, 1):
                assert L.pjds_set_compression(mode) == 0
                for sym in (False, True):
                    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=128, symmetric=sym)
                    assert A.info["col_compressible"] == mode * granted, (name, mode, A.info["col_compressible"])
                    if sym:
                        assert np.array_equal(A.export()["col"], np.asarray(ref["col"], np.int32))
                    xin = A.to_permuted(torch.empty_like(xt), xt) if sym else xt
                    y = torch.full_like(xt, float("nan"))
                    A.spmv(y, xin)
                    yo = A.from_permuted(torch.empty_like(y), y) if sym else y
                    torch.cuda.synchronize()
                    assert np.array_equal(yo.cpu().numpy(), chain), (name, dtype, mode, sym)
                    del A
                E = pj.EllrMatrix.from_crs(n, rp, col, val)
                assert E.info["col_compressible"] == mode * granted
                y = torch.full_like(xt, float("nan"))
                E.spmv(y, xt)
                torch.cuda.synchronize()
                assert np.array_equal(y.cpu().numpy(), chain), (name, dtype, mode, "ellr")
                del E
    finally:
        L.pjds_set_compression(1)
