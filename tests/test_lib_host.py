"""CPU-side tests of libpjds (no GPU needed): the library loads and exports every symbol the
header declares; host conversion (PJDS_HOST_ONLY) is bit-exact against the independent oracle
converters; input validation returns the documented status codes; info/histogram agree with the
oracle's accounting; the dist plan (split + halo schedule) equals the oracle's emulator."""
import ctypes
import os
import re

import numpy as np
import pytest

import inputs
from oracle import convert, dist as odist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pj():
    import build_native
    build_native.build_pjds()
    import paper_1112_5588_b200 as pj
    return pj


def test_exports_every_header_symbol(pj):
    hdr = open(os.path.join(ROOT, "include", "pjds.h")).read()
    names = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+((?:pjds|ellr)_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 25
    L = pj.lib()
    for nm in sorted(names):
        assert hasattr(L, nm), nm
    assert names == set(pj._lib.EXPORTED)
    assert b"sm_100a" in L.pjds_version()


CASES = [("uniform", 300, {}), ("clustered", 257, {}), ("empty_rows", 190, {}), ("duplicates", 100, {}),
         ("random", 333, dict(max=70)), ("adversarial", 130, {}), ("constant", 64, dict(k=5)), ("zero", 40, {}),
         ("identity", 33, {})]


def assert_pjds_equal(got, P):
    assert np.array_equal(got["perm"], P["perm"])
    assert np.array_equal(got["block_len"], P["block_len"])
    assert np.array_equal(got["col_start"], P["col_start"])
    assert np.array_equal(got["col"], P["col"])
    assert got["val"].dtype == P["val"].dtype
    assert got["val"].tobytes() == P["val"].tobytes()  # bit-exact, +0.0 padding included


@pytest.mark.parametrize("kind,n,kw", CASES)
@pytest.mark.parametrize("br", [32, 64, 96, 128, 160])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pjds_conversion_bit_exact(pj, kind, n, kw, br, dtype):
    _, rp, col, val = inputs.small(kind, n, seed=br, dtype=dtype, **kw)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br, host_only=True)
    P = convert.pjds_reference(n, rp, col, val, b_r=br)
    assert_pjds_equal(A.export(), P)
    i = A.info
    assert (i["n"], i["nnz"], i["n_pad"], i["n_blocks"], i["stored"], i["width"]) == \
        (n, len(col), P["n_pad"], P["n_blocks"], P["stored"], P["width"])
    fp = convert.footprint(P, value_bytes=np.dtype(dtype).itemsize)["pjds"]
    for k in ("bytes_values", "bytes_indices", "bytes_aux", "bytes_total"):
        assert i[k] == fp[k], k
    assert i["data_reduction_vs_ellpack"] == pytest.approx(fp["data_reduction_vs_ellpack"], abs=1e-15)
    u = convert.utilisation(P, nnz=len(col))["pjds"]
    assert (i["useful_fma"], i["padded_fma"], i["idle_lane_slots"]) == (u["useful"], u["padded"], u["idle"])
    lens = np.diff(rp)
    assert np.array_equal(A.histogram(), np.bincount(lens, minlength=i["len_max"] + 1))


def test_pjds_symmetric_conversion(pj):
    n = 200
    _, rp, col, val = inputs.small("uniform", n, seed=3)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=32, symmetric=True, host_only=True)
    assert_pjds_equal(A.export(), convert.pjds_reference(n, rp, col, val, b_r=32, symmetric=True))


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_pjds_conversion_configs(pj, name):
    n, rp, col, val = inputs.config_crs(name)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, host_only=True)
    assert_pjds_equal(A.export(), convert.pjds_reference(n, rp, col, val, b_r=32))
    E = pj.EllrMatrix.from_crs(n, rp, col, val, host_only=True)
    R = convert.ellr_reference(n, rp, col, val)
    got = E.export()
    assert np.array_equal(got["rowmax"], R["rowmax"]) and np.array_equal(got["col"], R["col"])
    assert got["val"].tobytes() == R["val"].tobytes()


@pytest.mark.parametrize("kind,n,kw", CASES)
def test_ellr_conversion_bit_exact(pj, kind, n, kw):
    _, rp, col, val = inputs.small(kind, n, seed=1, **kw)
    E = pj.EllrMatrix.from_crs(n, rp, col, val, host_only=True)
    R = convert.ellr_reference(n, rp, col, val)
    got = E.export()
    assert np.array_equal(got["rowmax"], R["rowmax"])
    assert np.array_equal(got["col"], R["col"])
    assert got["val"].tobytes() == R["val"].tobytes()
    i = E.info
    assert (i["n_pad"], i["width"], i["stored"]) == (R["n_pad"], R["width"], R["stored"])
    assert i["idle_lane_slots"] == convert.utilisation(E=R, nnz=len(col))["ellr"]["idle"]
    fp = convert.footprint(E=R)["ellr"]
    assert i["bytes_total"] == fp["bytes_total"]


@pytest.mark.parametrize("kind,n,kw", CASES[:5])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_footprint_and_stats_entry_points(pj, kind, n, kw, dtype):
    """pjds_footprint / pjds_stats / ellr_footprint (SURVEY §8(b) names) against the oracle's
    accounting (oracle/convert.py footprint + utilisation)."""
    _, rp, col, val = inputs.small(kind, n, seed=5, dtype=dtype, **kw)
    sv = np.dtype(dtype).itemsize
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=64, host_only=True)
    P = convert.pjds_reference(n, rp, col, val, b_r=64)
    ref = convert.footprint(P, value_bytes=sv)["pjds"]
    f = A.footprint()
    assert (f["bytes_values"], f["bytes_indices"], f["bytes_total"]) == \
        (ref["bytes_values"], ref["bytes_indices"], ref["bytes_total"])
    assert (f["bytes_col_start"], f["bytes_block_len"], f["bytes_perm"], f["bytes_rowmax"]) == \
        ((P["width"] + 1) * 8, P["n_blocks"] * 4, n * 4, 0)
    assert (f["stored"], f["nnz"], f["n_pad"]) == (P["stored"], len(col), P["n_pad"])
    st = A.stats()
    lens = np.diff(rp)
    u = convert.utilisation(P, nnz=len(col))["pjds"]
    assert (st["n"], st["nnz"], st["n_pad"], st["n_blocks"], st["padding"], st["width"], st["block_rows"]) == \
        (n, len(col), P["n_pad"], P["n_blocks"], P["stored"] - len(col), P["width"], 64)
    assert (st["len_min"], st["len_max"]) == (int(lens.min()), int(lens.max()))
    assert st["len_mean"] == pytest.approx(lens.mean(), rel=1e-15)
    assert st["reduction_vs_ellpack"] == pytest.approx(ref["data_reduction_vs_ellpack"], abs=1e-15)
    assert (st["useful_fma"], st["padded_fma"], st["idle_lane_slots"]) == (u["useful"], u["padded"], u["idle"])
    E = pj.EllrMatrix.from_crs(n, rp, col, val, host_only=True)
    R = convert.ellr_reference(n, rp, col, val)
    fe = E.footprint()
    refe = convert.footprint(E=R, value_bytes=sv)["ellr"]
    assert (fe["bytes_values"], fe["bytes_indices"], fe["bytes_rowmax"], fe["bytes_total"]) == \
        (refe["bytes_values"], refe["bytes_indices"], refe["bytes_aux"], refe["bytes_total"])
    assert (fe["bytes_col_start"], fe["bytes_block_len"], fe["bytes_perm"]) == (0, 0, 0)


def test_adversarial_closed_form_in_library(pj):
    n = 1024
    _, rp, col, val = inputs.small("adversarial", n, seed=2)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, host_only=True)
    E = pj.EllrMatrix.from_crs(n, rp, col, val, host_only=True)
    assert A.info["stored"] == 33760 and E.info["stored"] == 1024 * 1024


def test_error_codes(pj):
    from paper_1112_5588_b200 import PjdsError
    n = 4
    rp = np.array([0, 1, 2, 3, 4], np.int64)
    col = np.array([0, 1, 2, 3], np.int32)
    val = np.ones(4)
    with pytest.raises(PjdsError) as e:
        pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=48, host_only=True)
    assert e.value.status == -1
    with pytest.raises(PjdsError) as e:
        pj.PjdsMatrix.from_crs(n, np.array([1, 1, 2, 3, 4]), col, val, host_only=True)
    assert e.value.status == -2
    with pytest.raises(PjdsError) as e:
        pj.PjdsMatrix.from_crs(n, np.array([0, 2, 1, 3, 4]), col, val, host_only=True)
    assert e.value.status == -2 and "decreasing" in str(e.value)
    with pytest.raises(PjdsError) as e:
        pj.PjdsMatrix.from_crs(n, rp, np.array([0, 1, 2, 4], np.int32), val, host_only=True)
    assert e.value.status == -2
    with pytest.raises(PjdsError) as e:
        pj.EllrMatrix.from_crs(n, rp, np.array([0, -1, 2, 3], np.int32), val, host_only=True)
    assert e.value.status == -2
    L = pj.lib()
    h = ctypes.c_void_p()
    assert L.pjds_create_from_crs(ctypes.byref(h), 4, rp.ctypes.data, col.ctypes.data, val.ctypes.data, 7, 32, 2) == -1
    assert L.pjds_create_from_crs(None, 4, rp.ctypes.data, col.ctypes.data, val.ctypes.data, 1, 32, 2) == -1
    # host-only handles refuse spmv
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, host_only=True)
    assert L.pjds_spmv(A._h, ctypes.c_void_p(16), ctypes.c_void_p(32), None) == -1
    # empty matrix converts
    A0 = pj.PjdsMatrix.from_crs(0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0), host_only=True)
    assert A0.info["stored"] == 0 and A0.info["n_blocks"] == 0


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
def test_dist_plan_matches_oracle(pj, R):
    n = 400
    _, rp, col, val = inputs.small("random", n, seed=10 + R, max=30)
    offs = np.array([n * r // R for r in range(R + 1)], np.int64)
    _check_plan(pj, n, rp, col, val, offs)


def test_dist_plan_empty_ranks(pj):
    """Ranks that own no rows (offsets repeat) plan an empty local part and receive nothing."""
    n = 300
    _, rp, col, val = inputs.small("random", n, seed=4, max=40)
    _check_plan(pj, n, rp, col, val, np.array([0, 0, 120, 120, 300, 300], np.int64))


def _check_plan(pj, n, rp, col, val, offs):
    R = len(offs) - 1
    ref = odist.split(n, rp, col, val, offs)
    for r in range(R):
        lo, hi = offs[r], offs[r + 1]
        plan = pj.DistPlan(R, r, n, offs, rp[lo:hi + 1] - rp[lo], col[rp[lo]:rp[hi]])
        counts, cols = plan.recv()
        assert counts.tolist() == [len(a) for a in ref[r]["recv"]]
        assert cols.tolist() == ref[r]["halo_cols"].tolist()
        inf = plan.info
        assert inf["rows_nonlocal"] == len(ref[r]["rows_nl"])
        assert inf["nnz_nonlocal_part"] == len(ref[r]["nl"][2])
        assert inf["nnz_local_part"] == len(ref[r]["loc"][2])
        assert inf["halo"] == len(ref[r]["halo_cols"])


def test_dist_plan_hmep_segments(pj):
    """C1 split over 4 ranks: every halo is a set of whole 1024-long segments."""
    g = inputs.Generator.from_config("C1")
    rp, col, val = g.crs()
    n = g.n
    offs = np.array([0, 4096, 8192, 12288, 16384], np.int64)
    for r in range(4):
        lo, hi = offs[r], offs[r + 1]
        plan = pj.DistPlan(4, r, n, offs, rp[lo:hi + 1] - rp[lo], col[rp[lo]:rp[hi]])
        counts, cols = plan.recv()
        assert all(c % 1024 == 0 for c in counts)
        runs = 1 + int(np.count_nonzero(np.diff(cols) != 1)) if len(cols) else 0
        assert runs == len(cols) // 1024 or runs < len(cols) // 1024  # adjacent segments merge


def test_round2_knobs_and_collective_create_validation(pj):
    """Argument checks of the round-2 entry points that need no GPU: the A_nl sort scope, the
    per-handle y store, pjds_spmv_accum on host-only / symmetric handles, and the one-call
    collective create's validation before any NCCL call (NULL id with nranks > 1, bad offsets)."""
    L = pj.lib()
    assert L.pjds_set_dist_nl_sigma(1000) == -1 and L.pjds_set_dist_nl_sigma(-1024) == -1
    assert L.pjds_set_dist_nl_sigma(0) == 0 and L.pjds_set_dist_nl_sigma(2048) == 0
    assert L.pjds_set_dist_nl_sigma(1024) == 0  # back to the default
    assert L.pjds_set_schedule(2) == -1 and L.pjds_set_schedule(0) == 0
    assert L.pjds_set_tile_order(4) == -1 and L.pjds_set_tile_order(2) == 0
    assert L.pjds_set_launch_overlap(4, 0) == -1 and L.pjds_set_launch_overlap(-1, 0) == -1
    assert L.pjds_set_launch_overlap(1, 65) == -1 and L.pjds_set_launch_overlap(1, -1) == -1
    assert L.pjds_set_launch_overlap(1, 4) == 0 and L.pjds_set_launch_overlap(2, 2) == 0
    assert L.pjds_set_compression(2) == -1 and L.pjds_set_compression(-1) == -1
    assert L.pjds_set_compression(0) == 0 and L.pjds_set_compression(1) == 0
    n = 64
    _, rp, col, val = inputs.small("random", n, seed=2, max=9)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, host_only=True)
    assert L.pjds_set_y_store(A._h, 5) == -1 and L.pjds_set_y_store(A._h, -2) == -1
    assert L.pjds_set_y_store(A._h, 3) == 0 and L.pjds_set_y_store(A._h, -1) == 0
    assert L.pjds_set_y_store(None, 0) == -1
    assert L.pjds_spmv_accum(A._h, ctypes.c_void_p(16), ctypes.c_void_p(32), None) == -1  # host-only
    S = pj.PjdsMatrix.from_crs(n, rp, col, val, host_only=True, symmetric=True)
    assert S.symmetric and not A.symmetric
    h = ctypes.c_void_p()
    offs = np.array([0, 32, 64], np.int64)
    lo_rp = rp[:33] - rp[0]
    # nranks > 1 needs the NCCL unique id
    st = L.pjds_dist_create_crs(ctypes.byref(h), None, 2, 0, n, offs.ctypes.data, lo_rp.ctypes.data,
                                col.ctypes.data, val.ctypes.data, 1, 32, 0)
    assert st == -1 and not h.value
    # offsets that do not span [0, n]
    bad = np.array([0, 32, 60], np.int64)
    uid = (ctypes.c_char * 128)()
    st = L.pjds_dist_create_crs(ctypes.byref(h), uid, 2, 0, n, bad.ctypes.data, lo_rp.ctypes.data,
                                col.ctypes.data, val.ctypes.data, 1, 32, 0)
    assert st == -1 and not h.value
    assert L.pjds_dist_create_crs(None, uid, 1, 0, n, offs.ctypes.data, rp.ctypes.data, col.ctypes.data,
                                  val.ctypes.data, 1, 32, 0) == -1
