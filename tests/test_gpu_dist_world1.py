"""DistPjds through the NCCL-transport entry points in a one-rank torch.distributed group (the only
size one GPU allows): plan -> list exchange -> pjds_dist_create -> pjds_dist_spmv (both bases, both
modes) -> pjds_dist_trace, checked against the oracle."""
import os

import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29613")
        dist.init_process_group("gloo", rank=0, world_size=1)
    yield dist


@pytest.mark.parametrize("permuted", [False, True])
def test_dist_world1(pg, permuted):
    import paper_1112_5588_b200 as pj
    n, rp, col, val = inputs.config_crs("C1")
    x = inputs.vector(n)
    D = pj.DistPjds.create(n, np.array([0, n]), rp, col, val, permuted=permuted)
    assert D.info["halo"] == 0 and D.info["permuted"] == int(permuted)
    xt = torch.from_numpy(x).cuda()
    if permuted:
        xt = D.to_permuted(torch.empty_like(xt), xt)
    y_ref, bound = oracle.spmv_ld(n, rp, col, val, x)
    for no_overlap in (False, True):
        y = torch.full_like(xt, float("nan"))
        D.spmv(y, xt, no_overlap=no_overlap, trace=True)
        if permuted:
            y = D.from_permuted(torch.empty_like(y), y)
        torch.cuda.synchronize()
        yh = y.cpu().numpy()
        assert oracle.acceptance(yh, y_ref, bound, np.diff(rp), np.float64).all()
        assert np.array_equal(yh, oracle.spmv_chain(n, rp, col, val, x))
        ph = D.trace()
        # one rank: no exchange (back-to-back events only), the local part is the whole product
        assert ph["total"] > 0 and ph["exchange"] < 0.05 and ph["local"] <= ph["total"] + 1e-6
    D.close()


@pytest.mark.parametrize("permuted", [False, True])
def test_direct_world1_and_error_contract(pg, permuted):
    """PJDS_TRANSPORT_DIRECT on one rank (window = the local x; the kernel decodes every column
    through the window table), plus the error contract include/pjds.h states for its entry points."""
    import ctypes
    import paper_1112_5588_b200 as pj
    n, rp, col, val = inputs.config_crs("C1")
    x = inputs.vector(n)
    D = pj.DistPjds.create(n, np.array([0, n]), rp, col, val, permuted=permuted, transport="direct")
    xt = torch.from_numpy(x).cuda()
    if permuted:
        xt = D.to_permuted(torch.empty_like(xt), xt)
    chain = oracle.spmv_chain(n, rp, col, val, x)
    w = D.x_window()
    assert w.numel() == n and w.dtype == torch.float64
    for xin in (xt, w):  # x copied into the window, and x computed in the window
        if xin is w:
            w.copy_(xt)
        y = torch.full_like(xt, float("nan"))
        for _ in range(3):
            D.spmv(y, xin, trace=True)
        if permuted:
            y = D.from_permuted(torch.empty_like(y), y)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), chain)
    assert not D.p2p_timed_out()
    L = pj.lib()
    # y aliasing the window, second connect, window of a non-DIRECT handle: INVALID_ARG
    with pytest.raises(pj.PjdsError):
        D.spmv(w, xt)
    blob = (ctypes.c_char * 4096)()
    INVALID = -1  # PJDS_ERR_INVALID_ARG
    assert L.pjds_dist_direct_connect(D._h, None, blob, 1) == INVALID  # already connected
    D2 = pj.DistPjds.create(n, np.array([0, n]), rp, col, val, permuted=permuted)
    p = ctypes.c_void_p()
    assert L.pjds_dist_x_window(D2._h, ctypes.byref(p)) == INVALID
    assert L.pjds_dist_direct_positions(D2._h, None) == INVALID
    D2.close()
    D.close()
