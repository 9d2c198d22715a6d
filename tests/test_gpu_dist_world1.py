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
