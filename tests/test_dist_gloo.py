"""Multi-process (world_size 2 and 3, gloo, CPU) test of the distributed setup path: each rank
builds its plan with libpjds, the recv lists are exchanged with torch.distributed
(exchange_lists, the same code DistPjds.create uses), and the resulting send lists / halo schedule
must equal the oracle's split emulator (oracle/dist.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    import inputs
    import paper_1112_5588_b200 as pj
    from oracle import dist as odist
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        for kind, n in (("random", 300), ("C1", None)):
            if kind == "C1":
                n, rp, col, val = inputs.config_crs("C1")
            else:
                _, rp, col, val = inputs.small("random", n, seed=7, max=30)
            offs = np.array([n * r // world for r in range(world + 1)], np.int64)
            lo, hi = offs[rank], offs[rank + 1]
            plan = pj.DistPlan(world, rank, n, offs, rp[lo:hi + 1] - rp[lo], col[rp[lo]:rp[hi]])
            rc, rcols = plan.recv()
            sc, scols = pj.exchange_lists(rc, rcols)
            ref = odist.split(n, rp, col, val, offs)[rank]
            assert sc.tolist() == [len(s) for s in ref["send"]], (kind, sc)
            want = np.concatenate([s + lo for s in ref["send"]]) if len(ref["send"]) else np.zeros(0)
            assert scols.tolist() == want.astype(np.int64).tolist()
            assert rcols.tolist() == ref["halo_cols"].tolist()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_dist_setup_gloo(world):
    import build_native
    build_native.build_pjds()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert res[r] == "ok", res[r]
