"""bench.py host logic (no GPU): the same-run parity check (SURVEY §8(d) step 6, O2 vs the
long-double oracle + bitwise O3), the row sampling, the rank -> rank-0 gather of sampled rows
(gloo, world size 2), and the multi-GPU launch contract (--gpus N re-launches under torchrun, fails
loudly without N GPUs unless --oversubscribe, and refuses a world size that differs from --gpus)."""
import os
import socket
import subprocess
import sys

import numpy as np
import torch.multiprocessing as mp

import bench
import inputs
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref(g, chunks, x):
    return bench.oracle_rows(g, chunks, x, np.float64)


def test_parity_o2_accepts_and_rejects():
    g = inputs.Generator.from_config("C1")
    n = g.n
    rp, col, val = g.crs()
    x = inputs.vector(n)
    chunks = bench.sample_chunks(n, 10, 300, seed=3)
    rows = bench.chunk_rows(chunks)
    ref = _ref(g, chunks, x)
    y_chain = oracle.spmv_chain(n, rp, col, val, x)  # the default kernels' arithmetic
    ok = bench.parity_o2(y_chain[rows], ref, np.float64, chain_expected=True)
    assert ok["within_bound"] and ok["bitwise_o3_chain"] and ok["rows_checked"] == len(rows)
    y_crs = oracle.spmv_crs(n, rp, col, val, x)  # a differently rounded correct product
    res = bench.parity_o2(y_crs[rows], ref, np.float64, chain_expected=False)
    assert res["within_bound"]
    bad = y_chain.copy()
    r = int(rows[3])
    k = int(rp[r])
    bad[r] -= 2 * val[k] * x[col[k]]  # one term with the wrong sign
    res = bench.parity_o2(bad[rows], ref, np.float64, chain_expected=True)
    assert not res["within_bound"] and res["rows_outside"] == 1 and not res["bitwise_o3_chain"]
    nan = y_chain.copy()
    nan[int(rows[5])] = np.nan
    assert not bench.parity_o2(nan[rows], ref, np.float64, chain_expected=True)["within_bound"]


def test_sample_chunks_cover_boundaries_and_are_disjoint():
    n = 100_000
    ch = bench.sample_chunks(n, 50, 1000, seed=1, boundaries=[25_000, 50_000, 75_000])
    assert ch[0][0] == 0 and ch[-1][1] == n
    for (s0, e0), (s1, e1) in zip(ch, ch[1:]):
        assert s0 < e0 < s1 < e1  # sorted, disjoint, not touching (merged otherwise)
    for b in (25_000, 50_000, 75_000):
        assert any(s < b < e for s, e in ch)
    rows = bench.chunk_rows(ch)
    assert np.all(np.diff(rows) > 0) and rows[0] == 0 and rows[-1] == n - 1
    tiny = bench.sample_chunks(5, 3, 1000)
    assert tiny == [(0, 5)]


def test_check_world_and_launch_command():
    a = bench.parse(["--gpus", "2"])
    assert bench.check_world(a, {"WORLD_SIZE": "2"}, 8) is None
    assert "WORLD_SIZE=4" in bench.check_world(a, {"WORLD_SIZE": "4"}, 8)
    assert "needs 2 visible GPUs" in bench.check_world(a, {"WORLD_SIZE": "2"}, 1)
    a2 = bench.parse(["--gpus", "2", "--oversubscribe"])
    assert bench.check_world(a2, {"WORLD_SIZE": "2"}, 1) is None
    assert bench.check_world(bench.parse([]), {}, 1) is None  # plain N=1
    assert "needs 1 visible GPUs" in bench.check_world(bench.parse([]), {}, 0)  # no CPU fallback
    cmd = bench.launch_command(["--gpus", "4", "--steps", "3"], 4, 29999)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and "--master-port=29999" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")


def test_gpus_without_gpus_fails_loudly():
    """`python bench.py --gpus 2` on a box with fewer GPUs exits non-zero with a message instead of
    silently measuring one GPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 2 and "needs 2 visible GPUs" in p.stderr, (p.returncode, p.stderr[-500:])
    assert p.stdout.strip() == ""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench as b
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        n = 1000
        offs = [0, 430, n]
        lo, hi = offs[rank], offs[rank + 1]
        rows = b.chunk_rows(b.sample_chunks(n, 6, 40, seed=5, boundaries=[430]))
        y_loc = np.arange(lo, hi, dtype=np.float64) * 0.5  # y_i = i / 2 on the owning rank
        out = b.gather_rows(dist, rank, rows, y_loc, lo, hi)
        if rank == 0:
            q.put(bool(np.array_equal(out, rows * 0.5)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(repr(e))


def test_gather_rows_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = q.get(timeout=120)
    for p in ps:
        p.join(60)
    assert res is True, res
