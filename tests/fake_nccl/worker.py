"""Worker for tests/test_gpu_fake_nccl.py: one rank of the NCCL-transport dist path (all ranks on
cuda:0; PJDS_NCCL_LIB selects the one-GPU NCCL stand-in).  Prints one JSON line per rank."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, ROOT)
import torch, torch.distributed as dist
import inputs, oracle, paper_1112_5588_b200 as pj
from oracle import dist as odist
rank = int(os.environ["RANK"]); R = int(os.environ["WORLD_SIZE"])


def emit(obj):
    """One JSON line in a single write(2): the ranks share the parent's stdout pipe, and print()
    may split a line into several writes that interleave with another rank's."""
    os.write(1, (json.dumps(obj) + "\n").encode())


torch.cuda.set_device(0)
dist.init_process_group("gloo")
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
transport = sys.argv[2] if len(sys.argv) > 2 else "nccl"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
npdt = np.float32 if (len(sys.argv) > 4 and sys.argv[4] == "f32") else np.float64
if name in ("rand", "rand_empty"):
    n, rp, col, val = inputs.small("random", 3000, seed=3, max=60, dtype=npdt)
else:
    n, rp, col, val = inputs.config_crs(name, dtype=npdt)
seg = {"C1": 1024, "C3": 15504, "rand": 1, "rand_empty": 1}[name]
nb = n // seg
offs = np.array([(nb * r // R) * seg for r in range(R + 1)], np.int64)
if name == "rand_empty":  # rank 1 owns no rows (it still takes part in every call)
    offs[1] = offs[2]
lo, hi = offs[rank], offs[rank + 1]
x = inputs.vector(n, npdt)
out = {}
# DIRECT: one kernel over the unsplit rows -> bitwise the plain FMA chain; others: the split rule
chain = oracle.spmv_chain(n, rp, col, val, x) if transport == "direct" else None
for permuted in (False, True):
    try:
        D = pj.DistPjds.create(n, offs, rp[lo:hi + 1] - rp[lo], col[rp[lo]:rp[hi]], val[rp[lo]:rp[hi]],
                               permuted=permuted, transport=transport)
    except Exception as e:
        emit({"rank": rank, "create_error": str(e)[:300]}); sys.exit(0)
    xt = torch.from_numpy(x[lo:hi].copy()).cuda()
    if permuted:
        xt = D.to_permuted(torch.empty_like(xt), xt)
    for no in (False, True):
        xin = xt
        if transport == "direct" and no:  # x computed in the exported window: no per-call copy
            xin = D.x_window()
            xin.copy_(xt)
        y = torch.full_like(xt, float("nan"))
        for _ in range(reps):  # several calls: exercises the double-buffered halo / flag sequence
            D.spmv(y, xin, no_overlap=no, trace=True)
        if permuted:
            y = D.from_permuted(torch.empty_like(y), y)
        torch.cuda.synchronize()
        ys = [None] * R
        dist.all_gather_object(ys, y.cpu().numpy())
        yall = np.concatenate(ys)
        ref = chain if chain is not None else (odist.spmv(odist.split(n, rp, col, val, offs), x) if name != "C3" else None)
        yl, b = oracle.spmv_ld(n, rp, col, val, x)
        ok = bool(oracle.acceptance(yall, yl, b, np.diff(rp), npdt).all())
        out[f"perm{int(permuted)}_noov{int(no)}"] = {"o2": ok, "bitwise_vs_split_oracle": bool(np.array_equal(yall, ref)) if ref is not None else None,
                                                     "trace": D.trace(), "halo": D.info["halo"], "messages": D.info["send_messages"],
                                                     "timed_out": D.p2p_timed_out()}
    D.close()
emit({"rank": rank, **out})
dist.destroy_process_group()
