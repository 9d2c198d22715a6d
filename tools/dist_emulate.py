"""Single-GPU emulation of the row-partitioned dist spMVM (dev tool; NOT a bench number).

Builds all R ranks' handles on one GPU (LOCAL transport), times each rank's local part, nonlocal
part and pack kernel in isolation with CUDA events, and combines them with the halo volume into
the task-mode model t_r = max(T_loc, T_pack + bytes/B_link) + T_nl, B_link = the
measured NVLink peer bandwidth (770 GB/s per direction, B200_PROFILING.md).  Prints JSON lines.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1112_5588_b200 as pj  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C5")
p.add_argument("--ranks", default="1,2,4,8")
p.add_argument("--dtype", default="f64")
p.add_argument("--modes", default="permuted,rows")
p.add_argument("--reps", type=int, default=20)
a = p.parse_args()
SEG = {"C1": 1024, "C3": 15504, "C5": 142506}[a.config]
npdt = np.float64 if a.dtype == "f64" else np.float32
sv = np.dtype(npdt).itemsize
n, rp, col, val = inputs.config_crs(a.config, dtype=npdt)
nnz = len(col)
B_LINK = 770e9
# HBM contention of the exchange: on every rank the halo traffic also crosses the rank's own HBM
# (gather reads of the send entries, incoming writes of the halo).  Emulated on one GPU by a device
# copy of max(send, recv) bytes on a high-priority side stream while A_loc runs (same bytes read and
# written as the P2P transport's gather+put; it runs faster than NVLink, so it contends harder but
# for less time -- same total bytes).  t_model_contended = max(T_loc | copy, T_pack + bytes/B_link) + T_nl.
S_HI = torch.cuda.Stream(priority=-1)


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


t1 = {}
# the single-GPU bench kernel (pjds_spmv on the whole matrix, same basis) as T_1 as well
t_single = None
if "permuted" in a.modes.split(","):
    A1 = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=32, symmetric=True)
    x1 = torch.zeros(n, dtype=torch.float64 if sv == 8 else torch.float32, device="cuda")
    y1 = torch.zeros_like(x1)
    t_single = timeit(lambda: A1.spmv(y1, x1), a.reps)
    del A1, x1, y1
    torch.cuda.empty_cache()
for mode in a.modes.split(","):
    for R in map(int, a.ranks.split(",")):
        nb = n // SEG
        offs = np.array([(nb * r // R) * SEG for r in range(R + 1)], np.int64)
        offs[-1] = n
        hs = pj.DistPjds.create_group(n, rp, col, val, offs, permuted=(mode == "permuted"))
        ranks = []
        for r, h in enumerate(hs):
            nl = int(offs[r + 1] - offs[r])
            A_loc, A_nl = h.parts()
            x = torch.zeros(max(nl, h.info["halo"], 1), dtype=torch.float64 if sv == 8 else torch.float32, device="cuda")
            y = torch.zeros(max(nl, 1), dtype=x.dtype, device="cuda")
            tl = timeit(lambda: A_loc.spmv(y, x), a.reps)
            tn = timeit(lambda: A_nl.spmv(y, x), a.reps) if A_nl is not None else 0.0
            send = h.info["send_total"] * sv
            recv = h.info["halo"] * sv
            cbytes = max(send, recv)
            src = torch.zeros(max(cbytes // 8, 1), dtype=torch.float64, device="cuda")
            dst = torch.empty_like(src)

            def loc_with_copy():
                main = torch.cuda.current_stream()
                S_HI.wait_stream(main)
                with torch.cuda.stream(S_HI):
                    dst.copy_(src)
                A_loc.spmv(y, x)
                main.wait_stream(S_HI)

            tlc = timeit(loc_with_copy, a.reps) if cbytes > 0 else tl
            tcopy = timeit(lambda: dst.copy_(src), a.reps) if cbytes > 0 else 0.0
            del src, dst
            tp = h.info["packed_send"] * sv * 2 / 5.5e12  # pack: read + write at ~5.5 TB/s
            tc = max(send, recv) / B_LINK
            ranks.append(dict(rank=r, t_loc_us=tl * 1e6, t_nl_us=tn * 1e6, t_comm_us=tc * 1e6, t_pack_us=tp * 1e6,
                              t_model_us=(max(tl, tp + tc) + tn) * 1e6,
                              t_loc_with_copy_us=tlc * 1e6, t_copy_alone_us=tcopy * 1e6,
                              t_model_contended_us=(max(tlc, tp + tc) + tn) * 1e6, halo=h.info["halo"], n_loc=nl,
                              nnz_nl=h.info["nnz_nonlocal_part"], messages=h.info["send_messages"]))
        tmax = max(r["t_model_us"] for r in ranks)
        tmaxc = max(r["t_model_contended_us"] for r in ranks)
        if R == 1:
            t1[mode] = tmax
        eff = t1.get(mode, tmax) / (R * tmax)
        effc = t1.get(mode, tmax) / (R * tmaxc)
        print(json.dumps({"config": a.config, "dtype": a.dtype, "mode": mode, "R": R, "t_model_max_us": round(tmax, 1),
                          "gflops_model": round(2 * nnz / (tmax * 1e-6) / 1e9, 1), "efficiency_model": round(eff, 3),
                          "t_model_contended_max_us": round(tmaxc, 1), "efficiency_model_contended": round(effc, 3),
                          "t1_single_gpu_kernel_us": round(t_single * 1e6, 1) if t_single else None,
                          "efficiency_vs_single_gpu_kernel": round(t_single * 1e6 / (R * tmaxc), 3) if t_single else None,
                          "ranks": [{k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()} for r in ranks]}),
              flush=True)
        del hs
        torch.cuda.empty_cache()
