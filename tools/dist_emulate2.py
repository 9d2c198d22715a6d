"""Single-GPU emulation of one rank of the row-partitioned NCCL dist spMVM under its own HBM load
(dev tool; a model, NOT a bench number).  Replaces the r01 model's "A_loc beside a copy" with the
whole per-call sequence of one rank, timed as one stream-ordered unit on one B200:

  side stream (high priority): [pack: gather of the packed send entries from x]
                               -> [exchange: a device copy of max(send, recv) bytes, i.e. the
                                   send reads + halo writes that NCCL puts on this rank's HBM]
  main stream                : A_loc (y = ...)  ->  wait(side)  ->  A_nl (y += ...)

so the pack and the exchange contend with A_loc for HBM, and A_nl runs with whatever A_loc and the
exchange left in L2, exactly as on a real rank.  NVLink is not emulated (a local copy is faster
than a peer link), so t_rank = max(T_unit, T_pack + halo_bytes / B_link + T_nl); efficiency =
T_1 / (R * max_r t_rank) with T_1 = the single-GPU kernel on the whole matrix (same basis).
Variants: --ystore (A_loc y-store override, pjds_set_y_store) and --pstore (scattered +=
policy of A_nl, pjds_set_cache_policy bits 16-23)."""
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
p.add_argument("--ranks", default="2,4,8")
p.add_argument("--dtype", default="f64")
p.add_argument("--modes", default="permuted")
p.add_argument("--ystore", default="-1", help="comma list of A_loc y-store overrides (-1 default, 0 plain, 1+kind)")
p.add_argument("--pstore", default="0", help="comma list of perm-store kinds for A_nl (0 plain, 1+kind)")
p.add_argument("--all-ranks", action="store_true", help="emulate every rank (default: ranks 0 and R/2)")
p.add_argument("--reps", type=int, default=20)
p.add_argument("--nl-sigma", default="1024", help="comma list of A_nl sort scopes (pjds_set_dist_nl_sigma)")
p.add_argument("--nl-variants", default="", help="comma list RxU: time A_nl alone under each kernel variant")
a = p.parse_args()
SEG = {"C1": 1024, "C3": 15504, "C5": 142506}[a.config]
npdt = np.float64 if a.dtype == "f64" else np.float32
sv = np.dtype(npdt).itemsize
tdt = torch.float64 if sv == 8 else torch.float32
n, rp, col, val = inputs.config_crs(a.config, dtype=npdt)
nnz = len(col)
xg = inputs.vector(n, npdt)
B_LINK = 770e9
S_HI = torch.cuda.Stream(priority=-1)
main = torch.cuda.current_stream()


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


t_single = {}
for mode in a.modes.split(","):
    A1 = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=32, symmetric=(mode == "permuted"))
    x1 = torch.from_numpy(xg).cuda()
    if mode == "permuted":
        x1 = A1.to_permuted(torch.empty_like(x1), x1)
    y1 = torch.empty_like(x1)
    t_single[mode] = timeit(lambda: A1.spmv(y1, x1), a.reps)
    del A1, x1, y1
    torch.cuda.empty_cache()

for mode, R, nls in [(m_, r_, s_) for m_ in a.modes.split(",") for r_ in map(int, a.ranks.split(","))
                     for s_ in map(int, a.nl_sigma.split(","))]:
    if True:
        nb = n // SEG
        offs = np.array([(nb * r // R) * SEG for r in range(R + 1)], np.int64)
        offs[-1] = n
        assert pj.lib().pjds_set_dist_nl_sigma(nls) == 0
        hs = pj.DistPjds.create_group(n, rp, col, val, offs, permuted=(mode == "permuted"))
        which = range(R) if a.all_ranks else sorted({0, R // 2})
        for ys in map(int, a.ystore.split(",")):
            for ps in map(int, a.pstore.split(",")):
                pj.lib().pjds_set_cache_policy(1 | (2 << 8) | (ps << 16), 2)
                ranks = []
                for r in which:
                    h = hs[r]
                    nl = int(offs[r + 1] - offs[r])
                    A_loc, A_nl = h.parts()
                    pj.lib().pjds_set_y_store(A_loc._h, ys)
                    x = torch.from_numpy(xg[offs[r]:offs[r + 1]].copy()).cuda()
                    halo = torch.from_numpy(np.resize(xg, max(h.info["halo"], h.info["rows_nonlocal"], 1))).cuda()
                    y = torch.empty(max(nl, 1), dtype=tdt, device="cuda")
                    npk = h.info["packed_send"]
                    idx = torch.randint(0, max(nl, 1), (max(npk, 1),), device="cuda") if npk else None
                    packbuf = torch.empty(max(npk, 1), dtype=tdt, device="cuda")
                    xb = max(h.info["send_total"], h.info["halo"]) * sv
                    src = torch.zeros(max(xb // 8, 1), dtype=torch.float64, device="cuda")
                    dst = torch.empty_like(src)

                    def side():
                        if idx is not None:
                            torch.index_select(x, 0, idx, out=packbuf)
                        if xb:
                            dst.copy_(src)

                    def unit():
                        S_HI.wait_stream(main)
                        with torch.cuda.stream(S_HI):
                            side()
                        A_loc.spmv(y, x)
                        main.wait_stream(S_HI)
                        if A_nl is not None:
                            A_nl.spmv_accum(y, halo)

                    t_unit = timeit(unit, a.reps)
                    t_loc = timeit(lambda: A_loc.spmv(y, x), a.reps)
                    t_side = timeit(lambda: side(), a.reps)
                    t_pack = timeit(lambda: torch.index_select(x, 0, idx, out=packbuf), a.reps) if idx is not None else 0.0

                    t_nl = timeit(lambda: A_nl.spmv_accum(y, halo), a.reps) if A_nl is not None else 0.0
                    nl_var = {}
                    for v in [q for q in a.nl_variants.split(",") if q]:
                        vr, vu = map(int, v.split("x"))
                        pj.lib().pjds_set_kernel_variant(vr, vu)
                        nl_var[v] = round(timeit(lambda: A_nl.spmv_accum(y, halo), a.reps) * 1e6, 1) if A_nl is not None else 0.0
                    pj.lib().pjds_set_kernel_variant(0, 0)
                    t_link = t_pack + xb / 2 / B_LINK + t_nl  # one direction's bytes over NVLink
                    ranks.append({"rank": r, "t_unit_us": t_unit * 1e6, "t_loc_us": t_loc * 1e6,
                                  "t_nl_us": t_nl * 1e6, "t_side_us": t_side * 1e6, "t_pack_us": t_pack * 1e6,
                                  "t_link_path_us": t_link * 1e6, "t_rank_us": max(t_unit, t_link) * 1e6,
                                  "halo": h.info["halo"], "packed_send": npk, "rows_nl": h.info["rows_nonlocal"],
                                  "t_nl_by_variant_us": nl_var or None})
                    pj.lib().pjds_set_y_store(A_loc._h, -1)
                    del src, dst, x, y, halo, packbuf
                tmax = max(rr["t_rank_us"] for rr in ranks)
                print(json.dumps({"config": a.config, "dtype": a.dtype, "mode": mode, "R": R, "ystore": ys, "pstore": ps,
                                  "nl_sigma": nls,
                                  "t1_us": round(t_single[mode] * 1e6, 1), "t_rank_max_us": round(tmax, 1),
                                  "efficiency_vs_t1": round(t_single[mode] * 1e6 / (R * tmax), 4),
                                  "ranks": [{k: (round(v, 1) if isinstance(v, float) else v) for k, v in rr.items()}
                                            for rr in ranks]}), flush=True)
        pj.lib().pjds_set_cache_policy(1 | (2 << 8) | (2 << 16), 2)
        del hs
        torch.cuda.empty_cache()
