"""Kernel sweep (development tool): every config x format x dtype, CUDA-event timed, one JSON line each.
Not the bench contract (bench.py is); used to pick kernel variants and to drive ncu passes."""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import inputs
try:
    import pynvml
    pynvml.nvmlInit()
    _nvh = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    _nvh = None


def clocks():
    if _nvh is None:
        return None
    return (pynvml.nvmlDeviceGetClockInfo(_nvh, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetClockInfo(_nvh, pynvml.NVML_CLOCK_MEM),
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(_nvh), pynvml.nvmlDeviceGetTemperature(_nvh, 0))
import paper_1112_5588_b200 as pj

p = argparse.ArgumentParser()
p.add_argument("--configs", default="C2,C3,C4,C5")
p.add_argument("--dtypes", default="f64,f32")
p.add_argument("--fmts", default="pjds32,pjds64,pjds128,ellr")
p.add_argument("--reps", type=int, default=30)
p.add_argument("--variants", default="0x0")
p.add_argument("--policies", default="513x2", help="stream x x; stream bits 8-15 = y store (0 plain, 1+kind vector); 513x2 = the library default")
p.add_argument("--orders", default="2")
p.add_argument("--scheds", default="0", help="0 static CTA grid, 1 dynamic warp tiles")
p.add_argument("--sigmas", default="0")
p.add_argument("--keys", default="none", help="tile keys: none (original index) or wW = HMEp phonon window of W rows")
SEG = {"C1": 1024, "C3": 15504, "C5": 142506}
p.add_argument("--once", action="store_true", help="single launch per variant (for ncu)")
p.add_argument("--pdls", default="0:0", help="launch overlap mode:prefetch_cols list (pjds_set_launch_overlap)")
p.add_argument("--rotate", type=int, default=1, help="x/y pairs cycled over the timed launches (L2 carry-over)")
p.add_argument("--compress", type=int, default=1, help="pjds_set_compression mode for the handles built")
a = p.parse_args()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.3
assert pj.lib().pjds_set_compression(a.compress) == 0
pj.bw_probe(1 << 30, 20)  # bring the GPU out of its idle clocks before the first measurement
for cfg in a.configs.split(","):
    for dts in a.dtypes.split(","):
        npdt = np.float64 if dts == "f64" else np.float32
        sv = np.dtype(npdt).itemsize
        n, rp, col, val = inputs.config_crs(cfg, dtype=npdt)
        nnz = len(col)
        x = torch.from_numpy(inputs.vector(n, npdt)).cuda()
        y = torch.empty_like(x)
        xs = [x] + [x.clone() for _ in range(a.rotate - 1)]
        ys = [y] + [torch.empty_like(x) for _ in range(a.rotate - 1)]
        bmin = nnz * (sv + 4) + 2 * n * sv
        for fmt, sg in [(f, g) for f in a.fmts.split(",") for g in (a.sigmas.split(",") if f.startswith("pjds") else ["0"])]:
          if fmt.startswith("pjds"):
              sym = fmt.endswith("s")
              A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=int(fmt[4:].rstrip("s")), symmetric=sym,
                                         sigma=int(sg))
          else:
              A = pj.EllrMatrix.from_crs(n, rp, col, val)
          pj.bw_probe(1 << 30, 20)  # host-side conversion leaves the GPU idle: re-raise clocks
          for var, polk, order, kspec, sch, pdl in [(v, q, o, kk, sc, pd) for v in a.variants.split(",") for q in a.policies.split(",")
                                               for o in a.orders.split(",") for kk in a.keys.split(",")
                                               for sc in a.scheds.split(",") for pd in a.pdls.split(",")]:
            pj.lib().pjds_set_schedule(int(sch))
            pm, pf = map(int, pdl.split(":"))
            assert pj.lib().pjds_set_launch_overlap(pm, pf) == 0
            if fmt.startswith("pjds"):
                if kspec == "none":
                    A.set_tile_keys(None)
                else:  # 2-D order: phonon window of the row, then the original index
                    W, P = int(kspec[1:]), SEG[cfg]
                    r = np.arange(n, dtype=np.int64)
                    A.set_tile_keys(((r % P) // W) * n + r)
            pj.lib().pjds_set_tile_order(int(order))
            vr, vu = map(int, var.split("x"))
            pj.lib().pjds_set_kernel_variant(vr, vu)
            ps, px = map(int, polk.split("x"))
            pj.lib().pjds_set_cache_policy(ps, px)

            if a.once:
                A.spmv(y, x); torch.cuda.synchronize(); continue
            # warm-up by time, not by count: after the host-side matrix build the GPU has idled and
            # its clocks ramp for tens of ms (a 5-launch warm-up left the first variant 25 % slow)
            t_w = time.perf_counter()
            while time.perf_counter() - t_w < 0.1:
                for _ in range(5): A.spmv(y, x)
                torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(a.reps): A.spmv(ys[i % a.rotate], xs[i % a.rotate])
            e1.record()
            ck = clocks()  # after e1 is enqueued: a slow first NVML query must not delay e1 (it did: C2 +28 us)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / a.reps * 1e-3
            print(json.dumps({"cfg": cfg, "dtype": dts, "fmt": fmt, "var": var, "pol": polk, "order": order, "sched": int(sch), "keys": kspec, "sigma": int(sg), "pdl": pdl, "rotate": a.rotate, "us": round(t * 1e6, 1), "gflops": round(2 * nnz / t / 1e9, 1),
                              "eff_gbs": round(bmin / t / 1e9, 1), "frac": round(bmin / t / 1e9 / peak, 3),
                              "stored_bytes": A.info.get("bytes_total"), "col_compressible": A.info.get("col_compressible"), "clk": ck}), flush=True)
          del A
        del rp, col, val
