#!/usr/bin/env python
"""Benchmark of the pJDS spMVM hot path (BASELINE.json metric: pJDS DP spMVM GFlop/s and HBM GB/s
(% roofline) at 1/2/4/8 B200; bytes vs ELLPACK-R).

One step = one y = A x over the whole matrix (SURVEY §8(a) a7+a8 at N=1; a12 = local part
overlapped with the NCCL halo exchange + nonlocal part at N>1).  Default workload C5: HMEp-shaped
Holstein-Hubbard matrix, M = 25 phonons, N = 57,002,400, nnz = 942,439,680, DP, synthetic values
(inputs/gen.cpp), the same matrix for every N (strong scaling, rows partitioned on e-block
boundaries of the nested spin-grid ordering).

At N=1 the product runs in the permuted basis (PJDS_PERM_SYMMETRIC), the paper's usage for
iterative solvers: "permutation of the indices needs to be done only before the start and after
the end of the algorithm, while the complete iterative scheme works on the permuted elements"
(PAPER.md L241-246); x is permuted once before the timed region (--basis rows: y stored through
perm every step instead).  The rows-only pJDS and ELLPACK-R kernels are timed beside it
("compare").  e2e includes the basis change on the GPU, both ways, every step.

  python bench.py [--gpus N --steps K --warmup W] [--config C5] [--dtype f64|f32] [--impl pjds|ellr|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.  Timing: CUDA events on the launching stream around exactly K
steps, barrier + synchronize on both sides, max over ranks.  The matrix (12.2 GB at C5 DP) is far
larger than L2, so no explicit flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_DESC = {
    "C1": "tiny HMEp-shaped banded N=16384",
    "C2": "sAMG-shaped 7-point Poisson 150x150x151 Morton, N=3397500",
    "C3": "HMEp Holstein-Hubbard M=15, N=6201600",
    "C4": "DLR1-shaped 46417 points x 6, N=278502",
    "C5": "HMEp Holstein-Hubbard M=25 nested spin-grid, N=57002400",
    "W4": "DLR2-shaped 108396 points x 5 (dense 5x5 blocks), N=541980, N_nzr~314",
    "W5": "UHBR-shaped 900000 points x 5, N=4500000, N_nzr~122",
}
METRIC = "pJDS DP spMVM GFlop/s & HBM GB/s (% roofline) at 1/2/4/8 B200; bytes vs ELLPACK-R"
# electronic-block size P (rows per contiguous off-diagonal segment) for partitioning
SEGMENT = {"C1": 1024, "C3": 15504, "C5": 142506}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="pjds", choices=["pjds", "ellr", "reference"])
    p.add_argument("--config", default="C5", choices=sorted(CONFIG_DESC))
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    p.add_argument("--basis", default="permuted", choices=["permuted", "rows"])
    p.add_argument("--block-rows", type=int, default=32, help="pJDS b_r (the paper's warp size; 128 = rows per warp at R=4)")
    p.add_argument("--no-overlap", action="store_true", help="dist: vector mode (exchange, then compute)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-compare", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=30)
    p.add_argument("--tile-window", type=int, default=0,
                   help="HMEp configs, N=1: run tiles by (phonon window of this many rows, original row); 0 = off")
    p.add_argument("--probe-bytes", type=int, default=4 << 30)
    p.add_argument("--dist", action="store_true", help="use the distributed path even at N=1 (one-rank NCCL group)")
    p.add_argument("--transport", default="nccl", choices=["nccl", "p2p", "direct"],
                   help="dist: NCCL send/recv on a side stream, the fused gather+put P2P kernel, or DIRECT "
                        "(no exchange: one kernel whose nonlocal gathers read the owners' x windows)")
    return p.parse_args()


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self._nv = None
            self.error = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                self.reasons |= self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self._nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        r = [name for bit, name in self.REASONS.items() if self.reasons & bit and name != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": r, "samples": len(self.samples)}


def committed_traffic(key: str):
    """DRAM bytes per launch of the bench kernel from the committed ncu capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            return json.load(f).get(key, {}).get("traffic")
    except Exception:
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _allreduce(dist, t, op):
    """all_reduce of a small CUDA tensor on either backend (gloo reduces host copies)."""
    o = dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM
    if dist.get_backend() == "gloo":
        c = t.cpu()
        dist.all_reduce(c, op=o)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=o)


# ------------------------------------------------------------------------------------------ CPU oracle
def time_oracle(n, rp, col, val, x, budget_s: float, max_reps: int, min_reps: int = 1, threads: int = 0,
                warmup: int = 1):
    """The oracle's plain CRS loop (oracle_spmv_crs: OpenMP static over rows, all visible cores or
    `threads`), repeated until the time budget is spent.  Returns (median s per product, reps, cores,
    total s, y of the warm-up product)."""
    import oracle
    cores = threads or len(os.sched_getaffinity(0))
    for _ in range(max(warmup, 1)):
        y_cpu = oracle.spmv_crs(n, rp, col, val, x, nthreads=cores)
    ts = []
    t_end = time.perf_counter() + budget_s
    while (time.perf_counter() < t_end and len(ts) < max_reps) or len(ts) < min_reps:
        t0 = time.perf_counter()
        oracle.spmv_crs(n, rp, col, val, x, nthreads=cores)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), len(ts), cores, float(sum(ts)), y_cpu


def parity_vs_cpu(y_gpu, y_cpu, rp, col, val, x, rows):
    """SURVEY §8(d) step 6, parity in the same run: sampled rows of the GPU product against the
    cpu_baseline leg's own product on the same inputs.  Both are O2-bounded approximations of the
    exact row sum, so |y_gpu - y_cpu| <= 2 * 4 nnz_i eps sum_j |a_ij x_j| (triangle inequality)."""
    lens = (rp[rows + 1] - rp[rows]).astype(np.int64)
    idx = np.repeat(rp[rows], lens) + (np.arange(int(lens.sum())) - np.repeat(np.cumsum(lens) - lens, lens))
    bound = np.zeros(len(rows))
    np.add.at(bound, np.repeat(np.arange(len(rows)), lens), np.abs(val[idx].astype(np.float64) * x[col[idx]]))
    eps = np.finfo(val.dtype).eps
    diff = np.abs(y_gpu[rows].astype(np.float64) - y_cpu[rows].astype(np.float64))
    tol = 8.0 * lens * eps * bound * (1 + 1e-6)
    ok = (diff <= tol) & np.isfinite(y_gpu[rows])
    rel = diff / np.maximum(bound, np.finfo(np.float64).tiny)
    return {"rows_checked": int(len(rows)), "within_bound": bool(ok.all()), "rows_outside": int((~ok).sum()),
            "max_err_over_sum_abs": float(rel.max()) if len(rows) else 0.0,
            "bound": "|y_gpu - y_cpu| <= 8 nnz_i eps sum_j |a_ij x_j| (both O2-bounded)",
            "reference": "the cpu_baseline leg's oracle_spmv_crs product on the same inputs",
            "gpu_finite_all_rows": bool(np.isfinite(y_gpu).all())}


# ------------------------------------------------------------------------------------------ main
def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    npdt = np.float64 if a.dtype == "f64" else np.float32
    sv = np.dtype(npdt).itemsize

    if a.impl == "reference":
        if rank != 0:
            return 0
        return reference_arm(a, world, npdt)

    import torch
    import inputs
    import paper_1112_5588_b200 as pj
    from paper_1112_5588_b200 import perfmodel

    ngpu = torch.cuda.device_count()
    dev_index = local_rank % max(ngpu, 1)  # more ranks than GPUs only in the one-GPU transport test
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    tdt = torch.float64 if npdt == np.float64 else torch.float32
    dist = None
    use_dist = world > 1 or a.dist
    if use_dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29611")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        if world <= ngpu:
            dist.init_process_group("nccl", device_id=dev)
        else:  # oversubscribed (test of the transport on one GPU): NCCL refuses duplicate GPUs
            dist.init_process_group("gloo")

    t_setup = time.perf_counter()
    g = inputs.Generator.from_config(a.config)
    n = g.n
    if use_dist:
        seg = SEGMENT.get(a.config, 32)
        nb = n // seg
        offs = np.array([(nb * r // world) * seg for r in range(world + 1)], np.int64)
        offs[-1] = n
    else:
        offs = np.array([0, n], np.int64)
    lo, hi = int(offs[rank]), int(offs[rank + 1])
    rp, col, val = g.crs(lo, hi, dtype=npdt)
    nnz_loc = int(rp[-1])
    x_host = inputs.vector(hi - lo, npdt, i0=lo)
    permuted = a.impl == "pjds" and a.basis == "permuted"
    compare = {}
    footprint = None
    if use_dist:
        D = pj.DistPjds.create(n, offs, rp, col, val, block_rows=a.block_rows, permuted=permuted,
                               transport=a.transport)
        A = None
    else:
        if a.impl == "ellr":
            A = pj.EllrMatrix.from_crs(n, rp, col, val)
        else:
            A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=a.block_rows, symmetric=permuted)
            if a.tile_window:  # opt-in 2-D (phonon window, original row) tile order for HMEp
                r_ = np.arange(n, dtype=np.int64)
                A.set_tile_keys(((r_ % SEGMENT[a.config]) // a.tile_window) * n + r_)
                del r_
            st = A.info
            ell_rows = (n + 31) // 32 * 32
            ell_entries = ell_rows * st["len_max"]
            footprint = {"pjds_bytes": st["bytes_total"], "pjds_stored": st["stored"],
                         "ellr_bytes": ell_entries * (sv + 4) + ell_rows * 4, "ellr_stored": ell_entries,
                         "data_reduction_vs_ellpack": round(st["data_reduction_vs_ellpack"], 5),
                         "padding_entries": st["stored"] - st["nnz"]}
            footprint["bytes_ratio_pjds_over_ellr"] = round(footprint["pjds_bytes"] / footprint["ellr_bytes"], 4)
    # CPU oracle baseline on the same matrix (rank 0, N=1 only), bounded to ~10 s
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        t, reps, cores, tot, y_cpu = time_oracle(n, rp, col, val, x_host, budget_s=10.0, max_reps=200)
        cpu = {"value": round(2.0 * nnz_loc / t / 1e9, 3), "unit": "GFlop/s", "cores": cores, "kind": "oracle",
               "sample": f"whole {a.config} matrix ({nnz_loc} nnz), {reps} products, median; {tot:.1f} s of "
                         f"oracle_spmv_crs ({np.dtype(npdt).name}, OpenMP {cores} threads)"}
        t1, reps1, _, _, _ = time_oracle(n, rp, col, val, x_host, budget_s=3.0, max_reps=3, threads=1)
        cpu["single_thread"] = {"value": round(2.0 * nnz_loc / t1 / 1e9, 3), "reps": reps1}
    nnz = nnz_loc
    if use_dist:
        tt = torch.tensor([nnz_loc], dtype=torch.int64, device=dev)
        _allreduce(dist, tt, "sum")
        nnz = int(tt.item())
    x = torch.from_numpy(x_host).to(dev)
    y = torch.empty(hi - lo, dtype=tdt, device=dev)
    if permuted:
        xp = torch.empty_like(x)
        (D if use_dist else A).to_permuted(xp, x)  # once, before the "iterative scheme"
        x = xp
    if use_dist and a.transport == "direct":  # x lives in the exported window: no per-call copy
        w = D.x_window()
        w.copy_(x)
        x = w
    t_setup = time.perf_counter() - t_setup

    # roofline denominator measured in this run (copy and read streams)
    probe_copy, probe_read = pj.bw_probe(a.probe_bytes, 5)
    peak_file = measured_peaks().get("hbm_gbs")
    stream = torch.cuda.current_stream()

    def step():
        if use_dist:
            D.spmv(y, x, stream=stream, no_overlap=a.no_overlap)
        else:
            A.spmv(y, x, stream=stream)

    def timed(fn, k):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = pj.launch_count()
    with ClockSampler(dev_index) as clk:
        ms = timed(step, a.steps)
    launches = pj.launch_count() - launches0
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    if use_dist:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        _allreduce(dist, tt, "max")
        ms = float(tt.item())
        lt = torch.tensor([launches], dtype=torch.int64, device=dev)
        _allreduce(dist, lt, "sum")
        launches = int(lt.item())
    # SURVEY §8(d) protocol beside the contract timing: 5 trials of >= 20 ms of back-to-back steps
    kt = max(10, int(np.ceil(20.0 / max(ms, 1e-3))))
    tr = []
    for _ in range(5):
        if use_dist:
            dist.barrier()
        tr.append(timed(step, kt))
    if use_dist:
        tv = torch.tensor(tr, dtype=torch.float64, device=dev)
        _allreduce(dist, tv, "max")
        tr = tv.tolist()
    trials = {"n": 5, "steps_each": kt, "median_ms": round(float(np.median(tr)), 5), "best_ms": round(min(tr), 5),
              "best_gflops": round(2.0 * nnz / (min(tr) * 1e-3) / 1e9, 2)}
    parity = None
    if cpu is not None:  # same-run parity against the cpu_baseline leg's product
        yo = y
        if permuted:
            yo = torch.empty_like(y)
            A.from_permuted(yo, y)
        y_gpu_host = yo.cpu().numpy()
        rows = np.unique(np.concatenate([np.random.default_rng(7).integers(0, n, 100000), [0, n - 1]]))
        parity = parity_vs_cpu(y_gpu_host, y_cpu, rp, col, val, x_host, rows)
        del y_gpu_host, y_cpu
    dist_info = None
    if use_dist:
        # vector mode (exchange, then compute) as the reference point for "communication hidden",
        # and one traced call of each mode: per-phase device times, max over ranks
        dist.barrier()
        ms_no = timed(lambda: D.spmv(y, x, stream=stream, no_overlap=True), max(5, a.steps // 4))
        tt = torch.tensor([ms_no], dtype=torch.float64, device=dev)
        _allreduce(dist, tt, "max")
        ms_no = float(tt.item())
        phases = {}
        for mode, no in (("task", False), ("vector", True)):
            dist.barrier()
            D.spmv(y, x, stream=stream, no_overlap=no, trace=True)
            ph = D.trace()
            vec = torch.tensor([ph[k] for k in sorted(ph)], dtype=torch.float64, device=dev)
            _allreduce(dist, vec, "max")
            phases[mode] = {k: round(v, 4) for k, v in zip(sorted(ph), vec.tolist())}
        tp = phases["task"]
        comm = max(tp["exchange"], 1e-9)
        dist_info = {"ms_vector_mode": round(ms_no, 4), "speedup_task_over_vector": round(ms_no / ms, 3),
                     "phases_ms_max_over_ranks": phases,
                     "hidden_fraction": round(1.0 - max(0.0, tp["total"] - tp["local"] - tp["nonlocal"]
                                                        - tp["pack"]) / comm, 3),
                     "halo_entries_rank0": D.info["halo"], "nnz_nonlocal_rank0": D.info["nnz_nonlocal_part"],
                     "messages_rank0": D.info["send_messages"]}
    t_s = ms * 1e-3
    gflops = 2.0 * nnz / t_s / 1e9
    # algorithmic bytes (Eq. 1 at alpha = 1/N_nzr, write-only y): val+col once, x once, y once
    b_min = nnz * (sv + 4) + 2 * n * sv
    achieved = b_min / t_s / 1e9 / world  # per GPU
    peak = peak_file if peak_file else max(probe_copy, probe_read)

    traffic_key = (f"{a.config}/{a.dtype}/{a.basis}" + ("" if a.block_rows == 32 else f"/br{a.block_rows}")
                   + (f"/tw{a.tile_window}" if a.tile_window else ""))

    # side-by-side kernels on the same matrix (N=1): rows-only pJDS and ELLPACK-R
    if not use_dist and a.impl == "pjds" and not a.no_compare:
        x0 = torch.from_numpy(x_host).to(dev)
        legs = [("pjds_rows_only" if permuted else "pjds_permuted",
                 lambda: pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=a.block_rows, symmetric=not permuted)),
                ("ellpack_r", lambda: pj.EllrMatrix.from_crs(n, rp, col, val))]
        # b_r sweep point: b_r = 32 (paper) vs 128 (= rows one warp owns at R=4)
        br_alt = 128 if a.block_rows == 32 else 32
        legs.insert(0, (f"pjds_br{br_alt}", lambda: pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br_alt,
                                                                           symmetric=permuted)))
        for name, mk in legs:
            B = mk()
            for _ in range(3):
                B.spmv(y, x0, stream=stream)
            mb = timed(lambda: B.spmv(y, x0, stream=stream), 20)
            compare[name] = {"GFlop/s": round(2.0 * nnz / (mb * 1e-3) / 1e9, 1), "ms": round(mb, 4),
                             "frac": round(b_min / (mb * 1e-3) / 1e9 / peak, 4),
                             "bytes": B.info["bytes_total"]}
            del B
            torch.cuda.synchronize()
        # NVIDIA's library CRS SpMV on the same matrix and the same device (cuSPARSE via torch.sparse
        # CSR): the vendor baseline beside the pJDS kernel, not part of the product path
        warnings.filterwarnings("ignore", message="Sparse CSR tensor support is in beta")
        C = torch.sparse_csr_tensor(torch.from_numpy(rp.astype(np.int32)).to(dev), torch.from_numpy(col).to(dev),
                                    torch.from_numpy(val).to(dev), size=(n, n), check_invariants=False)
        for _ in range(3):
            torch.mv(C, x0)
        mb = timed(lambda: torch.mv(C, x0), 20)
        compare["cusparse_csr"] = {"GFlop/s": round(2.0 * nnz / (mb * 1e-3) / 1e9, 1), "ms": round(mb, 4),
                                   "frac": round(b_min / (mb * 1e-3) / 1e9 / peak, 4),
                                   "bytes": int(nnz * (sv + 4) + (n + 1) * 4)}
        del C
        torch.cuda.synchronize()
        del x0
    del col, val

    # end-to-end through the public API with host buffers in the original basis (H2D x, basis
    # change, kernel, basis change back, D2H y, every step)
    e2e = None
    model = None
    if not use_dist and a.impl == "pjds":
        xh = torch.from_numpy(x_host).pin_memory().numpy()
        yh = torch.empty(n, dtype=tdt).pin_memory().numpy()
        A.spmv_host(yh, xh)
        te = timed(lambda: A.spmv_host(yh, xh), a.e2e_steps) * 1e-3
        # pipelined (pjds_spmv_host_batch): H2D of step i+1 and D2H of step i-1 overlap product i;
        # every step still moves its own x in and its own y out
        xh2 = torch.from_numpy(inputs.vector(n, npdt, seed=inputs.BASE_SEED + 7)).pin_memory().numpy()
        yh2 = torch.empty(n, dtype=tdt).pin_memory().numpy()
        xs = [xh, xh2] * ((a.e2e_steps + 1) // 2)
        ys = [yh, yh2] * ((a.e2e_steps + 1) // 2)
        A.spmv_host_batch(ys[:2], xs[:2])
        tb = timed(lambda: A.spmv_host_batch(ys[:a.e2e_steps], xs[:a.e2e_steps]), 1) * 1e-3 / a.e2e_steps
        e2e = {"value": round(2.0 * nnz / tb / 1e9, 2), "unit": "GFlop/s", "h2d_bytes_per_step": n * sv,
               "d2h_bytes_per_step": n * sv, "ms_per_step": round(tb * 1e3, 3),
               "mode": f"pjds_spmv_host_batch of {a.e2e_steps} products, pinned host buffers, original basis",
               "unpipelined": {"value": round(2.0 * nnz / te / 1e9, 2), "ms_per_step": round(te * 1e3, 3),
                               "mode": "pjds_spmv_host per step (H2D, basis change, kernel, basis change, D2H)"}}
        # the bound of the pipelined leg: x in and y out at once on two streams, same pinned buffers
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        dx_, dy_ = torch.empty(n, dtype=tdt, device=dev), torch.empty(n, dtype=tdt, device=dev)
        hx_, hy_ = torch.from_numpy(xh), torch.from_numpy(yh)

        def duplex():
            s_in.wait_stream(torch.cuda.current_stream())
            s_out.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_in):
                dx_.copy_(hx_, non_blocking=True)
            with torch.cuda.stream(s_out):
                hy_.copy_(dy_, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s_in)
            torch.cuda.current_stream().wait_stream(s_out)

        duplex()
        tp = timed(duplex, 10) * 1e-3
        e2e["pcie_duplex_ms"] = round(tp * 1e3, 3)
        e2e["frac_of_pcie_duplex"] = round(tp / tb, 3)
        del dx_, dy_
        # the paper's PCIe model (Eq. 2-4) with this box's measured bandwidths:
        # B_PCI from the e2e transfer time, B_GPU = the read probe
        t_pci_meas = max(te - t_s, 1e-9)
        b_pci = 2 * n * sv / t_pci_meas
        ratio = max(probe_copy, probe_read) * 1e9 / b_pci
        traffic = committed_traffic(traffic_key)
        alpha = (perfmodel.measured_alpha(traffic - n * sv, A.info["stored"], nnz, n, sv,
                                          aux_bytes=A.info["bytes_aux"] - A.info["n"] * 4 * permuted)
                 if traffic else None)
        model = {"B_pci_GBs": round(b_pci / 1e9, 1), "B_gpu_over_B_pci": round(ratio, 1),
                 "alpha_measured": round(alpha, 4) if alpha is not None else None,
                 "alpha_ideal": round(n / nnz, 4),
                 "eq3_nnzr_upper_50pct_penalty": round(perfmodel.n_nzr_upper(ratio, alpha or perfmodel.RECIPROCAL), 1),
                 "eq4_nnzr_lower_10pct_penalty": round(perfmodel.n_nzr_lower(ratio, alpha or perfmodel.RECIPROCAL), 1),
                 "n_nzr": round(nnz / n, 2),
                 "pci_share_of_e2e": round(t_pci_meas / te, 3)}
    elif use_dist:
        # per rank: pinned host x_loc -> device, basis change, dist product, basis change back,
        # device -> pinned host y_loc, every step; max over ranks
        xh = torch.from_numpy(x_host).pin_memory()
        yh = torch.empty(hi - lo, dtype=tdt).pin_memory()
        xd, yd = torch.empty_like(x), torch.empty_like(y)
        xw, yw = torch.empty_like(x), torch.empty_like(y)

        def e2e_step():
            xd.copy_(xh, non_blocking=True)
            if permuted:
                D.to_permuted(xw, xd, stream=stream)
                D.spmv(yw, xw, stream=stream, no_overlap=a.no_overlap)
                D.from_permuted(yd, yw, stream=stream)
            else:
                D.spmv(yd, xd, stream=stream, no_overlap=a.no_overlap)
            yh.copy_(yd, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        te = timed(e2e_step, a.e2e_steps) * 1e-3
        tt = torch.tensor([te], dtype=torch.float64, device=dev)
        _allreduce(dist, tt, "max")
        te = float(tt.item())
        e2e = {"value": round(2.0 * nnz / te / 1e9, 2), "unit": "GFlop/s", "h2d_bytes_per_step": n * sv,
               "d2h_bytes_per_step": n * sv, "ms_per_step": round(te * 1e3, 3),
               "note": "all ranks' pinned host buffers; max over ranks"}

    if rank == 0:
        wl = f"{a.config}: {CONFIG_DESC[a.config]}, nnz={nnz}, {a.dtype}, {a.impl}"
        if a.impl == "pjds":
            wl += ", permuted basis (PAPER.md L241-246)" if permuted else ", original basis (rows permuted)"
        out = {
            "metric": METRIC,
            "value": round(gflops, 2), "unit": "GFlop/s", "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": a.dtype,
            "data": "synthetic (inputs/gen.cpp, seed 0x11125588)",
            "config": {"workload": wl, "n": n, "nnz": nnz, "block_rows": a.block_rows,
                       "parallelism": f"row-partition r{world}" if world > 1 else "single GPU",
                       "overlap": (not a.no_overlap) if use_dist else None,
                       "transport": a.transport if use_dist else None,
                       "tile_window": a.tile_window or None,
                       "l2": f"inputs larger than L2: {b_min / 1e9:.2f} GB streamed per step, no flush"},
            "hbm_gbs_effective": round(b_min / t_s / 1e9, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": (committed_traffic(traffic_key)
                                     if not use_dist and a.impl == "pjds" else None),
                         "traffic_source": "profiles/r01_traffic.json (ncu --set full, per launch)",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if peak_file else "bw probe (this run)",
                         "probe_copy_gbs": round(probe_copy, 1), "probe_read_gbs": round(probe_read, 1),
                         "frac_of_probe_max": round(achieved / max(probe_copy, probe_read), 4),
                         "frac_of_nominal_8000": round(achieved / 8000.0, 4),
                         "algorithmic_bytes_per_step": b_min},
            "trials": trials,
            "e2e": e2e,
            "perf_model": model,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "parity": parity,
            "footprint": footprint,
            "compare": compare or None,
            "dist": dist_info,
            "setup_s": round(t_setup, 2),
        }
        print(json.dumps(out), flush=True)
    if use_dist:
        dist.barrier()
        D.close()
        dist.destroy_process_group()
    return 0


def reference_arm(a, world, npdt):
    """--impl reference: the oracle (plain CRS, OpenMP over all host cores) on the same config,
    metric and unit; each step is one product over the whole matrix, bounded to ~2 minutes."""
    import inputs
    g = inputs.Generator.from_config(a.config)
    rp, col, val = g.crs(dtype=npdt)
    x = inputs.vector(g.n, npdt)
    nnz = int(rp[-1])
    w = max(a.warmup, 3)
    t, reps, cores, tot, _ = time_oracle(g.n, rp, col, val, x, budget_s=120.0, max_reps=a.steps, warmup=w)
    v = 2.0 * nnz / t / 1e9
    sample = f"whole {a.config} matrix ({nnz} nnz) per step, {reps} steps (median), oracle_spmv_crs"
    print(json.dumps({
        "impl": "reference", "metric": METRIC,
        "value": round(v, 3), "unit": "GFlop/s", "n_gpus": world, "steps": reps, "warmup": w,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": a.dtype, "data": "synthetic (inputs/gen.cpp, seed 0x11125588)",
        "config": {"workload": f"{a.config}: {CONFIG_DESC[a.config]}, nnz={nnz}, CPU oracle CRS"},
        "cpu_baseline": {"value": round(v, 3), "unit": "GFlop/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "GFlop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
