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
perm every step instead).  At N>1 the NCCL / P2P split runs in the original basis by default (its
halo lists are then contiguous runs of x: no pack kernel), DIRECT in the permuted basis.  Beside the headline the N=1 line carries:
  compare     rows-only pJDS, b_r = 128, ELLPACK-R and cuSPARSE CSR on the same matrix;
  per_config  the SURVEY §8(d) targets table: C2/C3 DP+SP, C4 DP+SP, C5 SP, each pJDS and
              ELLPACK-R timed with L2 carry-over of x defeated (x/y rotated over sets larger than
              L2) and without, O2 parity on sampled rows, footprints from pjds/ellr_footprint;
  parity      sampled rows of the timed product vs the oracle (O1, long double) at the O2 bound,
              plus bitwise equality with the O3 FMA chain (the default kernels' arithmetic);
  e2e         the product through the C ABI with pinned HOST buffers, copies in the timed region.

  python bench.py [--gpus N --steps K --warmup W] [--config C5] [--dtype f64|f32] [--impl pjds|ellr|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU); with fewer than N visible
GPUs it fails loudly unless --oversubscribe is given (test mode: N ranks share the GPUs, gloo
process group, the one-GPU NCCL stand-in of tests/fake_nccl; timings meaningless).  Under torchrun
the world size must equal --gpus.

Prints ONE JSON line on rank 0.  Timing: CUDA events on the launching stream around exactly K
steps, barrier + synchronize on both sides, max over ranks.  The matrix (12.2 GB at C5 DP) is far
larger than L2, so no explicit flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
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
# SURVEY §8(d) targets table: the configurations reported beside the headline at N=1
PER_CONFIG = [("C2", "f64"), ("C2", "f32"), ("C3", "f64"), ("C3", "f32"), ("C4", "f64"), ("C4", "f32"),
              ("C5", "f32")]
L2_BYTES = 126 << 20
FAKE_NCCL = os.path.join(ROOT, "tests", "fake_nccl", "libfakenccl.so")


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="pjds", choices=["pjds", "ellr", "reference"])
    p.add_argument("--config", default="C5", choices=sorted(CONFIG_DESC))
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    p.add_argument("--basis", default="auto", choices=["auto", "permuted", "rows"],
                   help="auto: the permuted basis at N=1 and for the DIRECT transport; the original basis "
                        "(rows permuted, y stored through perm) for the NCCL / P2P split, whose halo lists "
                        "then are contiguous runs of x (no pack)")
    p.add_argument("--block-rows", type=int, default=128,
                   help="pJDS b_r.  The paper pads each block of 'warp size' rows (P:L219-220); the B200 kernel's warp "
                        "owns 32 x R = 128 consecutive sorted rows (R = 4), so the default is 128 (the library's own "
                        "default stays 32; compare reports the other value, timed the same way)")
    p.add_argument("--no-overlap", action="store_true", help="dist: vector mode (exchange, then compute)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-compare", action="store_true", help="N=1: no compare legs; N>1: no p2p/direct legs")
    p.add_argument("--no-per-config", action="store_true", help="N=1: skip the SURVEY §8(d) per-config table")
    p.add_argument("--per-config", default="", help="comma list CFG:dtype overriding the default per-config set")
    p.add_argument("--no-t1", action="store_true", help="N>1: skip the rank-0 single-GPU T1 run (efficiency)")
    p.add_argument("--sample-chunks", type=int, default=100, help="parity: random chunks of --chunk-rows rows")
    p.add_argument("--chunk-rows", type=int, default=1000)
    p.add_argument("--e2e-steps", type=int, default=30)
    p.add_argument("--tile-window", type=int, default=0,
                   help="HMEp configs, N=1: run tiles by (phonon window of this many rows, original row); 0 = off")
    p.add_argument("--probe-bytes", type=int, default=4 << 30)
    p.add_argument("--variant", default="", metavar="R,U",
                   help="kernel variant knob (pjds_set_kernel_variant; default: the library's automatic choice)")
    p.add_argument("--launch-overlap", default="2,2", metavar="MODE,COLS",
                   help="programmatic dependent launch (pjds_set_launch_overlap): 0 off, 1 on, 2 auto (grids of "
                        "more than one wave; the library default), and the jagged columns first-wave warps prefetch")
    p.add_argument("--compression", type=int, default=1, choices=[0, 1],
                   help="pjds_set_compression: column indices in generic compressible memory (1, the library "
                        "default) or plain device memory (0)")
    p.add_argument("--dist", action="store_true", help="use the distributed path even at N=1 (one-rank NCCL group)")
    p.add_argument("--transport", default="auto", choices=["auto", "nccl", "p2p", "direct"],
                   help="dist: NCCL send/recv on a side stream, the fused gather+put P2P kernel, DIRECT "
                        "(no exchange: one kernel whose nonlocal gathers read the owners' x windows), or auto "
                        "(default: each timed for 20 products on this partition, the fastest without a "
                        "timed-out peer wait is the contract transport; the others are reported beside it)")
    p.add_argument("--nccl-env", action="append", default=[], metavar="KEY=VALUE",
                   help="NCCL tuning variable set before the communicator is created and recorded in the line "
                        "(e.g. NCCL_P2P_USE_CUDA_MEMCPY=1, NCCL_MAX_CTAS=4, NCCL_MAX_P2P_NCHANNELS=8); repeatable")
    p.add_argument("--oversubscribe", action="store_true",
                   help="allow more ranks than visible GPUs (test mode: gloo group, one-GPU NCCL stand-in)")
    return p.parse_args(argv)


# ------------------------------------------------------------------------------------------ launch
def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_command(argv, nproc: int, port: int) -> list:
    """The torchrun command that runs this script with one rank per GPU (same arguments)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def check_world(a, env, visible_gpus: int):
    """None if this process may run; else the error message.  Under torchrun WORLD_SIZE must equal
    --gpus; more ranks than visible GPUs needs --oversubscribe."""
    world = int(env.get("WORLD_SIZE", "1"))
    if world != a.gpus and not (a.gpus == 1 and "WORLD_SIZE" not in env):
        return f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world} (launch one rank per GPU)"
    if a.gpus > visible_gpus and not a.oversubscribe:
        return (f"bench.py: --gpus {a.gpus} needs {a.gpus} visible GPUs, found {visible_gpus} "
                f"(--oversubscribe runs the one-GPU test mode)")
    return None


def relaunch(a, argv) -> int:
    """--gpus N > 1 outside torchrun: run N ranks under torch.distributed.run, return its exit code."""
    import torch
    err = check_world(a, {"WORLD_SIZE": str(a.gpus)}, torch.cuda.device_count())
    if err:
        print(err, file=sys.stderr, flush=True)
        return 2
    env = dict(os.environ)
    if a.oversubscribe and a.gpus > torch.cuda.device_count():
        env.setdefault("PJDS_NCCL_LIB", build_fake_nccl())
    return subprocess.run(launch_command(argv, a.gpus, free_port()), env=env).returncode


def build_fake_nccl() -> str:
    """The one-GPU NCCL stand-in (tests/fake_nccl), for --oversubscribe only."""
    src = os.path.join(ROOT, "tests", "fake_nccl", "fake_nccl.cpp")
    if not os.path.exists(FAKE_NCCL) or os.path.getmtime(FAKE_NCCL) < os.path.getmtime(src):
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I/usr/local/cuda/include", "-o", FAKE_NCCL,
                        src, "-L/usr/local/cuda/lib64", "-L/usr/local/cuda/lib64/stubs", "-lcudart", "-lcuda", "-lrt"],
                       check=True)
    return FAKE_NCCL


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
    """DRAM bytes per launch of a kernel from the committed ncu captures (profiles/), newest first."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                v = json.load(f).get(key, {}).get("traffic")
            if v:
                return v, f"profiles/{name}"
        except Exception:
            pass
    return None, None


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


def max_over_ranks(dist, dev, v: float) -> float:
    import torch
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    _allreduce(dist, t, "max")
    return float(t.item())


# ------------------------------------------------------------------------------------------ CPU oracle
def time_oracle(n, rp, col, val, x, budget_s: float, max_reps: int, min_reps: int = 1, threads: int = 0,
                warmup: int = 1):
    """The oracle's plain CRS loop (oracle_spmv_crs: OpenMP static over rows, all visible cores or
    `threads`), repeated until the time budget is spent.  Returns (median s per product, reps, cores,
    total s)."""
    import oracle
    cores = threads or len(os.sched_getaffinity(0))
    for _ in range(max(warmup, 1)):
        oracle.spmv_crs(n, rp, col, val, x, nthreads=cores)
    ts = []
    t_end = time.perf_counter() + budget_s
    while (time.perf_counter() < t_end and len(ts) < max_reps) or len(ts) < min_reps:
        t0 = time.perf_counter()
        oracle.spmv_crs(n, rp, col, val, x, nthreads=cores)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), len(ts), cores, float(sum(ts))


# ------------------------------------------------------------------------------------------ parity
def sample_chunks(n: int, k: int = 100, rows: int = 1000, seed: int = 7, boundaries=()):
    """Sorted disjoint row ranges: k random chunks of `rows` rows, the first and last chunk, and a
    chunk straddling every rank boundary (where the local/nonlocal split changes)."""
    rows = max(1, min(rows, n))
    rng = np.random.default_rng(seed)
    starts = list(rng.integers(0, max(n - rows, 0) + 1, k)) + [0, max(n - rows, 0)]
    for b in boundaries:
        if 0 < b < n:
            starts.append(min(max(b - rows // 2, 0), max(n - rows, 0)))
    iv = sorted((int(s), int(min(s + rows, n))) for s in starts)
    out = []
    for s, e in iv:
        if out and s <= out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], e))
        else:
            out.append((s, e))
    return out


def chunk_rows(chunks) -> np.ndarray:
    return np.concatenate([np.arange(s, e, dtype=np.int64) for s, e in chunks]) if chunks else np.zeros(0, np.int64)


def oracle_rows(g, chunks, x_full, npdt):
    """O1 (long double) and O3 (FMA chain) results of the sampled rows, regenerated from inputs/
    (the oracle's own copy of the rows; nothing comes from the CUDA path)."""
    import oracle
    yl, bd, nz, ch = [], [], [], []
    for s, e in chunks:
        rp, col, val = g.crs(s, e, dtype=npdt)
        y, b = oracle.spmv_ld(e - s, rp, col, val, x_full)
        yl.append(y)
        bd.append(b)
        nz.append(np.diff(rp))
        ch.append(oracle.spmv_chain(e - s, rp, col, val, x_full))
    cat = np.concatenate
    return cat(yl), cat(bd), cat(nz), cat(ch)


def parity_o2(y_rows, ref, npdt, chain_expected: bool):
    """SURVEY §8(c) O2 on the sampled rows: |y_gpu - y_ld| <= 4 nnz_i eps sum_j |a_ij x_j| (the
    north-star bound), and (default single-chain kernels) bitwise equality with the O3 chain."""
    import oracle
    y_ld, bound, nnz, chain = ref
    ok = oracle.acceptance(y_rows, y_ld, bound, nnz, npdt)
    eps = np.finfo(npdt).eps
    err = np.abs(np.asarray(y_rows, np.longdouble) - y_ld)
    scale = np.maximum(nnz.astype(np.longdouble) * eps * bound, np.finfo(np.float64).tiny)
    res = {"rows_checked": int(len(y_rows)), "within_bound": bool(ok.all()), "rows_outside": int((~ok).sum()),
           "max_err_over_nnz_eps_sum_abs": float((err / scale).max()) if len(y_rows) else 0.0,
           "bound": "|y_gpu - y_ld| <= 4 nnz_i eps sum_j |a_ij x_j| (O2 vs the long-double oracle O1)",
           "reference": "oracle.spmv_ld on the sampled rows, regenerated from inputs/"}
    eq = np.asarray(y_rows) == chain
    res["bitwise_o3_chain"] = bool(eq.all())
    res["rows_not_bitwise"] = int((~eq).sum())
    res["bitwise_expected"] = chain_expected
    return res


# ------------------------------------------------------------------------------------------ N = 1
def make_timer(stream):
    import torch

    def timed(fn, k):
        """ms per call of fn(i), i = 0..k-1, CUDA events on the launching stream, synchronised."""
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(k):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k
    return timed


def gflops_entry(nnz, b_min, ms, peak):
    return {"us": round(ms * 1e3, 2), "GFlop/s": round(2.0 * nnz / (ms * 1e-3) / 1e9, 1),
            "frac": round(b_min / (ms * 1e-3) / 1e9 / peak, 4)}


def per_config_leg(cfg, dt, dev, stream, peak, timed, crs_cache, chunks_n=20, reps=None, block_rows=32):
    """One row of the SURVEY §8(d) targets table: pJDS (permuted basis, the library's automatic
    variant and tile order) and ELLPACK-R on the same matrix, each timed (a) with x/y rotated over
    enough copies that L2 cannot carry x from one launch to the next (the table's number) and (b)
    back to back on one x/y pair (L2-warm, reported beside it); O2 parity + O3 bitwise on sampled
    rows; footprints from pjds_footprint / ellr_footprint."""
    import torch
    import inputs
    import paper_1112_5588_b200 as pj
    npdt = np.float64 if dt == "f64" else np.float32
    sv = np.dtype(npdt).itemsize
    tdt = torch.float64 if dt == "f64" else torch.float32
    g = inputs.Generator.from_config(cfg)
    n = g.n
    if cfg in crs_cache:  # SP values are the DP values rounded to nearest (inputs recipe)
        rp, col, v64 = crs_cache[cfg]
        val = v64 if npdt == np.float64 else v64.astype(np.float32)
    else:
        rp, col, val = g.crs(dtype=npdt)
    nnz = int(rp[-1])
    b_min = nnz * (sv + 4) + 2 * n * sv
    x_host = inputs.vector(n, npdt)
    A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=block_rows, symmetric=True)
    E = pj.EllrMatrix.from_crs(n, rp, col, val)
    fa, fe = A.footprint(), E.footprint()
    del rp, col, val
    x0 = torch.from_numpy(x_host).to(dev)
    xp = A.to_permuted(torch.empty_like(x0), x0)
    sets = max(2, int(np.ceil(2 * L2_BYTES / (2 * n * sv))) + 1)
    xs_p = [xp.clone() for _ in range(sets)]
    xs_o = [x0.clone() for _ in range(sets)]
    ys = [torch.empty(n, dtype=tdt, device=dev) for _ in range(sets)]
    k = reps or max(3 * sets, int(np.ceil(20.0 / max(b_min / 6.0e12 * 1e3, 1e-3))))
    out = {"config": cfg, "dtype": dt, "n": n, "nnz": nnz, "algorithmic_bytes": b_min, "block_rows": block_rows,
           "l2": f"x/y rotated over {sets} pairs ({sets * 2 * n * sv / 2**20:.0f} MiB > 2 x L2) between launches"}
    for name, M, xs in (("pjds", A, xs_p), ("ellr", E, xs_o)):
        for i in range(sets):
            M.spmv(ys[i], xs[i], stream=stream)
        cold = timed(lambda i: M.spmv(ys[i % sets], xs[i % sets], stream=stream), k)
        warm = timed(lambda i: M.spmv(ys[0], xs[0], stream=stream), k)
        e = gflops_entry(nnz, b_min, cold, peak)
        w = gflops_entry(nnz, b_min, warm, peak)
        e.update({"us_l2_warm": w["us"], "frac_l2_warm": w["frac"], "launches_timed": k})
        tr, src = committed_traffic(f"{cfg}/{dt}/{'permuted' if name == 'pjds' else 'ellr'}"
                                    + ("/br%d" % block_rows if name == "pjds" and block_rows != 32 else ""))
        e["traffic"] = tr
        e["traffic_over_algorithmic"] = round(tr / b_min, 4) if tr else None
        e["traffic_source"] = src
        # parity of the product just computed (set 0), in the original basis
        M.spmv(ys[0], xs[0], stream=stream)
        yo = A.from_permuted(torch.empty_like(ys[0]), ys[0], stream=stream) if name == "pjds" else ys[0]
        chunks = sample_chunks(n, chunks_n, 1000, seed=11)
        rows = torch.from_numpy(chunk_rows(chunks)).to(dev)
        torch.cuda.synchronize()
        y_rows = yo.index_select(0, rows).cpu().numpy()
        e["parity"] = parity_o2(y_rows, oracle_rows(g, chunks, x_host, npdt), npdt, chain_expected=True)
        e["parity"]["gpu_finite_all_rows"] = bool(torch.isfinite(yo).all().item())
        out[name] = e
    out["footprint"] = {"pjds_bytes": fa["bytes_total"], "ellr_bytes": fe["bytes_total"],
                        "bytes_ratio_pjds_over_ellr": round(fa["bytes_total"] / fe["bytes_total"], 4),
                        "data_reduction_vs_ellpack": round(A.info["data_reduction_vs_ellpack"], 5)}
    # the paper's "performance between 95 % and 130 % of ELLPACK-R"
    out["pjds_perf_over_ellr"] = round(out["ellr"]["us"] / out["pjds"]["us"], 4)
    out["paper_pjds_perf_over_ellr"] = "0.95-1.30 on Fermi C2070 (PAPER.md L19-22, Table 1 L292-295)"
    out["pjds_perf_over_ellr_l2_warm"] = round(out["ellr"]["us_l2_warm"] / out["pjds"]["us_l2_warm"], 4)
    del A, E, xs_p, xs_o, ys, x0, xp
    torch.cuda.synchronize()
    return out


def set_launch_overlap(a):
    import paper_1112_5588_b200 as pj
    m, c = (int(v) for v in a.launch_overlap.split(","))
    if pj.lib().pjds_set_launch_overlap(m, c) != 0:
        raise SystemExit(f"bench.py: bad --launch-overlap {a.launch_overlap}")
    if pj.lib().pjds_set_compression(a.compression) != 0:
        raise SystemExit(f"bench.py: bad --compression {a.compression}")


def launch_overlap_desc(a):
    m, c = (int(v) for v in a.launch_overlap.split(","))
    return {0: "off", 1: f"programmatic dependent launch, early trigger, {c}-column L2 prefetch",
            2: f"auto: programmatic dependent launch, early trigger + {c}-column L2 prefetch on grids of more "
               "than one wave, trigger after the row chains on one-wave grids",
            3: "programmatic dependent launch, trigger after the row chains"}[m]


def run_single(a, npdt, sv, argv_cfg):
    import torch
    import inputs
    import paper_1112_5588_b200 as pj
    from paper_1112_5588_b200 import perfmodel

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    tdt = torch.float64 if npdt == np.float64 else torch.float32
    set_launch_overlap(a)
    if a.variant:
        vr, vu = (int(v) for v in a.variant.split(","))
        if pj.lib().pjds_set_kernel_variant(vr, vu) != 0:
            raise SystemExit(f"bench.py: bad --variant {a.variant}")
    t_setup = time.perf_counter()
    g = inputs.Generator.from_config(a.config)
    n = g.n
    rp, col, val = g.crs(dtype=npdt)
    nnz = int(rp[-1])
    x_host = inputs.vector(n, npdt)
    permuted = a.impl == "pjds" and a.basis in ("permuted", "auto")
    if a.impl == "ellr":
        A = pj.EllrMatrix.from_crs(n, rp, col, val)
    else:
        A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=a.block_rows, symmetric=permuted)
        if a.tile_window:  # opt-in 2-D (phonon window, original row) tile order for HMEp
            r_ = np.arange(n, dtype=np.int64)
            A.set_tile_keys(((r_ % SEGMENT[a.config]) // a.tile_window) * n + r_)
            del r_
    # CPU oracle baseline on the same matrix (rank 0, N=1 only), bounded to ~10 s
    cpu = None
    if not a.no_cpu_baseline:
        t, reps, cores, tot = time_oracle(n, rp, col, val, x_host, budget_s=10.0, max_reps=200)
        cpu = {"value": round(2.0 * nnz / t / 1e9, 3), "unit": "GFlop/s", "cores": cores, "kind": "oracle",
               "sample": f"whole {a.config} matrix ({nnz} nnz), {reps} products, median; {tot:.1f} s of "
                         f"oracle_spmv_crs ({np.dtype(npdt).name}, OpenMP {cores} threads)"}
        t1, reps1, _, _ = time_oracle(n, rp, col, val, x_host, budget_s=3.0, max_reps=3, threads=1)
        cpu["single_thread"] = {"value": round(2.0 * nnz / t1 / 1e9, 3), "reps": reps1}
    x = torch.from_numpy(x_host).to(dev)
    y = torch.empty(n, dtype=tdt, device=dev)
    if permuted:
        xp = torch.empty_like(x)
        A.to_permuted(xp, x)  # once, before the "iterative scheme"
        x = xp
    t_setup = time.perf_counter() - t_setup

    probe_copy, probe_read = pj.bw_probe(a.probe_bytes, 5)
    peak_file = measured_peaks().get("hbm_gbs")
    peak = peak_file if peak_file else max(probe_copy, probe_read)
    stream = torch.cuda.current_stream()
    timed = make_timer(stream)

    def step(_i=0):
        A.spmv(y, x, stream=stream)

    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches0 = pj.launch_count()
    with ClockSampler(0) as clk:
        ms = timed(step, a.steps)
    launches = pj.launch_count() - launches0
    torch.cuda.synchronize()
    # SURVEY §8(d) protocol beside the contract timing: 5 trials of >= 20 ms of back-to-back steps
    kt = max(10, int(np.ceil(20.0 / max(ms, 1e-3))))
    tr = [timed(step, kt) for _ in range(5)]
    trials = {"n": 5, "steps_each": kt, "median_ms": round(float(np.median(tr)), 5), "best_ms": round(min(tr), 5),
              "best_gflops": round(2.0 * nnz / (min(tr) * 1e-3) / 1e9, 2)}
    # same-run parity of the timed product: sampled rows vs O1 at O2, and
    # bitwise vs the O3 chain (every default kernel runs one FMA chain per row in CRS order)
    yo = A.from_permuted(torch.empty_like(y), y) if permuted else y
    chunks = sample_chunks(n, a.sample_chunks, a.chunk_rows)
    rows_t = torch.from_numpy(chunk_rows(chunks)).to(dev)
    torch.cuda.synchronize()
    y_rows = yo.index_select(0, rows_t).cpu().numpy()
    finite_all = bool(torch.isfinite(yo).all().item())
    parity = parity_o2(y_rows, oracle_rows(g, chunks, x_host, npdt), npdt, chain_expected=True)
    parity["gpu_finite_all_rows"] = finite_all
    parity["chunks"] = f"{len(chunks)} row ranges ({a.sample_chunks} random x {a.chunk_rows} rows + first/last)"
    del yo
    t_s = ms * 1e-3
    gflops = 2.0 * nnz / t_s / 1e9
    # algorithmic bytes (Eq. 1 at alpha = 1/N_nzr, write-only y): val+col once, x once, y once
    b_min = nnz * (sv + 4) + 2 * n * sv
    achieved = b_min / t_s / 1e9
    traffic_key = (f"{a.config}/{a.dtype}/{('permuted' if permuted else 'rows') if a.impl == 'pjds' else 'ellr'}"
                   + ("" if a.block_rows == 32 else f"/br{a.block_rows}")
                   + (f"/tw{a.tile_window}" if a.tile_window else ""))
    traffic, traffic_src = committed_traffic(traffic_key)

    # side-by-side kernels on the same matrix: b_r alternative, the other basis, ELLPACK-R, cuSPARSE
    compare = {}
    x0 = torch.from_numpy(x_host).to(dev)
    E = None
    if a.impl == "pjds" and not a.no_compare:
        legs = [("pjds_rows_only" if permuted else "pjds_permuted",
                 lambda: pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=a.block_rows, symmetric=not permuted)),
                ("ellpack_r", lambda: pj.EllrMatrix.from_crs(n, rp, col, val))]
        br_alt = 128 if a.block_rows == 32 else 32
        legs.insert(0, (f"pjds_br{br_alt}", lambda: pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=br_alt,
                                                                           symmetric=permuted)))
        for name, mk in legs:
            B = mk()
            xb = x0
            if name.startswith("pjds") and getattr(B, "symmetric", False):
                xb = B.to_permuted(torch.empty_like(x0), x0)
            # timed exactly like the headline (warm-up, then --steps back-to-back launches, clocks
            # sampled): a short leg right after the host-side build would run at the idle GPU's
            # unthrottled clock and flatter it against the sustained headline
            for _ in range(max(a.warmup, 3)):
                B.spmv(y, xb, stream=stream)
            with ClockSampler(0) as ck:
                mb = timed(lambda i: B.spmv(y, xb, stream=stream), a.steps)
            compare[name] = {"GFlop/s": round(2.0 * nnz / (mb * 1e-3) / 1e9, 1), "ms": round(mb, 4),
                             "frac": round(b_min / (mb * 1e-3) / 1e9 / peak, 4),
                             "bytes": B.footprint()["bytes_total"], "sm_mhz": ck.summary().get("sm_mhz")}
            if name == "ellpack_r":
                E = B.footprint()
            del B, xb
            torch.cuda.synchronize()
        # NVIDIA's library CRS SpMV on the same matrix and device (cuSPARSE via torch.sparse CSR):
        # the vendor baseline beside the pJDS kernel, not part of the product path
        warnings.filterwarnings("ignore", message="Sparse CSR tensor support is in beta")
        warnings.filterwarnings("ignore", message="Sparse invariant checks")
        C = torch.sparse_csr_tensor(torch.from_numpy(rp.astype(np.int32)).to(dev), torch.from_numpy(col).to(dev),
                                    torch.from_numpy(val).to(dev), size=(n, n), check_invariants=False)
        for _ in range(max(a.warmup, 3)):
            torch.mv(C, x0)
        mb = timed(lambda i: torch.mv(C, x0), max(20, a.steps // 2))
        compare["cusparse_csr"] = {"GFlop/s": round(2.0 * nnz / (mb * 1e-3) / 1e9, 1), "ms": round(mb, 4),
                                   "frac": round(b_min / (mb * 1e-3) / 1e9 / peak, 4),
                                   "bytes": int(nnz * (sv + 4) + (n + 1) * 4)}
        del C
        torch.cuda.synchronize()
    footprint = None
    if a.impl == "pjds":
        if E is None:  # host-only ELLPACK-R build: ellr_footprint without a device copy
            Eh = pj.EllrMatrix.from_crs(n, rp, col, val, host_only=True)
            E = Eh.footprint()
            del Eh
        fp = A.footprint()
        footprint = {"pjds_bytes": fp["bytes_total"], "pjds_stored": fp["stored"],
                     "ellr_bytes": E["bytes_total"], "ellr_stored": E["stored"],
                     "data_reduction_vs_ellpack": round(A.info["data_reduction_vs_ellpack"], 5),
                     "padding_entries": fp["stored"] - fp["nnz"],
                     "bytes_ratio_pjds_over_ellr": round(fp["bytes_total"] / E["bytes_total"], 4),
                     "source": "pjds_footprint / ellr_footprint"}
    crs_cache = {a.config: (rp, col, val)} if npdt == np.float64 else {}
    del x0

    # the SURVEY §8(d) targets table (C2/C3 DP+SP, C4, C5 SP), L2 carry-over of x defeated
    per_config = None
    if a.impl == "pjds" and not a.no_per_config:
        per_config = []
        todo = argv_cfg if argv_cfg else PER_CONFIG
        for cfg, dt in todo:
            if cfg == a.config and dt == a.dtype:
                continue
            per_config.append(per_config_leg(cfg, dt, dev, stream, peak, timed, crs_cache, block_rows=a.block_rows))
    del crs_cache, col, val

    # end-to-end through the public API with host buffers in the original basis (H2D x, basis
    # change, kernel, basis change back, D2H y, every step)
    e2e = model = None
    if a.impl == "pjds":
        xh = torch.from_numpy(x_host).pin_memory().numpy()
        yh = torch.empty(n, dtype=tdt).pin_memory().numpy()
        A.spmv_host(yh, xh)
        te = timed(lambda i: A.spmv_host(yh, xh), a.e2e_steps) * 1e-3
        # pipelined (pjds_spmv_host_batch): H2D of step i+1 and D2H of step i-1 overlap product i;
        # every step still moves its own x in and its own y out
        xh2 = torch.from_numpy(inputs.vector(n, npdt, seed=inputs.BASE_SEED + 7)).pin_memory().numpy()
        yh2 = torch.empty(n, dtype=tdt).pin_memory().numpy()
        xs = [xh, xh2] * ((a.e2e_steps + 1) // 2)
        ys = [yh, yh2] * ((a.e2e_steps + 1) // 2)
        A.spmv_host_batch(ys[:2], xs[:2])
        tb = timed(lambda i: A.spmv_host_batch(ys[:a.e2e_steps], xs[:a.e2e_steps]), 1) * 1e-3 / a.e2e_steps
        e2e = {"value": round(2.0 * nnz / tb / 1e9, 2), "unit": "GFlop/s", "h2d_bytes_per_step": n * sv,
               "d2h_bytes_per_step": n * sv, "ms_per_step": round(tb * 1e3, 3),
               "mode": f"pjds_spmv_host_batch of {a.e2e_steps} products, pinned host buffers, original basis",
               "unpipelined": {"value": round(2.0 * nnz / te / 1e9, 2), "ms_per_step": round(te * 1e3, 3),
                               "mode": "pjds_spmv_host per step (H2D, basis change, kernel, basis change, D2H)"}}
        # the bound of the pipelined leg: x in and y out at once on two streams, same pinned buffers
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        dx_, dy_ = torch.empty(n, dtype=tdt, device=dev), torch.empty(n, dtype=tdt, device=dev)
        hx_, hy_ = torch.from_numpy(xh), torch.from_numpy(yh)

        def duplex(_i=0):
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

    wl = f"{a.config}: {CONFIG_DESC[a.config]}, nnz={nnz}, {a.dtype}, {a.impl}"
    if a.impl == "pjds":
        wl += ", permuted basis (PAPER.md L241-246)" if permuted else ", original basis (rows permuted)"
    out = {
        "metric": METRIC,
        "value": round(gflops, 2), "unit": "GFlop/s", "n_gpus": 1, "steps": a.steps,
        "warmup": max(a.warmup, 3), "ms_per_step": round(ms, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": a.dtype,
        "data": "synthetic (inputs/gen.cpp, seed 0x11125588)",
        "config": {"workload": wl, "n": n, "nnz": nnz, "block_rows": a.block_rows, "parallelism": "single GPU",
                   "variant": a.variant or "auto",
                   "launch_overlap": launch_overlap_desc(a),
                   "col_compressible": bool(A.info.get("col_compressible")),
                   "overlap": None, "transport": None, "tile_window": a.tile_window or None,
                   "l2": f"inputs larger than L2: {b_min / 1e9:.2f} GB streamed per step, no flush"},
        "hbm_gbs_effective": round(b_min / t_s / 1e9, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": f"{traffic_src} (ncu, DRAM bytes read + written per launch)" if traffic else None,
                     "traffic_over_algorithmic": round(traffic / b_min, 4) if traffic else None,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if peak_file else "bw probe (this run)",
                     "probe_copy_gbs": round(probe_copy, 1), "probe_read_gbs": round(probe_read, 1),
                     "frac_of_probe_max": round(achieved / max(probe_copy, probe_read), 4),
                     "frac_of_nominal_8000": round(achieved / 8000.0, 4),
                     "algorithmic_bytes_per_step": b_min,
                     "note": ("the column indices live in generic compressible memory (pjds_set_compression): "
                              "B200 compresses them between L2 and HBM, so the DRAM traffic can fall below the "
                              "algorithmic bytes and frac can exceed 1; the format and its bytes are unchanged")
                             if A.info.get("col_compressible") else None},
        "trials": trials,
        "e2e": e2e,
        "perf_model": model,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "parity": parity,
        "footprint": footprint,
        "compare": compare or None,
        "per_config": per_config,
        "dist": None,
        # the paper's own numbers, for context only (other hardware, real matrices)
        "paper_context": {"hardware": "Tesla C2070 (Fermi), ECC on for DP; streaming bandwidth 91 GB/s with ECC "
                                      "(PAPER.md L68-70)",
                          "pjds_dp_gflops": {"HMEp": 7.5, "sAMG": 8.5, "DLR1": 12.9, "DLR2": 9.5},
                          "ellpack_r_dp_gflops": {"HMEp": 7.9, "sAMG": 7.8, "DLR1": 12.9, "DLR2": 9.6},
                          "source": "PAPER.md Table 1 L292-295"},
        "setup_s": round(t_setup, 2),
    }
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ N > 1
def gather_rows(dist, rank, rows_global, y_orig_loc, lo, hi):
    """Every rank's values of the sampled rows it owns -> rank 0 (setup-time plumbing)."""
    mine = rows_global[(rows_global >= lo) & (rows_global < hi)]
    vals = y_orig_loc[mine - lo] if len(mine) else y_orig_loc[:0]
    objs = [None] * dist.get_world_size()
    dist.all_gather_object(objs, (mine, vals))  # small (~100 K values in total); works on gloo and NCCL
    if rank != 0:
        return None
    idx = np.concatenate([o[0] for o in objs])
    v = np.concatenate([o[1] for o in objs])
    out = np.full(len(rows_global), np.nan, dtype=v.dtype)
    out[np.searchsorted(rows_global, idx)] = v
    return out


def run_dist(a, world, rank, local_rank, npdt, sv):
    """N > 1 (or --dist): row-partitioned product, one rank per GPU."""
    import torch
    import torch.distributed as dist
    import inputs
    import paper_1112_5588_b200 as pj

    nccl_env = {}
    for kv in a.nccl_env:  # must precede the first communicator (torch's and the library's)
        k, _, v = kv.partition("=")
        if not k.startswith("NCCL_") or not v:
            raise SystemExit(f"bench.py: --nccl-env needs NCCL_*=value, got {kv!r}")
        os.environ[k] = v
        nccl_env[k] = v
    ngpu = torch.cuda.device_count()
    oversub = world > ngpu
    dev_index = local_rank % max(ngpu, 1)  # more ranks than GPUs only in --oversubscribe test mode
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    tdt = torch.float64 if npdt == np.float64 else torch.float32
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    if oversub:  # NCCL refuses duplicate GPUs: gloo group + the one-GPU NCCL stand-in
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)

    t_setup = time.perf_counter()
    g = inputs.Generator.from_config(a.config)
    n = g.n
    seg = SEGMENT.get(a.config, 32)
    nb = n // seg
    offs = np.array([(nb * r // world) * seg for r in range(world + 1)], np.int64)
    offs[-1] = n
    lo, hi = int(offs[rank]), int(offs[rank + 1])
    rp, col, val = g.crs(lo, hi, dtype=npdt)
    nnz_loc = int(rp[-1])
    x_host = inputs.vector(hi - lo, npdt, i0=lo)
    def basis_of(transport):
        return a.basis == "permuted" or (a.basis == "auto" and transport == "direct")

    def build(transport):
        D = pj.DistPjds.create(n, offs, rp, col, val, block_rows=a.block_rows, permuted=basis_of(transport),
                               transport=transport)
        xd = torch.from_numpy(x_host).to(dev)
        if basis_of(transport):
            xd = D.to_permuted(torch.empty_like(xd), xd)
        if transport == "direct":  # x lives in the exported window: no per-call copy
            w = D.x_window()
            w.copy_(xd)
            xd = w
        return D, xd

    t_start = time.perf_counter()

    def progress(msg):  # stderr trace of the N > 1 phases (the JSON line stays alone on stdout)
        print(f"bench.py[rank {rank}/{world}] {time.perf_counter() - t_start:8.1f}s {msg}", file=sys.stderr, flush=True)

    def timed_out(Dh):
        t = torch.tensor([int(Dh.p2p_timed_out())], dtype=torch.int64, device=dev)
        _allreduce(dist, t, "sum")
        return int(t.item()) > 0

    set_launch_overlap(a)
    stream = torch.cuda.current_stream()
    timed = make_timer(stream)
    selection = None
    built = {}  # transport -> (handle, x) created once per run (communicators are not re-created)
    if a.transport == "auto":
        # the library's three transports on this partition, 20 products each (max over ranks); the
        # fastest one without a timed-out peer wait becomes the contract transport, the others are
        # reported beside it (dist.transports) -- on NVSwitch the fused remote-gather kernel (DIRECT)
        # is expected to win at large R, NCCL where remote loads cost more than the exchange
        selection, best = {}, None
        for trn in ("nccl", "p2p", "direct"):
            dist.barrier()
            progress(f"transport selection: {trn}")
            try:
                Ds, xs = build(trn)
                ys = torch.empty(hi - lo, dtype=tdt, device=dev)
                for _ in range(3):
                    Ds.spmv(ys, xs, stream=stream)
                torch.cuda.synchronize()
                dist.barrier()
                m = max_over_ranks(dist, dev, timed(lambda i: Ds.spmv(ys, xs, stream=stream), 20))
                to = timed_out(Ds)
                selection[trn] = {"ms": round(m, 5), "peer_wait_timed_out": to}
                if not to and (best is None or m < best[1]):
                    best = (trn, m)
                built[trn] = (Ds, xs)  # kept: the contract transport and the legs reuse them
                del ys
            except Exception as e:  # a transport that cannot run here is reported, not chosen
                selection[trn] = {"error": str(e)[:300]}
            torch.cuda.synchronize()
        a.transport = best[0] if best else "nccl"
        progress(f"transport selection: {selection} -> {a.transport}")
    permuted = basis_of(a.transport)
    D, x = built.pop(a.transport) if a.transport in built else build(a.transport)
    tt = torch.tensor([nnz_loc], dtype=torch.int64, device=dev)
    _allreduce(dist, tt, "sum")
    nnz = int(tt.item())
    y = torch.empty(hi - lo, dtype=tdt, device=dev)
    t_setup = time.perf_counter() - t_setup
    probe_copy, probe_read = pj.bw_probe(a.probe_bytes, 5)
    peak_file = measured_peaks().get("hbm_gbs")
    peak = peak_file if peak_file else max(probe_copy, probe_read)

    def step(_i=0):
        D.spmv(y, x, stream=stream, no_overlap=a.no_overlap)

    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = pj.launch_count()
    with ClockSampler(dev_index) as clk:
        ms = timed(step, a.steps)
    launches = pj.launch_count() - launches0
    dist.barrier()
    torch.cuda.synchronize()
    ms = max_over_ranks(dist, dev, ms)
    progress(f"timed {a.steps} steps of {a.transport}: {ms:.4f} ms")
    lt = torch.tensor([launches], dtype=torch.int64, device=dev)
    _allreduce(dist, lt, "sum")
    launches = int(lt.item())
    kt = max(10, int(np.ceil(20.0 / max(ms, 1e-3))))
    tr = []
    for _ in range(5):
        dist.barrier()
        tr.append(max_over_ranks(dist, dev, timed(step, kt)))
    trials = {"n": 5, "steps_each": kt, "median_ms": round(float(np.median(tr)), 5), "best_ms": round(min(tr), 5),
              "best_gflops": round(2.0 * nnz / (min(tr) * 1e-3) / 1e9, 2)}

    chunks = sample_chunks(n, a.sample_chunks, a.chunk_rows, boundaries=offs[1:-1].tolist())
    rows_g = chunk_rows(chunks)
    ref = None
    x_full = None
    if rank == 0:  # the oracle's rows, regenerated from inputs/ (rank 0 only)
        x_full = inputs.vector(n, npdt)
        ref = oracle_rows(g, chunks, x_full, npdt)

    def parity_of(Dh, yv, chain_expected, perm_basis):
        yo = Dh.from_permuted(torch.empty_like(yv), yv, stream=stream) if perm_basis else yv
        torch.cuda.synchronize()
        finite = torch.tensor([int(bool(torch.isfinite(yo).all().item()))], dtype=torch.int64, device=dev)
        _allreduce(dist, finite, "sum")
        vals = gather_rows(dist, rank, rows_g, yo.cpu().numpy(), lo, hi)
        if rank != 0:
            return None
        p = parity_o2(vals, ref, npdt, chain_expected=chain_expected)
        p["gpu_finite_all_rows"] = int(finite.item()) == world
        p["chunks"] = f"{len(chunks)} row ranges incl. every rank boundary"
        return p

    progress("trials done; parity")
    to_main = timed_out(D)
    # NCCL / P2P split the row into local + nonlocal chains (combined by one add, DESIGN reading 25):
    # not the unsplit O3 chain; DIRECT runs every row's whole chain in one kernel (bitwise expected)
    parity = parity_of(D, y, chain_expected=a.transport == "direct", perm_basis=permuted)
    if parity is not None:
        parity["peer_wait_timed_out"] = to_main
        if to_main:
            parity["within_bound"] = False

    # vector mode (exchange, then compute) as the reference point for "communication hidden",
    # and one traced call of each mode: per-phase device times, max over ranks
    dist.barrier()
    ms_no = max_over_ranks(dist, dev, timed(lambda i: D.spmv(y, x, stream=stream, no_overlap=True),
                                            max(5, a.steps // 4)))
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
    gain = ms_no / ms
    dist_info = {"transport": a.transport, "transport_selection": selection, "ms_vector_mode": round(ms_no, 4), "speedup_task_over_vector": round(gain, 3),
                 # overlapping communication with computation gains at most 2x;
                 # not meaningful when ranks share a GPU (test mode: the stand-in NCCL serialises)
                 "m6_task_gain_le_2": None if oversub else bool(gain <= 2.0 + 1e-9),
                 "phases_ms_max_over_ranks": phases,
                 "hidden_fraction": round(1.0 - max(0.0, tp["total"] - tp["local"] - tp["nonlocal"] - tp["pack"]) / comm, 3),
                 "halo_entries_rank0": D.info["halo"], "nnz_nonlocal_rank0": D.info["nnz_nonlocal_part"],
                 "messages_rank0": D.info["send_messages"], "row_offsets": offs.tolist(),
                 "oversubscribed": oversub, "nccl_env": nccl_env or None,
                 "basis": "permuted" if permuted else "rows"}

    progress("vector mode and phases done")
    # T1: the single-GPU product on the full matrix (rank 0's GPU; the others wait), so that the
    # line carries T1 / (R t_R) beside the driver's own cross-N efficiency
    t1_ms = None
    if not a.no_t1 and world > 1:
        if rank == 0:
            rp1, col1, val1 = g.crs(dtype=npdt)
            # the N=1 bench's configuration (permuted basis unless --basis rows): the same T_1 the
            # driver divides by when it computes efficiency from the per-N lines
            p1 = a.basis != "rows"
            A1 = pj.PjdsMatrix.from_crs(n, rp1, col1, val1, block_rows=a.block_rows, symmetric=p1)
            del rp1, col1, val1
            x1 = torch.from_numpy(x_full).to(dev)
            if p1:
                x1 = A1.to_permuted(torch.empty_like(x1), x1)
            y1 = torch.empty(n, dtype=tdt, device=dev)
            for _ in range(5):
                A1.spmv(y1, x1, stream=stream)
            t1_ms = timed(lambda i: A1.spmv(y1, x1, stream=stream), 20)
            del A1, x1, y1
            torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            dist_info["t1_ms"] = round(t1_ms, 5)
            dist_info["parallel_efficiency_vs_t1"] = round(t1_ms / (world * ms), 4)

    # per rank: pinned host x_loc -> device, basis change, dist product, basis change back,
    # device -> pinned host y_loc, every step; max over ranks
    xh = torch.from_numpy(x_host).pin_memory()
    yh = torch.empty(hi - lo, dtype=tdt).pin_memory()
    xd, yd = torch.empty(hi - lo, dtype=tdt, device=dev), torch.empty_like(y)
    xw, yw = torch.empty_like(xd), torch.empty_like(y)
    xdst = D.x_window() if a.transport == "direct" else xw

    def e2e_step(_i=0):
        xd.copy_(xh, non_blocking=True)
        if permuted:
            D.to_permuted(xdst, xd, stream=stream)
            D.spmv(yw, xdst, stream=stream, no_overlap=a.no_overlap)
            D.from_permuted(yd, yw, stream=stream)
        else:
            if a.transport == "direct":
                xdst.copy_(xd)
            D.spmv(yd, xdst if a.transport == "direct" else xd, stream=stream, no_overlap=a.no_overlap)
        yh.copy_(yd, non_blocking=True)

    progress("T1 done; e2e")
    e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    te = max_over_ranks(dist, dev, timed(e2e_step, a.e2e_steps) * 1e-3)
    e2e = {"value": round(2.0 * nnz / te / 1e9, 2), "unit": "GFlop/s", "h2d_bytes_per_step": n * sv,
           "d2h_bytes_per_step": n * sv, "ms_per_step": round(te * 1e3, 3),
           "note": "all ranks' pinned host buffers; max over ranks"}

    # the other transports on the same partition, behind their bounded waits (compare legs); run
    # last, after every number of the contract transport is taken, so that a transport that
    # cannot run on this box costs only its own entry
    legs = {}
    if not a.no_compare and world > 1:
        for trn in ("nccl", "p2p", "direct"):
            if trn == a.transport:
                continue
            dist.barrier()
            progress(f"compare leg: {trn}")
            try:
                D2, x2 = built.pop(trn) if trn in built else build(trn)
                y2 = torch.empty_like(y)
                for _ in range(3):
                    D2.spmv(y2, x2, stream=stream)
                torch.cuda.synchronize()
                dist.barrier()
                m2 = max_over_ranks(dist, dev, timed(lambda i: D2.spmv(y2, x2, stream=stream), max(10, a.steps // 2)))
                to2 = timed_out(D2)
                p2 = parity_of(D2, y2, chain_expected=trn == "direct", perm_basis=basis_of(trn))
                leg = {"ms": round(m2, 5), "GFlop/s": round(2.0 * nnz / (m2 * 1e-3) / 1e9, 1),
                       "peer_wait_timed_out": to2, "basis": "permuted" if basis_of(trn) else "rows"}
                if p2 is not None:
                    leg["parity_within_bound"] = p2["within_bound"] and not to2
                    leg["parity_bitwise_o3_chain"] = p2["bitwise_o3_chain"]
                legs[trn] = leg
                D2.close()
                del D2, x2, y2
            except Exception as e:  # a transport that cannot run here is reported, not fatal
                legs[trn] = {"error": str(e)[:300]}
            torch.cuda.synchronize()
        dist_info["transports"] = legs
    for Dk, _ in built.values():  # selection handles no leg used (--no-compare)
        Dk.close()
    built.clear()

    t_s = ms * 1e-3
    b_min = nnz * (sv + 4) + 2 * n * sv
    achieved = b_min / t_s / 1e9 / world  # per GPU
    if rank == 0:
        wl = (f"{a.config}: {CONFIG_DESC[a.config]}, nnz={nnz}, {a.dtype}, pjds, "
              + ("local permuted basis (PAPER.md L241-246)" if permuted else "original basis"))
        out = {
            "metric": METRIC,
            "value": round(2.0 * nnz / t_s / 1e9, 2), "unit": "GFlop/s", "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": a.dtype,
            "data": "synthetic (inputs/gen.cpp, seed 0x11125588)",
            "config": {"workload": wl, "n": n, "nnz": nnz, "block_rows": a.block_rows,
                       "parallelism": f"row-partition r{world}", "overlap": not a.no_overlap,
                       "transport": a.transport, "tile_window": None, "launch_overlap": launch_overlap_desc(a),
                       "l2": f"inputs larger than L2: {b_min / 1e9 / world:.2f} GB streamed per GPU per step, no flush"},
            "hbm_gbs_effective": round(b_min / t_s / 1e9, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": None,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if peak_file else "bw probe (this run)",
                         "probe_copy_gbs": round(probe_copy, 1), "probe_read_gbs": round(probe_read, 1),
                         "algorithmic_bytes_per_step": b_min, "note": "achieved = algorithmic bytes / t / N (per GPU)"},
            "trials": trials,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": None,
            "parity": parity,
            "dist": dist_info,
            "setup_s": round(t_setup, 2),
        }
        print(json.dumps(out), flush=True)
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
    t, reps, cores, tot = time_oracle(g.n, rp, col, val, x, budget_s=120.0, max_reps=a.steps, warmup=w)
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


# ------------------------------------------------------------------------------------------ main
def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    a = parse(argv)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    npdt = np.float64 if a.dtype == "f64" else np.float32
    sv = np.dtype(npdt).itemsize
    if a.impl == "reference":  # rank 0 alone runs and prints; the other ranks exit without work
        return reference_arm(a, world, npdt) if rank == 0 else 0
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(a, argv)
    import torch
    err = check_world(a, os.environ, torch.cuda.device_count())
    if err:
        print(err, file=sys.stderr, flush=True)
        return 2
    if world > torch.cuda.device_count() and "PJDS_NCCL_LIB" not in os.environ:
        os.environ["PJDS_NCCL_LIB"] = build_fake_nccl()
    per_cfg = [tuple(s.split(":")) for s in a.per_config.split(",") if s] if a.per_config else None
    if world > 1 or a.dist:
        if a.impl != "pjds":
            print("bench.py: the distributed path is pJDS only", file=sys.stderr, flush=True)
            return 2
        local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        return run_dist(a, world, rank, local_rank, npdt, sv)
    return run_single(a, npdt, sv, per_cfg)


if __name__ == "__main__":
    sys.exit(main())
