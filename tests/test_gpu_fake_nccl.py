"""The NCCL transport of pjds_dist_spmv (libpjds dist.cpp: grouped ncclSend/ncclRecv on the comm
stream, direct-run or packed messages, task and vector modes, both bases) run by 2-4 processes that
share the one GPU of this run.  Real NCCL refuses duplicate GPUs, so PJDS_NCCL_LIB points libpjds at
tests/fake_nccl (CUDA-IPC copies behind the same six NCCL entry points); everything else is the
product path.  Results are checked against the oracle split emulator (bitwise) and the O2 bound."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.join(ROOT, "tests", "fake_nccl")


def build_fake():
    out = os.path.join(HERE, "libfakenccl.so")
    src = os.path.join(HERE, "fake_nccl.cpp")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I/usr/local/cuda/include", "-o", out, src,
                        "-L/usr/local/cuda/lib64", "-L/usr/local/cuda/lib64/stubs", "-lcudart", "-lcuda", "-lrt"],
                       check=True)
    return out


def run_workers(case, R, transport, reps, port, dtype="f64"):
    env = dict(os.environ, OMP_NUM_THREADS="1")
    if transport == "nccl":
        env["PJDS_NCCL_LIB"] = build_fake()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={R}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(HERE, "worker.py"), case, transport,
           str(reps), dtype]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and len(lines) == R, p.stdout[-2000:] + p.stderr[-3000:]
    for rec in lines:
        assert "create_error" not in rec, rec
        for mode in ("perm0_noov0", "perm0_noov1", "perm1_noov0", "perm1_noov1"):
            assert rec[mode]["o2"], (rec["rank"], mode)
            assert rec[mode]["bitwise_vs_split_oracle"], (rec["rank"], mode)
            assert not rec[mode]["timed_out"], (rec["rank"], mode)


@pytest.mark.parametrize("case,R", [("C1", 2), ("rand", 3), ("C1", 4)])
def test_p2p_transport_multiprocess_one_gpu(case, R):
    """PJDS_TRANSPORT_P2P (fused gather+put into IPC-mapped peer halos, flag ordering), several calls
    per mode so both halo buffers and the done/ready sequence are exercised."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    run_workers(case, R, "p2p", 5, 29740 + R + (10 if case == "rand" else 0))


@pytest.mark.parametrize("case,R,dtype", [("C1", 2, "f64"), ("rand", 3, "f64"), ("C1", 4, "f64"), ("rand", 8, "f64"),
                                          ("rand_empty", 3, "f64"), ("C1", 2, "f32"), ("rand", 4, "f32")])
def test_direct_transport_multiprocess_one_gpu(case, R, dtype):
    """PJDS_TRANSPORT_DIRECT (one kernel per call; nonlocal gathers read the owners' IPC-mapped x
    windows; ready/done flags): bitwise equal to the oracle's unsplit FMA chain, both bases, x
    passed separately (copied into the window) and computed in the window, several calls."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    run_workers(case, R, "direct", 5, 29780 + R + {"C1": 0, "rand": 10, "rand_empty": 20}[case] + (30 if dtype == "f32" else 0),
                dtype)


@pytest.mark.parametrize("case,R", [("C1", 2), ("rand", 3), ("C1", 4)])
def test_nccl_transport_multiprocess_one_gpu(case, R):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    lib = build_fake()
    env = dict(os.environ, PJDS_NCCL_LIB=lib, OMP_NUM_THREADS="1")
    port = 29700 + R + (10 if case == "rand" else 0)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={R}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(HERE, "worker.py"), case]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and len(lines) == R, p.stdout[-2000:] + p.stderr[-3000:]
    for rec in lines:
        assert "create_error" not in rec, rec
        for mode in ("perm0_noov0", "perm0_noov1", "perm1_noov0", "perm1_noov1"):
            assert rec[mode]["o2"], (rec["rank"], mode)
            assert rec[mode]["bitwise_vs_split_oracle"], (rec["rank"], mode)


def test_direct_c5_sampled():
    """DIRECT on the bench matrix (C5, 942 M nonzeros) with 2 processes on the one GPU: sampled rows
    bitwise = the oracle's unsplit FMA chain and within O2, every row finite, no flag timeout."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    env = dict(os.environ, OMP_NUM_THREADS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port=29841", os.path.join(HERE, "worker_c5.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and len(lines) == 2, p.stdout[-2000:] + p.stderr[-3000:]
    for rec in lines:
        assert rec["bitwise"] and rec["o2"] and rec["finite"] and not rec["timed_out"], rec
        assert rec["halo"] > 0
