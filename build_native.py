"""Build every native artefact in-tree (no JIT cache; the .so files travel with gpurun).

  inputs/libpjdsgen.so                    g++  -O3 -fopenmp         (seeded generators)
  oracle/liboracle.so                     gcc  -O2 -fopenmp         (CPU oracle; test infra only)
  paper_1112_5588_b200/libpjds.so         nvcc -gencode arch=compute_100a,code=sm_100a (the product)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_include() -> str:
    import site
    for d in site.getsitepackages():
        p = os.path.join(d, "nvidia", "nccl", "include")
        if os.path.isdir(p):
            return p
    raise RuntimeError("NCCL headers (nvidia/nccl/include) not found")


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)


def build_inputs(force: bool = False) -> str:
    src = os.path.join(ROOT, "inputs", "gen.cpp")
    out = os.path.join(ROOT, "inputs", "libpjdsgen.so")
    if force or _stale(out, [src]):
        _run(["g++", "-O3", "-std=c++17", "-fopenmp", "-shared", "-fPIC", "-o", out, src])
    return out


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "oracle.c")
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, [src]):
        # -ffp-contract=off: no compiler-introduced FMAs; the oracle's arithmetic is exactly as written.
        _run(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC", "-o", out, src, "-lm"])
    return out


def build_pjds(force: bool = False) -> str:
    csrc = os.path.join(ROOT, "paper_1112_5588_b200", "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cpp")))
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))
    out = os.path.join(ROOT, "paper_1112_5588_b200", "libpjds.so")
    if not (force or _stale(out, srcs + hdrs)):
        return out
    extra = os.environ.get("PJDS_NVCC_DEFINES", "").split()  # dev experiments (e.g. -DPJDS_CTA_THREADS=128)
    cmd = [NVCC, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-fopenmp,-O3"] + extra + [
           "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xptxas", "-v",
           "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(),
           "-o", out] + srcs + ["-lgomp", "-ldl", "-lcudart"]
    _run(cmd)
    return out


def build_all(force: bool = False) -> None:
    build_inputs(force)
    build_oracle(force)
    build_pjds(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
