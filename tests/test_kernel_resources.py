"""Static checks of the built sm_100a kernels (no GPU): register budgets that keep the bandwidth-bound
pJDS kernels at their measured occupancy, no local-memory spills, and SASS evidence of the 256-bit
evict-first loads.  (A launch-bounds change once let ptxas take 84 registers for the R=4 DP kernel
and halved occupancy: C2 DP 58 -> 147 us; this test pins the budget.)"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1112_5588_b200", "libpjds.so")


@pytest.fixture(scope="module")
def usage():
    import build_native
    build_native.build_pjds()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-res-usage", LIB], capture_output=True, text=True,
                         check=True).stdout
    res = {}
    lines = out.splitlines()
    for i, l in enumerate(lines):
        m = re.search(r"Function (\S+):", l)
        if m and i + 1 < len(lines):
            r = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", lines[i + 1])
            if r:
                res[m.group(1)] = tuple(int(v) for v in r.groups())
    return res


def pick(usage, pattern):
    hits = {k: v for k, v in usage.items() if re.search(pattern, k)}
    assert hits, pattern
    return hits


def test_default_pjds_kernels_register_budget(usage):
    # pjds_spmv_kernel<T, int, R, U, MODE, PIPE=false> for the auto variants (4,2), (2,4), (1,8)
    for T in ("d", "f"):
        for R, U in ((4, 2), (2, 4), (1, 8)):
            for name, (reg, stack, smem, local) in pick(usage, rf"pjds_spmv_kernelI{T}iLi{R}ELi{U}ELi\dELb0E").items():
                assert reg <= 64, (name, reg)
                assert local == 0, (name, local)


def test_no_spills_in_any_default_kernel(usage):
    for name, (reg, stack, smem, local) in usage.items():
        if "ELb1E" in name:  # pipelined / lane-interleaved variants may use a small stack frame
            continue
        if re.search(r"LiELi8E|Li2ELi8E|Li4ELi4E", name):  # large-unroll variants (tuning knob only)
            continue
        assert local == 0, name


def test_sass_has_256bit_evict_first_loads(usage):
    """The R=4 DP permuted-basis kernel streams val with 256-bit L1-no-allocate / L2-evict-first loads."""
    name = next(k for k in usage if re.search(r"pjds_spmv_kernelIdiLi4ELi2ELi1ELb0ELb0E", k))
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun", name, LIB], capture_output=True,
                         text=True).stdout
    assert re.search(r"LDG\.E(\.NA)?\.EFL2\.256", out), "no 256-bit evict-first LDG in the pJDS kernel"
    assert re.search(r"LDG\.E\.NA\.", out), "no L1::no_allocate streaming loads"


def test_split_kernels_do_not_spill(usage):
    """The long-row split-j kernels (__launch_bounds__(256, 4)): ptxas once capped them at 32
    registers with local-memory spills."""
    for name, (reg, stack, smem, local) in pick(usage, r"pjds_spmv_split_kernel").items():
        assert stack == 0 and local == 0, name
