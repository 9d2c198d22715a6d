# round 2, call 17: sanitizers on the round-2 code paths (warp tile order, accumulate, A_nl windows,
# one-call create through the NCCL stand-in, bench N>1 test mode)
set -x
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest "tests/test_gpu_parity.py::test_warp_tile_order_variants_bitwise" "tests/test_gpu_parity.py::test_schedule_bitwise" -x -q > gpurun_out/r02c17_racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c17_racecheck.txt
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest "tests/test_gpu_parity.py::test_schedule_bitwise" tests/test_gpu_dist_world1.py -x -q > gpurun_out/r02c17_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c17_memcheck.txt
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest "tests/test_gpu_parity.py::test_warp_tile_order_variants_bitwise" -x -q > gpurun_out/r02c17_synccheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c17_synccheck.txt
