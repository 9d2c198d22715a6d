# round 2, call 8: full GPU suite, rows-only probe with clocks, sanitizer on the new kernels' paths
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c08_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c08_gputests.txt
python tools/rows_only_probe.py > gpurun_out/r02c08_rows_probe.jsonl 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest "tests/test_gpu_parity.py::test_warp_tile_order_variants_bitwise" "tests/test_gpu_dist_world1.py" -x -q > gpurun_out/r02c08_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c08_memcheck.txt
