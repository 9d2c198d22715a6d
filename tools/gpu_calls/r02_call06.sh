# round 2, call 6: dist/tile-order GPU tests, A_nl sort scope in the full-contention emulation,
# warp-granular tile order sweep, rows-only timing probe
set -x
python -m pytest tests/test_gpu_dist_world1.py tests/test_gpu_fake_nccl.py tests/test_gpu_bench_dist.py tests/test_lanczos.py "tests/test_gpu_parity.py::test_tile_order_bitwise" "tests/test_gpu_parity.py::test_warp_tile_order_variants_bitwise" -x -q > gpurun_out/r02c06_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c06_tests.txt
python tools/rows_only_probe.py > gpurun_out/r02c06_rows_probe.jsonl 2>&1
python tools/kbench.py --configs C5,C3,C2,C4 --dtypes f64,f32 --fmts pjds32s,pjds32 --orders 2,3 --reps 40 > gpurun_out/r02c06_order3.jsonl 2> gpurun_out/r02c06_order3.err
timeout 1200 python tools/dist_emulate2.py --ranks 2,4,8 --modes rows,permuted --nl-sigma 0,1024 > gpurun_out/r02c06_dist_emul2.jsonl 2> gpurun_out/r02c06_dist_emul2.err
