# round 2, call 35: bench --transport auto reusing the selection handles (no communicator re-creation)
set -x
timeout 1200 python -m pytest tests/test_gpu_bench_dist.py -x -q > gpurun_out/r02c35_bench_dist.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c35_bench_dist.txt
timeout 900 python bench.py --gpus 4 --oversubscribe --config C5 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/r02c35_bench_c5_r4_auto.json 2> gpurun_out/r02c35_bench_c5_r4_auto.err; echo "rc=$?" >> gpurun_out/r02c35_bench_c5_r4_auto.err
