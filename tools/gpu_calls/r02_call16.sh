# round 2, call 16: the N>1 bench path at full C5 size, 2 and 4 ranks sharing the one GPU (oversubscribed test mode)
set -x
timeout 1200 python bench.py --gpus 2 --oversubscribe --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/r02c16_bench_r2.json 2> gpurun_out/r02c16_bench_r2.err
timeout 1200 python bench.py --gpus 4 --oversubscribe --steps 20 --warmup 3 --e2e-steps 3 --no-t1 > gpurun_out/r02c16_bench_r4.json 2> gpurun_out/r02c16_bench_r4.err
python bench.py --no-per-config --no-compare --no-cpu-baseline > gpurun_out/r02c16_bench_n1.json 2> /dev/null
