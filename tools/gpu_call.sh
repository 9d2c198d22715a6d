# round 2, call 39: compressible column indices by default -- full GPU suite, bench, refreshed ncu
# traffic of every reported kernel, launch list and --set full of the headline kernel
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c39_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c39_gputests.txt
python bench.py > gpurun_out/r02c39_bench.json 2> gpurun_out/r02c39_bench.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c39_traffic.csv python tools/traffic_capture.py > gpurun_out/r02c39_traffic_order.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c39_launches.csv python bench.py --steps 5 --warmup 3 --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c39_bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv_kernel -s 3 -c 1 -o gpurun_out/r02c39_full_C5 python bench.py --steps 5 --warmup 3 --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c39_full.log 2>&1
