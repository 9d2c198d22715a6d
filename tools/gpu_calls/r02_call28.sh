# round 2, call 28: bench with launch overlap auto (late trigger for one-wave grids); refreshed ncu
# traffic of every reported kernel, launch list and --set full of the headline kernel
set -x
python bench.py > gpurun_out/r02c28_bench.json 2> gpurun_out/r02c28_bench.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c28_traffic.csv python tools/traffic_capture.py > gpurun_out/r02c28_traffic_order.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c28_launches.csv python bench.py --steps 5 --warmup 3 --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c28_bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv_kernel -s 3 -c 1 -o gpurun_out/r02c28_full_C5 python bench.py --steps 5 --warmup 3 --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c28_full.log 2>&1
