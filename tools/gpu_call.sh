# round 2, call 45: ncu evidence of the final build -- DRAM traffic of every kernel the bench reports,
# the bench launch list, --set full of the headline kernel (lane-interleaved DP, compressed col),
# Lanczos per-step device time
set -x
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c45_traffic.csv python tools/traffic_capture.py > gpurun_out/r02c45_traffic_order.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c45_launches.csv python bench.py --steps 5 --warmup 3 --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c45_bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv_kernel -s 3 -c 1 -o gpurun_out/r02c45_full_C5 python bench.py --steps 5 --warmup 3 --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c45_full.log 2>&1
timeout 900 python tools/lanczos_bench.py C5 50 > gpurun_out/r02c45_lanczos.jsonl 2> gpurun_out/r02c45_lanczos.err; timeout 600 python tools/lanczos_bench.py C3 200 >> gpurun_out/r02c45_lanczos.jsonl 2>> gpurun_out/r02c45_lanczos.err
