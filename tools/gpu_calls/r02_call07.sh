# round 2, call 7: full GPU suite, bench N=1, auto tile order check, dist emulation (rows basis),
# ncu: bench launch list, --set full of the headline kernel, DRAM traffic of every reported kernel
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c07_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c07_gputests.txt
python bench.py > gpurun_out/r02c07_bench.json 2> gpurun_out/r02c07_bench.err
python tools/kbench.py --configs C5,C3,C2,C4 --dtypes f64 --fmts pjds32 --orders 1,2,3 --reps 40 > gpurun_out/r02c07_auto_order.jsonl 2>&1
timeout 900 python tools/dist_emulate2.py --ranks 2,4,8 --modes rows --nl-sigma 1024 > gpurun_out/r02c07_dist_emul2.jsonl 2> gpurun_out/r02c07_dist_emul2.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c07_traffic.csv python tools/traffic_capture.py > gpurun_out/r02c07_traffic_order.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c07_launches.csv python bench.py --steps 5 --warmup 3 --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c07_bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv_kernel -s 3 -c 1 -o gpurun_out/r02c07_full_C5 python bench.py --steps 5 --warmup 3 --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c07_full.log 2>&1
ls -la gpurun_out
