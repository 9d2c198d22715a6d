# round 2, call 40: col + perm + rowmax in compressible memory -- full GPU suite, bench, refreshed
# ncu traffic of every reported kernel, compression off/on kernel sweep incl. the row-only basis
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c40_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c40_gputests.txt
python bench.py > gpurun_out/r02c40_bench.json 2> gpurun_out/r02c40_bench.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c40_traffic.csv python tools/traffic_capture.py > gpurun_out/r02c40_traffic_order.txt 2>&1
for C in 0 1 0 1; do
  timeout 900 python tools/kbench.py --configs C5,C3 --dtypes f64,f32 --fmts pjds128,pjds128s,ellr --reps 40 --rotate 2 --compress $C >> gpurun_out/r02c40_kbench.jsonl 2>> gpurun_out/r02c40_kbench.err
done
