# round 2, call 60: final-tree validation (row-only interleaving limited to x <= 64 MB) -- smoke,
# full GPU suite, default bench, refreshed ncu traffic of every reported kernel
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c60_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c60_smoke.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02c60_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c60_gputests.txt
python bench.py > gpurun_out/r02c60_bench.json 2> gpurun_out/r02c60_bench.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c60_traffic.csv python tools/traffic_capture.py > gpurun_out/r02c60_traffic_order.txt 2>&1
