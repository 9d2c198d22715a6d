# round 2, call 59: ncu DRAM traffic of every kernel the bench line reports, final build
set -x
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c59_traffic.csv python tools/traffic_capture.py > gpurun_out/r02c59_traffic_order.txt 2>&1
