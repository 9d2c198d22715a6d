# round 2, call 3: L2 persisting set-aside probe on C5 (time + DRAM bytes per setting), tile keys
set -x
python tools/l2_persist_probe.py --keys none,w4096,w16384 > gpurun_out/r02c03_persist.jsonl 2> gpurun_out/r02c03_persist.err
python tools/l2_persist_probe.py --config C5 --dtype f32 --keys none,w4096 >> gpurun_out/r02c03_persist.jsonl 2>> gpurun_out/r02c03_persist.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pjds_spmv --csv --log-file gpurun_out/r02c03_ncu_persist.csv python tools/l2_persist_probe.py --once --keys none,w4096,w16384 > /dev/null 2>&1
