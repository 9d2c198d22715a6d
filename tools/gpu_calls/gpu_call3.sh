python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/kbench.py --fmts pjds32,pjds32s,pjds128,ellr --variants 1x8,2x4,2x8,4x2,4x4 > gpurun_out/kbench2.jsonl 2> gpurun_out/kbench2.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none -k regex:spmv --csv --log-file gpurun_out/ncu_metrics2.csv python tools/kbench.py --once --configs C3,C5 --dtypes f64 --fmts pjds32,pjds32s,ellr --variants 2x4,4x2 > /dev/null 2>&1
tail -3 gpurun_out/kbench2.err
