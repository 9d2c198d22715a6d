python tools/kbench.py --configs C3,C2,C2 --fmts pjds32s,pjds32 --dtypes f64 --variants 0x0,4x2,2x4 --reps 50 > gpurun_out/kbench26.jsonl 2> gpurun_out/kbench26.err
ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,launch__grid_size,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers --clock-control none -k regex:pjds_spmv --csv --log-file gpurun_out/ncu26.csv python tools/kbench.py --once --configs C2 --dtypes f64,f32 --fmts pjds32s > /dev/null 2>&1
tail -2 gpurun_out/kbench26.err
