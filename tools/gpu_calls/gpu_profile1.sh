set -x
python tools/kbench.py > gpurun_out/kbench1.jsonl 2> gpurun_out/kbench1.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none -k regex:spmv --csv --log-file gpurun_out/ncu_metrics1.csv python tools/kbench.py --once --configs C2,C3,C4,C5 --dtypes f64,f32 --fmts pjds32,pjds64,ellr > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -c 1 -o gpurun_out/prof_c3_pjds32 python tools/kbench.py --once --configs C3 --dtypes f64 --fmts pjds32 > /dev/null 2>&1
ls -la gpurun_out
