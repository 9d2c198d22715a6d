python -m pytest tests -m gpu -x -q -k "tile_order or variants" 2>&1 | tail -2
python tools/kbench.py --configs C5,C3,C2,C4 --fmts pjds32s,pjds32 --dtypes f64,f32 --orders 0,1 > gpurun_out/kbench8.jsonl 2> gpurun_out/kbench8.err; tail -2 gpurun_out/kbench8.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct
ncu --metrics $M --clock-control none -k regex:pjds_spmv --csv --log-file gpurun_out/ncu_metrics8.csv python tools/kbench.py --once --configs C5 --dtypes f64 --fmts pjds32s,pjds32 --orders 0,1 > /dev/null 2>&1
