python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/kbench.py --configs C3,C5,C2 --fmts pjds32s,pjds32 --dtypes f64 --sigmas 0,16384,262144,4194304 --reps 30 > gpurun_out/kbench28.jsonl 2> gpurun_out/kbench28.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:pjds_spmv --csv --log-file gpurun_out/ncu28.csv python tools/kbench.py --once --configs C3,C5 --fmts pjds32s,pjds32 --dtypes f64 --sigmas 0,16384,262144,4194304 > /dev/null 2>&1
tail -2 gpurun_out/kbench28.err
