# larger phonon windows for the 2-D tile key on C5 DP
python tools/kbench.py --configs C5 --dtypes f64 --fmts pjds32s --keys none,w32768,w49152,w71253,none,w32768,w49152,w71253 --reps 60 > gpurun_out/keys2.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pjds_spmv --csv --log-file gpurun_out/keys2_ncu.csv python tools/kbench.py --configs C5 --dtypes f64 --fmts pjds32s --keys none,w32768,w49152,w71253 --once > /dev/null 2>&1
