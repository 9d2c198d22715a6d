# 2-D (phonon window, original row) tile keys on C5: timing and DRAM bytes
python tools/kbench.py --configs C5 --dtypes f64,f32 --fmts pjds32s --keys none,w4096,w8192,w16384,w32768,none --reps 40 > gpurun_out/keys.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pjds_spmv --csv --log-file gpurun_out/keys_ncu.csv python tools/kbench.py --configs C5 --dtypes f64 --fmts pjds32s --keys none,w4096,w8192,w16384,w32768 --once > /dev/null 2>&1
