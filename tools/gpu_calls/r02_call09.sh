# round 2, call 9: balanced persistent grid vs static (sched 2 vs 0) on the few-wave configs; tests
set -x
python tools/kbench.py --configs C2,C4,C3,W4 --dtypes f64,f32 --fmts pjds32s,pjds32 --scheds 0,2 --reps 40 > gpurun_out/r02c09_bal.jsonl 2> gpurun_out/r02c09_bal.err
python -m pytest tests/test_gpu_parity.py -x -q -k "schedule or warp_tile or tile_order or configs_full" > gpurun_out/r02c09_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c09_tests.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.avg --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c09_ncu_bal.csv python tools/kbench.py --once --configs C4,C2 --dtypes f32,f64 --fmts pjds32s --scheds 0,2 > /dev/null 2>&1
