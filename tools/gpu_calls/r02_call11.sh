# round 2, call 11: TMA-staged long-row kernel: parity test, then staging 0 vs 1 on long- and short-row configs
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "tma_staged" > gpurun_out/r02c11_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c11_tests.txt
python tools/kbench.py --configs C4,W4,W5,C3,C2 --dtypes f64,f32 --fmts pjds32s,pjds32 --stagings 0,1 --reps 40 > gpurun_out/r02c11_tma.jsonl 2> gpurun_out/r02c11_tma.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:spmv --csv --log-file gpurun_out/r02c11_ncu_tma.csv python tools/kbench.py --once --configs C4 --dtypes f32,f64 --fmts pjds32s --stagings 0,1 > /dev/null 2>&1
