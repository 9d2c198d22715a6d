# DLR1 (C4): lane-interleaved rows put the 6 rows of a point (same columns) in adjacent lanes of one gather
mkdir -p gpurun_out
python tools/kbench.py --configs C4 --dtypes f32,f64 --fmts pjds32s,pjds64s,pjds128s --variants 0x0,2x4,2x20,2x36,2x52,1x8,4x2,4x34,4x4,4x36 --reps 60 > gpurun_out/k56_c4_il.jsonl 2> gpurun_out/k56.err
python tools/kbench.py --configs C4 --dtypes f32,f64 --fmts pjds64,pjds128 --variants 0x0,2x36,4x34 --reps 60 >> gpurun_out/k56_c4_il.jsonl 2>> gpurun_out/k56.err
for v in 0x0 2x36 4x34; do
ncu --set full --clock-control none -k regex:pjds_spmv -c 1 --csv --page raw python tools/kbench.py --configs C4 --dtypes f32 --fmts pjds128s --variants $v --once > gpurun_out/k56_ncu_c4f32_$v.csv 2>>gpurun_out/k56.err
done
tail -3 gpurun_out/k56.err
