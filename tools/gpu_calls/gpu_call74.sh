# ELLPACK-R DP after reverting its y-store change (is the slowdown seen in call 73 the change or the box?)
mkdir -p gpurun_out
python tools/kbench.py --configs C2,C3,C5 --dtypes f64 --fmts ellr,pjds32s --policies 513x2,1x2 --reps 60 > gpurun_out/k74.jsonl 2> gpurun_out/k74.err
