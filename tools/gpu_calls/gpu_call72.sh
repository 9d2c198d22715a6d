# Roofline table refresh (kbench: NVML query moved out of the timed region): every config, both precisions, pJDS permuted / rows-only, ELLPACK-R
mkdir -p gpurun_out
python tools/kbench.py --configs C2,C3,C4,C5 --dtypes f64,f32 --fmts pjds32s,pjds32,ellr --reps 60 > gpurun_out/k72_all.jsonl 2> gpurun_out/k72.err
tail -n 3 gpurun_out/k72.err
