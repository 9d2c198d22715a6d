python tools/kbench.py --configs C2,C3,C4,C5,W4,W5 --fmts pjds32s --dtypes f64,f32 --variants 0x0 --reps 50 > gpurun_out/kbench16.jsonl 2> gpurun_out/kbench16.err
tail -2 gpurun_out/kbench16.err
