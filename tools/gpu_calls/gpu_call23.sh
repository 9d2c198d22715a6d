python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/kbench.py --configs C4,W4,C2,C3,W5 --fmts pjds32s --dtypes f32,f64 --variants 0x0 --reps 50 > gpurun_out/kbench23.jsonl 2> gpurun_out/kbench23.err
tail -2 gpurun_out/kbench23.err
