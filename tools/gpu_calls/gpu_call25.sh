python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/kbench.py --configs C2,C3,C4,C5,W4,W5 --fmts pjds32s --dtypes f64,f32 --variants 0x0 --reps 50 > gpurun_out/kbench25.jsonl 2> gpurun_out/kbench25.err
python tools/kbench.py --configs C4,W4 --fmts pjds32s --dtypes f32,f64 --variants 2x4,2x20,1x8,1x24 --reps 50 > gpurun_out/kbench25b.jsonl 2>> gpurun_out/kbench25.err
python bench.py > gpurun_out/bench25.json 2>> gpurun_out/kbench25.err
tail -2 gpurun_out/kbench25.err
