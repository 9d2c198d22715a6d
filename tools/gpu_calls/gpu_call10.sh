python -m pytest tests -m gpu -x -q -k "ellr or variants or configs_full" 2>&1 | tail -2
python tools/kbench.py --configs C2,C3,C4,C5 --fmts ellr --dtypes f64,f32 --variants 0x0,1x8,2x4,4x2 > gpurun_out/kbench10_ellr.jsonl 2> gpurun_out/kbench10.err
python tools/kbench.py --configs C4 --fmts pjds32s --dtypes f32,f64 --variants 1x8,2x4,2x8,4x2,4x4 > gpurun_out/kbench10_c4.jsonl 2>> gpurun_out/kbench10.err
tail -2 gpurun_out/kbench10.err
