python -m pytest tests -m gpu -x -q -k "variants" 2>&1 | tail -2
python tools/kbench.py --configs C4,C2,C3,C5 --fmts pjds32s --dtypes f32,f64 --variants 0x0,2x4,2x20,4x2,4x18,2x8,2x24,1x24 > gpurun_out/kbench13.jsonl 2> gpurun_out/kbench13.err
tail -3 gpurun_out/kbench13.err
