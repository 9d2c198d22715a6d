python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/kbench.py --configs W4,W5 --fmts pjds32s,pjds32,ellr --dtypes f64,f32 --variants 0x0,1x8,2x4,1x24,2x20 > gpurun_out/kbench14.jsonl 2> gpurun_out/kbench14.err
python bench.py --steps 300 > gpurun_out/bench14.json 2> gpurun_out/bench14.err
tail -3 gpurun_out/kbench14.err gpurun_out/bench14.err
