python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/kbench.py --configs C3,C5,C2,C4 --fmts ellr --dtypes f64,f32 --variants 1x8,2x4,4x2 > gpurun_out/kbench12_ellr.jsonl 2> gpurun_out/kbench12.err
python tools/lanczos_bench.py C5 50 > gpurun_out/lanczos12.json 2>> gpurun_out/kbench12.err
python tools/lanczos_bench.py C3 200 >> gpurun_out/lanczos12.json 2>> gpurun_out/kbench12.err
tail -3 gpurun_out/kbench12.err
