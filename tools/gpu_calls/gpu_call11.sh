python -m pytest tests -m gpu -x -q -k "lanczos" 2>&1 | tail -2
python tools/kbench.py --configs C3,C5,C2 --fmts ellr --dtypes f64 --variants 1x8,2x4,4x2,4x4 > gpurun_out/kbench11_ellr.jsonl 2> gpurun_out/kbench11.err
python tools/lanczos_bench.py C5 50 > gpurun_out/lanczos11.json 2>> gpurun_out/kbench11.err
python tools/lanczos_bench.py C3 200 >> gpurun_out/lanczos11.json 2>> gpurun_out/kbench11.err
tail -3 gpurun_out/kbench11.err
