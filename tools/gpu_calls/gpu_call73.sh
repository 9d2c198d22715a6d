# ELLPACK-R with the same vector y store: tests, interleaved A/B
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "ellr or ELLR or ellpack" > gpurun_out/t73.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/t73.txt
python tools/kbench.py --configs C2,C3,C4,C5 --dtypes f64,f32 --fmts ellr --policies 1x2,513x2,1x2,513x2 --reps 60 > gpurun_out/k73_ellr_ystore.jsonl 2> gpurun_out/k73.err
tail -n 3 gpurun_out/t73.txt
