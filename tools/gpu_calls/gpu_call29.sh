python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/kbench.py --configs C5,C3 --fmts pjds32s,pjds32 --dtypes f64 --reps 30 > gpurun_out/kbench29.jsonl 2> gpurun_out/kbench29.err
tail -2 gpurun_out/kbench29.err
