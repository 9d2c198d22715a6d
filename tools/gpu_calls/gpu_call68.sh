# y store experiment (permuted basis): R-wide vector store with an L2 policy vs plain scalar stores
mkdir -p gpurun_out
python tools/kbench.py --configs C5,C3,C2 --dtypes f64,f32 --fmts pjds32s --policies 1x2,257x2,513x2,769x2,1025x2,1x2 --reps 60 > gpurun_out/k68_ystore.jsonl 2> gpurun_out/k68.err
tail -n 3 gpurun_out/k68.err
