# y store experiment, interleaved A/B (plain vs vector+evict_normal vs vector+evict_first)
mkdir -p gpurun_out
python tools/kbench.py --configs C5,C3,C2,C4 --dtypes f64,f32 --fmts pjds32s --policies 1x2,257x2,513x2,1x2,257x2,513x2,1x2,257x2,513x2 --reps 60 > gpurun_out/k69_ystore_ab.jsonl 2> gpurun_out/k69.err
tail -n 3 gpurun_out/k69.err
