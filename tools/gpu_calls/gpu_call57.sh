# C4 (DLR1, one partial wave, chain-latency bound): deeper unroll and split-j variants
mkdir -p gpurun_out
python tools/kbench.py --configs C4 --dtypes f32,f64 --fmts pjds32s --variants 2x20,2x20,2x8,2x24,2x40,2x56,1x8,1x24,4x20,18x4,18x8,20x4,20x8,24x4 --reps 60 > gpurun_out/k57_c4.jsonl 2> gpurun_out/k57.err
tail -3 gpurun_out/k57.err
