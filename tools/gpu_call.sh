# round 2, call 56: launch-overlap prefetch columns re-checked with the final kernels (compressed
# index arrays, lane-interleaved rows), x/y rotated
set -x
timeout 1200 python tools/kbench.py --configs C2,C3 --dtypes f64,f32 --fmts pjds128s --pdls 2:2,2:0,2:4,3:0,2:2,2:0,2:4,3:0 --reps 60 --rotate 8 > gpurun_out/r02c56_pdl.jsonl 2> gpurun_out/r02c56_pdl.err
