# round 2, call 50: the one-wave DLR1 matrix (C4) with compression + launch overlap: variant sweep
# incl. the long-row split-j kernel, x/y rotated
set -x
timeout 1200 python tools/kbench.py --configs C4 --dtypes f32,f64 --fmts pjds128s --variants 0x0,1x8,1x4,2x8,2x20,18x4,18x8,20x4,0x0 --reps 120 --rotate 64 > gpurun_out/r02c50_c4.jsonl 2> gpurun_out/r02c50_c4.err
