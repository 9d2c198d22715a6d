# round 2, call 30: row-only basis with the lane-interleaved variant (one gather instruction covers
# 32 consecutive sorted rows); dist full-contention emulation re-run with the final build
set -x
timeout 900 python tools/kbench.py --configs C5,C3,C2 --dtypes f64,f32 --fmts pjds128 --variants 0x0,4x34,2x36,4x2,0x0,4x34 --orders 2,1 --reps 40 --rotate 2 > gpurun_out/r02c30_rows_il.jsonl 2> gpurun_out/r02c30_rows_il.err
timeout 900 python tools/dist_emulate2.py --ranks 2,4,8 --modes rows --nl-sigma 1024 > gpurun_out/r02c30_dist_emul2.jsonl 2> gpurun_out/r02c30_dist_emul2.err
