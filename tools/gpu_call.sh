# round 2, call 47: row-only basis (y stored through perm) with the lane-interleaved layout, now that
# the index arrays are compressed; plain auto (warp-granular order) vs IL (CTA original-row order)
set -x
timeout 1200 python tools/kbench.py --configs C5,C3,C2 --dtypes f64,f32 --fmts pjds128 --variants 0x0,4x34,0x0,4x34 --reps 40 --rotate 2 > gpurun_out/r02c47_rows_il.jsonl 2> gpurun_out/r02c47_rows_il.err
