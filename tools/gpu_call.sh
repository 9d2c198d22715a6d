# round 2, call 55: row-only basis tile orders under compression (0 storage, 1 CTA original-row,
# 3 warp-granular = auto for mixed classes)
set -x
timeout 1200 python tools/kbench.py --configs C5,C3 --dtypes f64,f32 --fmts pjds128 --orders 3,1,0,3,1 --reps 40 --rotate 2 > gpurun_out/r02c55_rows_orders.jsonl 2> gpurun_out/r02c55_rows_orders.err
