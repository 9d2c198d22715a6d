# round 2, call 25: programmatic dependent launch (pjds_set_launch_overlap): dependent-chain test,
# then a kernel sweep, launch overlap off/on x L2 prefetch columns, L2-cold (x/y rotated) and warm
set -x
python -m pytest tests -m gpu -x -q -k "launch_overlap or kernel_variants_bitwise or tile_order_bitwise" > gpurun_out/r02c25_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c25_tests.txt
timeout 1200 python tools/kbench.py --configs C2,C3,C4,C5 --dtypes f64,f32 --fmts pjds128s,ellr --reps 60 --rotate 8 --pdls 0:0,1:0,1:2,1:4,1:8,1:64,0:0,1:0,1:4 > gpurun_out/r02c25_pdl_cold.jsonl 2> gpurun_out/r02c25_pdl_cold.err
timeout 600 python tools/kbench.py --configs C2,C4 --dtypes f64,f32 --fmts pjds128s --reps 60 --rotate 1 --pdls 0:0,1:0,1:4,0:0,1:0,1:4 > gpurun_out/r02c25_pdl_warm.jsonl 2> gpurun_out/r02c25_pdl_warm.err
timeout 600 python tools/kbench.py --configs C5 --dtypes f64 --fmts pjds128 --reps 40 --rotate 2 --pdls 0:0,1:0,1:4,0:0,1:0,1:4 > gpurun_out/r02c25_pdl_rows.jsonl 2> gpurun_out/r02c25_pdl_rows.err
