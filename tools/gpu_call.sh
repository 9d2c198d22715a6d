# round 2, call 57: lane-interleaved rows inside the warp-granular order (row-only / y += stores):
# bitwise tests, then the row-only sweep plain vs interleaved under the automatic order
set -x
python -m pytest tests -m gpu -x -q -k "warp_tile_order or tile_order_bitwise or y_store or kernel_variants" > gpurun_out/r02c57_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c57_tests.txt
timeout 1200 python tools/kbench.py --configs C5,C3,C2 --dtypes f64,f32 --fmts pjds128 --variants 0x0,4x34,0x0,4x34 --reps 40 --rotate 2 > gpurun_out/r02c57_rows_il_worder.jsonl 2> gpurun_out/r02c57_rows.err
