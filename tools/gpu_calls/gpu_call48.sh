# dynamic warp-tile schedule: bitwise tests, then static vs dynamic on the few-wave configs (and C3/C5 as controls)
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "schedule or tile_order or variants_bitwise or configs_full or dist_group or small" > gpurun_out/pytest48b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest48.log
timeout 1500 python tools/kbench.py --configs C4,C2,W4,C3 --dtypes f64,f32 --fmts pjds32,pjds32s --scheds 0,1,0,1 --reps 40 > gpurun_out/kbench48b.jsonl 2> gpurun_out/kbench48b.err
timeout 900 python tools/kbench.py --configs C5 --dtypes f64 --fmts pjds32s --scheds 0,1,0,1 --reps 20 >> gpurun_out/kbench48b.jsonl 2>> gpurun_out/kbench48b.err
