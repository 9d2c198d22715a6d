# round 2, call 13: TMA-staged kernel with one mbarrier poller per warp and 512-row tiles
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "tma_staged" > gpurun_out/r02c13_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c13_tests.txt
timeout 600 python tools/kbench.py --configs C4,W4,C2 --dtypes f32,f64 --fmts pjds32s --stagings 0,1,3 --reps 40 > gpurun_out/r02c13_tma.jsonl 2> gpurun_out/r02c13_tma.err
