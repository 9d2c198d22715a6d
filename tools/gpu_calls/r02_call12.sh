# round 2, call 12: TMA ring depth (staging 1: U=2, 8/12 stages; 3: U=4, 16 stages) vs the static kernel
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "tma_staged" > gpurun_out/r02c12_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c12_tests.txt
timeout 600 python tools/kbench.py --configs C4,W4,C2 --dtypes f32,f64 --fmts pjds32s --stagings 0,1,3 --reps 40 > gpurun_out/r02c12_tma.jsonl 2> gpurun_out/r02c12_tma.err
