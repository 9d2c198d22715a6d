# round 2, call 27: late-trigger dependent launch for one-wave grids (mode 3 / auto)
set -x
python -m pytest tests -m gpu -x -q -k "launch_overlap" > gpurun_out/r02c27_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c27_tests.txt
timeout 900 python tools/kbench.py --configs C4 --dtypes f64,f32 --fmts pjds128s,ellr --reps 120 --rotate 64 --pdls 0:0,3:0,2:2,1:0,0:0,3:0,2:2 > gpurun_out/r02c27_late.jsonl 2> gpurun_out/r02c27_late.err
timeout 900 python tools/kbench.py --configs C2,C3 --dtypes f64,f32 --fmts pjds128s,ellr --reps 60 --rotate 8 --pdls 0:0,3:0,2:2,0:0,3:0,2:2 >> gpurun_out/r02c27_late.jsonl 2>> gpurun_out/r02c27_late.err
