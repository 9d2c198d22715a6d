# round 2, call 21: extended dist / y-store parity tests
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "dist_group or y_store" > gpurun_out/r02c21_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c21_tests.txt
