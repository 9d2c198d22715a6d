# round 2, call 51: the Lanczos fused-dot product with the lane-interleaved DP layout at b_r 128 --
# Lanczos GPU tests, per-step device times at b_r 32 and 128
set -x
python -m pytest tests/test_lanczos.py -x -q > gpurun_out/r02c51_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c51_tests.txt
for BR in 32 128; do
  timeout 900 python tools/lanczos_bench.py C5 50 $BR >> gpurun_out/r02c51_lanczos.jsonl 2>> gpurun_out/r02c51_lanczos.err
  timeout 600 python tools/lanczos_bench.py C3 200 $BR >> gpurun_out/r02c51_lanczos.jsonl 2>> gpurun_out/r02c51_lanczos.err
done
