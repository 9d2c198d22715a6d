# round 2, call 61: the compression test with the device-capability guard
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k compressible > gpurun_out/r02c61_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c61_tests.txt
