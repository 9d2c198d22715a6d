# DIRECT in SP, and sanitizers over the dynamic-schedule kernel
timeout 1500 python -m pytest tests/test_gpu_fake_nccl.py -x -q -k direct > gpurun_out/pytest51.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest51.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "schedule_bitwise and 1" > gpurun_out/memcheck51.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck51.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "schedule_bitwise and 1" > gpurun_out/racecheck51.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck51.log
