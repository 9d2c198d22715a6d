timeout 1500 python -m pytest tests/test_gpu_fake_nccl.py -x -q -k "c5_sampled" > gpurun_out/pytest53.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest53.log
