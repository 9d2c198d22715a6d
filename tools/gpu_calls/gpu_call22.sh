timeout 900 python -m pytest tests/test_gpu_fake_nccl.py -x -q 2>&1 | tail -30
