python -m pytest tests/test_gpu_fake_nccl.py tests/test_gpu_dist_world1.py -x -q 2>&1 | tail -30
