python -m pytest tests/test_gpu_parity.py tests/test_gpu_fake_nccl.py tests/test_gpu_dist_world1.py -x -q -k "dist or nccl or p2p" 2>&1 | tail -2
python tools/dist_emulate.py --modes permuted,rows > gpurun_out/dist_emul30.jsonl 2> gpurun_out/dist_emul30.err; tail -2 gpurun_out/dist_emul30.err
