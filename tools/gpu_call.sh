# round 2, call 48: DIRECT transport with the lane-interleaved DP kernel at b_r 128 -- its tests
# (bench N>1 legs, fake-NCCL / multi-process DIRECT) and the one-GPU emulation at b_r 128
set -x
python -m pytest tests/test_gpu_bench_dist.py tests/test_gpu_fake_nccl.py -x -q > gpurun_out/r02c48_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c48_tests.txt
for R in 1 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $R --master-addr 127.0.0.1 --master-port $((29880+R)) tools/direct_emulate.py C5 30 5 128 >> gpurun_out/r02c48_direct_br128.jsonl 2>> gpurun_out/r02c48_direct.err
done
