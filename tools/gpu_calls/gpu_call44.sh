# DIRECT transport (fused remote-gather kernel over IPC-mapped x windows): multi-process tests on one GPU,
# existing dist/parity tests, resource check, then the C5 one-GPU emulation at R = 1, 2, 4, 8
timeout 1500 python -m pytest tests/test_gpu_fake_nccl.py tests/test_gpu_dist_world1.py -x -q > gpurun_out/pytest44.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest44.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "dist or configs_full or c5" >> gpurun_out/pytest44.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/pytest44.log
for R in 1 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $R --master-addr 127.0.0.1 --master-port $((29850+R)) tools/direct_emulate.py C5 20 10 >> gpurun_out/direct44.jsonl 2>> gpurun_out/direct44.err
done
