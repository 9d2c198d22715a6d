# DIRECT transport after the coherent window loads + combined signal/wait kernels: tests, resources, emulation
timeout 1500 python -m pytest tests/test_gpu_fake_nccl.py tests/test_kernel_resources.py -x -q > gpurun_out/pytest45.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest45.log
for R in 1 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $R --master-addr 127.0.0.1 --master-port $((29860+R)) tools/direct_emulate.py C5 30 5 >> gpurun_out/direct45.jsonl 2>> gpurun_out/direct45.err
done
