timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 tools/nccl_2rank_1gpu.py C1 > gpurun_out/nccl2.log 2>&1
tail -8 gpurun_out/nccl2.log
