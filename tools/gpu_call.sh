# round 2, call 41: multi-GPU emulations with the final build (compressible index arrays, launch
# overlap): the NCCL split under full contention, and DIRECT with R processes on one GPU
set -x
timeout 900 python tools/dist_emulate2.py --ranks 2,4,8 --modes rows --nl-sigma 1024 > gpurun_out/r02c41_dist_emul2.jsonl 2> gpurun_out/r02c41_dist_emul2.err
for R in 1 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $R --master-addr 127.0.0.1 --master-port $((29870+R)) tools/direct_emulate.py C5 30 5 >> gpurun_out/r02c41_direct.jsonl 2>> gpurun_out/r02c41_direct.err
done
