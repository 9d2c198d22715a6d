# bench.py N>1 paths on one GPU after the trials/compare changes: NCCL transport through the
# one-GPU NCCL stand-in, and the P2P transport (CUDA IPC between processes on the same GPU)
g++ -O2 -std=c++17 -shared -fPIC -I/usr/local/cuda/include -o tests/fake_nccl/libfakenccl.so tests/fake_nccl/fake_nccl.cpp -L/usr/local/cuda/lib64 -L/usr/local/cuda/lib64/stubs -lcudart -lcuda -lrt
PJDS_NCCL_LIB=$PWD/tests/fake_nccl/libfakenccl.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 --config C3 --steps 20 --warmup 3 > gpurun_out/bench33_r2.json 2> gpurun_out/bench33.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 2 --config C3 --steps 20 --warmup 3 --transport p2p > gpurun_out/bench33_r2_p2p.json 2>> gpurun_out/bench33.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29663 bench.py --impl reference --gpus 2 --config C3 --steps 3 --warmup 3 > gpurun_out/bench33_ref_r2.json 2>> gpurun_out/bench33.err
