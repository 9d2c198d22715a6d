g++ -O2 -std=c++17 -shared -fPIC -I/usr/local/cuda/include -o tests/fake_nccl/libfakenccl.so tests/fake_nccl/fake_nccl.cpp -L/usr/local/cuda/lib64 -L/usr/local/cuda/lib64/stubs -lcudart -lcuda -lrt
PJDS_NCCL_LIB=$PWD/tests/fake_nccl/libfakenccl.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 --config C3 --steps 20 --warmup 3 > gpurun_out/bench21_r2.json 2> gpurun_out/bench21.err
PJDS_NCCL_LIB=$PWD/tests/fake_nccl/libfakenccl.so timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench21_r4.json 2>> gpurun_out/bench21.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29663 bench.py --impl reference --gpus 2 --steps 5 > gpurun_out/bench21_ref2.json 2>> gpurun_out/bench21.err
tail -5 gpurun_out/bench21.err
