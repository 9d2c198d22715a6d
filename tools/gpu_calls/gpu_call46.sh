# bench plumbing with the DIRECT transport (oversubscribed one-GPU mode: timings meaningless) and at N=1 through the
# dist path; memcheck + racecheck over a 2-process DIRECT worker
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 2 --config C3 --steps 20 --warmup 3 --transport direct > gpurun_out/bench46_r2_direct.json 2> gpurun_out/bench46.err
timeout 900 python bench.py --dist --transport direct --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench46_r1_direct.json 2>> gpurun_out/bench46.err
timeout 900 python bench.py --dist --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench46_r1_nccl.json 2>> gpurun_out/bench46.err
timeout 1200 compute-sanitizer --target-processes all --tool memcheck --error-exitcode 9 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29872 tests/fake_nccl/worker.py C1 direct 2 > gpurun_out/memcheck46.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck46.log
timeout 1200 compute-sanitizer --target-processes all --tool racecheck --error-exitcode 9 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29873 tests/fake_nccl/worker.py C1 direct 2 > gpurun_out/racecheck46.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck46.log
