python -m pytest tests/test_gpu_parity.py -x -q -k "host" 2>&1 | tail -2
python bench.py --steps 200 > gpurun_out/bench31.json 2> gpurun_out/bench31.err; tail -2 gpurun_out/bench31.err
