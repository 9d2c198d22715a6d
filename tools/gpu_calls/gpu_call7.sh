python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/dist_emulate.py > gpurun_out/dist_emul7.jsonl 2> gpurun_out/dist_emul7.err; tail -3 gpurun_out/dist_emul7.err
python bench.py --steps 300 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -2 gpurun_out/bench7.err
