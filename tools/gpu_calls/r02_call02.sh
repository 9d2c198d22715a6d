# round 2, call 2: new bench (per_config, O2 parity, dist oversubscribe), new parity tests, one-call dist create
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c02_gputests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02c02_gputests.txt
python bench.py > gpurun_out/r02c02_bench.json 2> gpurun_out/r02c02_bench.err
