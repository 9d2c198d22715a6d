# round 2, call 1: re-entry validation (GPU tests, smoke, default bench)
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c01_gputests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02c01_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c01_smoke.txt 2>&1
python bench.py > gpurun_out/r02c01_bench.json 2> gpurun_out/r02c01_bench.err
