# round 2, call 58: final-tree validation after extending lane interleaving to the row-only / y +=
# stores -- smoke, full GPU suite, default bench
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c58_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c58_smoke.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02c58_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c58_gputests.txt
python bench.py > gpurun_out/r02c58_bench.json 2> gpurun_out/r02c58_bench.err
