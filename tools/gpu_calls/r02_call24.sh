# round 2, call 24 (re-entry in a fresh container): full GPU suite, smoke, default bench
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c24_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c24_smoke.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02c24_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c24_gputests.txt
python bench.py > gpurun_out/r02c24_bench.json 2> gpurun_out/r02c24_bench.err
