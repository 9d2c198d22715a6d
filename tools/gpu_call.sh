# round 2, call 54: final-tree validation after the SP lane-interleaving rule -- smoke, full GPU
# suite, default bench
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c54_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c54_smoke.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02c54_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c54_gputests.txt
python bench.py > gpurun_out/r02c54_bench.json 2> gpurun_out/r02c54_bench.err
