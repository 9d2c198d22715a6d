# round 2, call 52: final-tree validation after the DIRECT / Lanczos lane-interleaved changes --
# smoke, full GPU suite, default bench
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c52_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c52_smoke.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02c52_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c52_gputests.txt
python bench.py > gpurun_out/r02c52_bench.json 2> gpurun_out/r02c52_bench.err
