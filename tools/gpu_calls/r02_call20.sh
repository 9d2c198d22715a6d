# round 2, call 20: final-tree validation (GPU suite, smoke, default bench, reference arm)
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c20_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c20_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c20_smoke.txt 2>&1
python bench.py --impl reference > gpurun_out/r02c20_reference.json 2> gpurun_out/r02c20_reference.err
python bench.py > gpurun_out/r02c20_bench.json 2> gpurun_out/r02c20_bench.err
