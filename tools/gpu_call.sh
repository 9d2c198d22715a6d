# round 2, call 46: final-tree validation -- smoke, full GPU suite, default bench, reference arm
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c46_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c46_smoke.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02c46_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c46_gputests.txt
python bench.py > gpurun_out/r02c46_bench.json 2> gpurun_out/r02c46_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02c46_reference.json 2> gpurun_out/r02c46_reference.err
