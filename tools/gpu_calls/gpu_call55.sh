# Re-entry validation of the current tree on a fresh box: GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v55_build.log 2>&1; echo "build rc=$?" >> gpurun_out/v55_tests.txt
python -m pytest tests -m gpu -x -q > gpurun_out/v55_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/v55_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/v55_tests.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/v55_tests.txt
python bench.py > gpurun_out/v55_bench.json 2> gpurun_out/v55_bench.err; echo "bench rc=$?" >> gpurun_out/v55_tests.txt
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v55_ref.json 2> gpurun_out/v55_ref.err; echo "ref rc=$?" >> gpurun_out/v55_tests.txt
tail -3 gpurun_out/v55_tests.txt
