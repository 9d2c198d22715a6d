# re-entry validation of the restored tree: GPU tests, smoke, default bench
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest41.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest41.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke41.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke41.log
timeout 900 python bench.py > gpurun_out/bench41.json 2> gpurun_out/bench41.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench41_ref.json 2>> gpurun_out/bench41.err
