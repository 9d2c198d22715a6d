# full GPU suite after the DIRECT changes, smoke, default bench (with same-run parity)
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest47.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest47.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke47.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke47.log
timeout 900 python bench.py > gpurun_out/bench47.json 2> gpurun_out/bench47.err
