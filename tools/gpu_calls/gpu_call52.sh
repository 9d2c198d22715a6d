# full GPU suite + smoke with the final tree
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest52.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest52.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke52.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke52.log
