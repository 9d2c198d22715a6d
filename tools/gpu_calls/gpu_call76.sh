# y-store alignment gate + aligned internal buffers: y-store tests, then the full GPU suite, smoke and bench
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "y_store" > gpurun_out/t76_ystore.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/t76_ystore.txt
python -m pytest tests -m gpu -x -q > gpurun_out/v76_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/v76_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/v76_tests.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/v76_tests.txt
timeout 900 python bench.py > gpurun_out/v76_bench.json 2> gpurun_out/v76_bench.err; echo "bench rc=$?" >> gpurun_out/v76_tests.txt
tail -n 2 gpurun_out/t76_ystore.txt; tail -n 5 gpurun_out/v76_tests.txt
