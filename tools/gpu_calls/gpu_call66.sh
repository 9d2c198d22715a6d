# Final-tree validation after the Lanczos reduction changes: GPU suite, smoke, default bench, Lanczos wall vs device time
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/v66_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/v66_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/v66_tests.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/v66_tests.txt
python bench.py > gpurun_out/v66_bench.json 2> gpurun_out/v66_bench.err; echo "bench rc=$?" >> gpurun_out/v66_tests.txt
python tools/lanczos_bench.py C5 50 > gpurun_out/v66_lz.jsonl 2> gpurun_out/v66_lz.err
python tools/lanczos_bench.py C5 50 >> gpurun_out/v66_lz.jsonl 2>> gpurun_out/v66_lz.err
tail -n 6 gpurun_out/v66_tests.txt
