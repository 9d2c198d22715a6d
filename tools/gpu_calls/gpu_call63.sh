mkdir -p gpurun_out
python -m pytest tests/test_lanczos.py -m gpu -q > gpurun_out/lz63_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/lz63_tests.txt
python tools/lanczos_bench.py C3 200 > gpurun_out/lz63.jsonl 2> gpurun_out/lz63.err
python tools/lanczos_bench.py C5 50 >> gpurun_out/lz63.jsonl 2>> gpurun_out/lz63.err
for f in gpurun_out/lz63_tests.txt gpurun_out/lz63_memcheck.txt gpurun_out/lz63_racecheck.txt; do tail -n 3 $f; done
