# Lanczos: 8-wide partial sums, own x rows via cp.async into shared memory (DOT epilogue); tests, sanitizer, timing
mkdir -p gpurun_out
python -m pytest tests/test_lanczos.py -m gpu -q > gpurun_out/lz64_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/lz64_tests.txt
compute-sanitizer --tool memcheck python -m pytest tests/test_lanczos.py -m gpu -q -k "matches_oracle or breakdown" > gpurun_out/lz64_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/lz64_memcheck.txt
compute-sanitizer --tool racecheck python -m pytest tests/test_lanczos.py -m gpu -q -k "breakdown" > gpurun_out/lz64_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/lz64_racecheck.txt
python tools/lanczos_bench.py C3 200 > gpurun_out/lz64.jsonl 2> gpurun_out/lz64.err
python tools/lanczos_bench.py C5 50 >> gpurun_out/lz64.jsonl 2>> gpurun_out/lz64.err
cat gpurun_out/lz64_tests.txt | tail -n 3; tail -n 2 gpurun_out/lz64_memcheck.txt gpurun_out/lz64_racecheck.txt 2>/dev/null; true
