# Lanczos: 8-wide partial sums, per-warp dot partials, no CTA barrier (DOT epilogue); tests, sanitizer, timing
mkdir -p gpurun_out
python -m pytest tests/test_lanczos.py -m gpu -q > gpurun_out/lz65_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/lz65_tests.txt
compute-sanitizer --tool memcheck python -m pytest tests/test_lanczos.py -m gpu -q -k "matches_oracle or breakdown" > gpurun_out/lz65_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/lz65_memcheck.txt
compute-sanitizer --tool racecheck python -m pytest tests/test_lanczos.py -m gpu -q -k "breakdown" > gpurun_out/lz65_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/lz65_racecheck.txt
python tools/lanczos_bench.py C3 200 > gpurun_out/lz65.jsonl 2> gpurun_out/lz65.err
python tools/lanczos_bench.py C5 50 >> gpurun_out/lz65.jsonl 2>> gpurun_out/lz65.err
cat gpurun_out/lz65_tests.txt | tail -n 3; tail -n 2 gpurun_out/lz65_memcheck.txt gpurun_out/lz65_racecheck.txt 2>/dev/null; true
