# Lanczos: 8-wide partial sums, R2 fused into the update kernel (last CTA); tests, sanitizer, timing
mkdir -p gpurun_out
python -m pytest tests/test_lanczos.py -m gpu -q > gpurun_out/lz59_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/lz59_tests.txt
compute-sanitizer --tool memcheck python -m pytest tests/test_lanczos.py -m gpu -q -k "matches_oracle or breakdown" > gpurun_out/lz59_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/lz59_memcheck.txt
compute-sanitizer --tool racecheck python -m pytest tests/test_lanczos.py -m gpu -q -k "breakdown" > gpurun_out/lz59_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/lz59_racecheck.txt
python tools/lanczos_bench.py C3 200 > gpurun_out/lz59.jsonl 2> gpurun_out/lz59.err
python tools/lanczos_bench.py C5 50 >> gpurun_out/lz59.jsonl 2>> gpurun_out/lz59.err
for f in gpurun_out/lz59_tests.txt gpurun_out/lz59_memcheck.txt gpurun_out/lz59_racecheck.txt; do tail -n 3 $f; done
