# Lanczos: 8-wide partial sums, R1 over 148 CTAs + last-CTA sum; tests, sanitizer, timing
mkdir -p gpurun_out
python -m pytest tests/test_lanczos.py -m gpu -q > gpurun_out/lz60_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/lz60_tests.txt
compute-sanitizer --tool memcheck python -m pytest tests/test_lanczos.py -m gpu -q -k "matches_oracle or breakdown" > gpurun_out/lz60_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/lz60_memcheck.txt
compute-sanitizer --tool racecheck python -m pytest tests/test_lanczos.py -m gpu -q -k "breakdown" > gpurun_out/lz60_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/lz60_racecheck.txt
python tools/lanczos_bench.py C3 200 > gpurun_out/lz60.jsonl 2> gpurun_out/lz60.err
python tools/lanczos_bench.py C5 50 >> gpurun_out/lz60.jsonl 2>> gpurun_out/lz60.err
for f in gpurun_out/lz60_tests.txt gpurun_out/lz60_memcheck.txt gpurun_out/lz60_racecheck.txt; do tail -n 3 $f; done
