# round 2, call 53: lane-interleaved SP rows when one length class dominates (sAMG C2) -- the
# compressible/bitwise and bench-instance tests, then the bench per_config A/B (auto vs R4U2 plain)
set -x
python -m pytest tests -m gpu -x -q -k "compressible or configs_full or bench_instance or launch_overlap" > gpurun_out/r02c53_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c53_tests.txt
for V in auto plain auto plain; do
  if [ $V = auto ]; then A=""; else A="--variant 4,2"; fi
  python bench.py --config C2 --dtype f32 --steps 200 --no-cpu-baseline --no-compare --per-config C2:f32,C3:f32,C2:f64 $A > gpurun_out/r02c53_$V.tmp 2>> gpurun_out/r02c53_bench.err
  cat gpurun_out/r02c53_$V.tmp >> gpurun_out/r02c53_bench_$V.jsonl
done
rm -f gpurun_out/*.tmp
