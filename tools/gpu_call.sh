# round 2, call 43: automatic lane-interleaved rows for DP permuted basis -- full GPU suite, then the
# bench A/B (auto vs the plain R4U2 variant) alternating twice on one box
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c43_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c43_gputests.txt
for V in auto plain auto plain; do
  if [ $V = auto ]; then A=""; else A="--variant 4,2"; fi
  python bench.py --no-cpu-baseline $A > gpurun_out/r02c43_bench_$V.json.tmp 2>> gpurun_out/r02c43_bench.err
  cat gpurun_out/r02c43_bench_$V.json.tmp >> gpurun_out/r02c43_bench_$V.jsonl
done
rm -f gpurun_out/*.tmp
