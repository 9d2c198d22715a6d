# round 2, call 18: sustained A/B of kernel variants in the bench loop (auto R4U2 vs lane-interleaved vs pipelined)
set -x
for i in 1 2; do
  for V in auto 4,34 4,18; do
    if [ "$V" = auto ]; then VA=""; else VA="--variant $V"; fi
    python bench.py $VA --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c18_${V/,/_}_$i.json 2> /dev/null
  done
done
