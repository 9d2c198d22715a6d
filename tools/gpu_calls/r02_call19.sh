# round 2, call 19: sustained A/B of more kernel variants (R4U4, R2U4, R2U8) against auto (R4U2), b_r 128
set -x
for i in 1 2; do
  for V in auto 4,4 2,4 2,8; do
    if [ "$V" = auto ]; then VA=""; else VA="--variant $V"; fi
    python bench.py $VA --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c19_${V/,/_}_$i.json 2> /dev/null
  done
done
