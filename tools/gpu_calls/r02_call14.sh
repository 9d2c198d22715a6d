# round 2, call 14: b_r 32 vs 128 in the sustained bench loop (200 steps), alternating, same box
set -x
for i in 1 2; do
  for BR in 32 128; do
    python bench.py --block-rows $BR --no-per-config --no-compare --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02c14_br${BR}_$i.json 2> /dev/null
  done
done
