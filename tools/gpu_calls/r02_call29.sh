# round 2, call 29: launch overlap A/B inside bench.py's own per_config timing (same box, alternating)
set -x
for LO in 0,0 2,2 0,0 2,2 3,0 1,2; do
  python bench.py --config C2 --steps 100 --no-compare --no-cpu-baseline --e2e-steps 3 --per-config C4:f64,C4:f32,C2:f32,C3:f64 --launch-overlap $LO > gpurun_out/r02c29_lo_$LO.json 2>> gpurun_out/r02c29.err
done
