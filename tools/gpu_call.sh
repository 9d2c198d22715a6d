# round 2, call 49: occupancy of the lane-interleaved DP kernel -- default build (56 registers,
# 4 CTAs/SM) vs dev builds with __launch_bounds__ min 5 (48 regs, 8 B spill) and 6 (40 regs, spills),
# alternating (build/alt/*.so, PJDS_LIB_PATH)
set -x
for L in default minb5 minb6 default minb5 minb6; do
  if [ $L = default ]; then unset PJDS_LIB_PATH; else export PJDS_LIB_PATH=$PWD/build/alt/libpjds_$L.so; fi
  timeout 900 python tools/kbench.py --configs C5,C3,C2 --dtypes f64 --fmts pjds128s --reps 40 --rotate 2 | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/r02c49_minb.jsonl 2>> gpurun_out/r02c49_minb.err
done
