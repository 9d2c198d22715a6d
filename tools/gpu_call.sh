# round 2, call 44: lane-interleaved DP kernel at 5 resident CTAs/SM (48 registers, 8-byte spill)
# vs the default (56 registers, 4 CTAs/SM), alternating
set -x
for L in default minb5 default minb5; do
  if [ $L = minb5 ]; then export PJDS_LIB_PATH=$PWD/experiments/libpjds_ilminb5.so; else unset PJDS_LIB_PATH; fi
  timeout 900 python tools/kbench.py --configs C5,C3,C2 --dtypes f64 --fmts pjds128s --reps 40 --rotate 2 | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/r02c44_minb.jsonl 2>> gpurun_out/r02c44_minb.err
done
