# round 2, call 32: L2 set-aside for evict_last x lines at intermediate sizes (C5, default order)
set -x
timeout 900 python tools/l2_persist_probe.py --keys none --limits 0,8388608,16777216,25165824,33554432,50331648,67108864,max,0 --reps 40 > gpurun_out/r02c32_persist.jsonl 2> gpurun_out/r02c32_persist.err
timeout 900 python tools/l2_persist_probe.py --dtype f32 --keys none --limits 0,16777216,33554432,max,0 --reps 40 >> gpurun_out/r02c32_persist.jsonl 2>> gpurun_out/r02c32_persist.err
