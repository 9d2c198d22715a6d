# round 2, call 23: the nonlocal part's kernel variant (A_nl alone), rows basis, R = 4 and 8
set -x
timeout 900 python tools/dist_emulate2.py --ranks 4,8 --modes rows --nl-variants 1x8,2x4,4x2,4x4,1x2 > gpurun_out/r02c23_nl_variants.jsonl 2> gpurun_out/r02c23_nl_variants.err
