# full ncu capture of the default kernel on the two weakest configs (C4 SP, C2 SP)
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 5 -c 1 -o gpurun_out/prof34_c4sp python tools/kbench.py --configs C4 --dtypes f32 --fmts pjds32s --reps 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 5 -c 1 -o gpurun_out/prof34_c2sp python tools/kbench.py --configs C2 --dtypes f32 --fmts pjds32s --reps 3 > /dev/null 2>&1
