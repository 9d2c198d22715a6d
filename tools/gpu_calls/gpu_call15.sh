ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 5 -c 1 -o gpurun_out/prof15_c2 python tools/kbench.py --configs C2 --dtypes f64 --fmts pjds32s --reps 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 5 -c 1 -o gpurun_out/prof15_c4sp python tools/kbench.py --configs C4 --dtypes f32 --fmts pjds32s --reps 3 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
