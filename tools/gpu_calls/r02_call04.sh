# round 2, call 4: row-only basis store policies (kbench) and the full-contention dist emulation
set -x
python tools/kbench.py --configs C5,C3,C2 --dtypes f64 --fmts pjds32 --policies 513x2,66049x2,131585x2,197121x2 --reps 40 > gpurun_out/r02c04_rows_pstore.jsonl 2> gpurun_out/r02c04_rows_pstore.err
python tools/kbench.py --configs C5 --dtypes f64 --fmts pjds32s,pjds32 --reps 40 >> gpurun_out/r02c04_rows_pstore.jsonl 2>> gpurun_out/r02c04_rows_pstore.err
timeout 1500 python tools/dist_emulate2.py --ranks 2,4,8 --modes permuted,rows --ystore -1,1,3 --pstore 0,3 > gpurun_out/r02c04_dist_emul2.jsonl 2> gpurun_out/r02c04_dist_emul2.err
