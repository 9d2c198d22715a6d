# round 2, call 5: full-contention dist emulation (y-store / perm-store variants), Lanczos drift,
# rows-only clock sensitivity (kbench after an idle pause vs back to back)
set -x
python tools/lanczos_drift.py > gpurun_out/r02c05_lanczos_drift.jsonl 2> gpurun_out/r02c05_lanczos_drift.err
python tools/kbench.py --configs C5 --dtypes f64 --fmts pjds32,pjds32s,pjds32 --reps 20 > gpurun_out/r02c05_rows_clock.jsonl 2>&1
timeout 1500 python tools/dist_emulate2.py --ranks 2,4,8 --modes permuted,rows --ystore=-1,1,3 --pstore=0,3 > gpurun_out/r02c05_dist_emul2.jsonl 2> gpurun_out/r02c05_dist_emul2.err
