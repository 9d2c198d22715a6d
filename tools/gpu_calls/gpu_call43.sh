# contention-aware single-GPU emulation of the dist step (C5 DP, permuted basis) and the ncu traffic of cuSPARSE CSR SpMV on C5
timeout 1500 python tools/dist_emulate.py --config C5 --ranks 1,2,4,8 --modes permuted > gpurun_out/emul43.jsonl 2> gpurun_out/emul43.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cusparse43.csv python tools/cusparse_c5.py --reps 2 > gpurun_out/cusparse43.log 2>&1
