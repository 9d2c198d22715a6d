# final-build ncu evidence: full capture + launch list of the bench command, full capture of the DIRECT window kernel (N=1 dist path), final bench
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 3 -c 1 -o gpurun_out/prof49_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches49.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:pjds_spmv -s 3 -c 1 -o gpurun_out/prof49_c5_direct python bench.py --dist --transport direct --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench49.json 2> gpurun_out/bench49.err
