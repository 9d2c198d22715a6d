# refresh the committed ncu evidence of the bench kernel with the final build
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 3 -c 1 -o gpurun_out/prof40_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches40.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 2 > /dev/null 2>&1
