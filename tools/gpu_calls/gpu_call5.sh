python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -2 gpurun_out/bench5.err
python bench.py --impl reference --steps 20 > gpurun_out/bench5_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 3 -c 1 -o gpurun_out/prof5_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 3 -c 1 -o gpurun_out/prof5_c3 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 1 > /dev/null 2>&1
ls gpurun_out
