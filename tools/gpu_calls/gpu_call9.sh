python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py > gpurun_out/bench9.json 2> gpurun_out/bench9.err; tail -2 gpurun_out/bench9.err
python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/bench9_f32.json 2> gpurun_out/bench9_f32.err
python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench9_c3.json 2>&1
python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench9_c2.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 3 -c 1 -o gpurun_out/prof9_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches9.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 2 > /dev/null 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "small and 32 and float64 and (random or empty or adversarial or identity)" > gpurun_out/memcheck9.log 2>&1; echo memcheck rc=$? >> gpurun_out/memcheck9.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "small and 128 and float32 and (random or clustered)" > gpurun_out/racecheck9.log 2>&1; echo racecheck rc=$? >> gpurun_out/racecheck9.log
tail -3 gpurun_out/memcheck9.log gpurun_out/racecheck9.log
