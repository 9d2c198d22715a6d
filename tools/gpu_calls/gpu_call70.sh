# After the vector y store default: GPU suite, smoke, bench, Lanczos, and refreshed ncu evidence of the bench kernel
mkdir -p gpurun_out /tmp/ncu70
python -m pytest tests -m gpu -x -q > gpurun_out/v70_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/v70_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/v70_tests.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/v70_tests.txt
timeout 900 python bench.py > gpurun_out/v70_bench.json 2> gpurun_out/v70_bench.err; echo "bench rc=$?" >> gpurun_out/v70_tests.txt
python tools/lanczos_bench.py C5 50 > gpurun_out/v70_lz.jsonl 2> gpurun_out/v70_lz.err
python tools/lanczos_bench.py C3 200 >> gpurun_out/v70_lz.jsonl 2>> gpurun_out/v70_lz.err
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 3 -c 1 -o /tmp/ncu70/c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 1 > /dev/null 2>&1
python tools/summarize_ncu.py full /tmp/ncu70/c5.ncu-rep gpurun_out/ncu70_full_C5.txt "C5 f64 permuted, bench default (b_r=32, vector y store evict_first)" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches70.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 2 > /dev/null 2>&1
python tools/summarize_ncu.py launches gpurun_out/launches70.csv gpurun_out/launches70.txt "bench.py --steps 5 --warmup 3 (C5 DP default), vector y store" > /dev/null 2>&1
tail -n 6 gpurun_out/v70_tests.txt
