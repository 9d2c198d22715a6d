# final-build ncu evidence (summarised on the box: full reports exceed the 64 MiB copy-back limit)
mkdir -p /tmp/ncu50
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 3 -c 1 -o /tmp/ncu50/c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 1 > /dev/null 2>&1
python tools/summarize_ncu.py full /tmp/ncu50/c5.ncu-rep gpurun_out/ncu50_full_C5.txt "C5 f64 permuted, bench default (b_r=32), final build" > /dev/null 2>&1
ncu -i /tmp/ncu50/c5.ncu-rep --page source --csv > /tmp/ncu50/c5_source.csv 2>/dev/null; head -c 2000000 /tmp/ncu50/c5_source.csv > gpurun_out/ncu50_source_C5_head.csv
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches50.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:pjds_spmv -s 3 -c 1 -o /tmp/ncu50/c5_direct python bench.py --dist --transport direct --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/summarize_ncu.py full /tmp/ncu50/c5_direct.ncu-rep gpurun_out/ncu50_full_C5_direct_r1.txt "C5 f64 permuted, DIRECT window kernel at N=1 (dist path), final build" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench50.json 2> gpurun_out/bench50.err
ls -la gpurun_out > gpurun_out/ls50.txt
