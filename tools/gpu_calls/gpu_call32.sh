# b_r = 128 default: DRAM traffic table, full ncu capture of the bench kernel, launch list, bench lines
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:spmv_kernel --csv --log-file gpurun_out/ncu32.csv python tools/kbench.py --configs C2,C3,C4,C5,W4,W5 --dtypes f64,f32 --fmts pjds128s,pjds128 --once > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pjds_spmv -s 3 -c 1 -o gpurun_out/prof32_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches32.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compare --e2e-steps 2 > /dev/null 2>&1
python bench.py > gpurun_out/bench32.json 2> gpurun_out/bench32.err
python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/bench32_f32.json 2> gpurun_out/bench32_f32.err
python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench32_c3.json 2> gpurun_out/bench32_c3.err
