# round 2, call 26: launch overlap auto (library default) -- full GPU suite, bench; then the
# row-only basis with sigma windows (exploration)
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02c26_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c26_gputests.txt
python bench.py > gpurun_out/r02c26_bench.json 2> gpurun_out/r02c26_bench.err
timeout 900 python tools/kbench.py --configs C2,C3,C5 --dtypes f64 --fmts pjds128,pjds128s --sigmas 0,1024,4096,16384 --reps 40 --rotate 2 > gpurun_out/r02c26_rows_sigma.jsonl 2> gpurun_out/r02c26_rows_sigma.err
