python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --dist --config C3 --no-cpu-baseline --steps 50 > gpurun_out/bench17_dist.json 2> gpurun_out/bench17_dist.err; tail -3 gpurun_out/bench17_dist.err
python bench.py --dist --config C3 --no-cpu-baseline --steps 50 --basis rows > gpurun_out/bench17_dist_rows.json 2>> gpurun_out/bench17_dist.err
