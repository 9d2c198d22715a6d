# round 2, call 22: non-default bench invocations still produce a valid line
set -x
python bench.py --config C3 --no-per-config > gpurun_out/r02c22_c3.json 2> gpurun_out/r02c22_c3.err
python bench.py --dtype f32 --no-per-config --no-compare > gpurun_out/r02c22_f32.json 2> gpurun_out/r02c22_f32.err
python bench.py --basis rows --no-per-config --no-compare --no-cpu-baseline > gpurun_out/r02c22_rows.json 2> gpurun_out/r02c22_rows.err
python bench.py --impl ellr --no-cpu-baseline > gpurun_out/r02c22_ellr.json 2> gpurun_out/r02c22_ellr.err
python bench.py --dist --config C3 --no-cpu-baseline > gpurun_out/r02c22_dist1.json 2> gpurun_out/r02c22_dist1.err
python bench.py --config C4 --no-per-config > gpurun_out/r02c22_c4.json 2> gpurun_out/r02c22_c4.err
