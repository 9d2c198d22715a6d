# cuSPARSE witness tests (SURVEY §8(c) O1 pin (ii)) and the bench with the cuSPARSE compare leg
timeout 1200 python -m pytest tests/test_gpu_cusparse.py -x -q > gpurun_out/pytest42.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest42.log
timeout 900 python bench.py > gpurun_out/bench42.json 2> gpurun_out/bench42.err
