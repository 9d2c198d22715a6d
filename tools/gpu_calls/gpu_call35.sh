# round-end style validation: GPU tests, smoke, default bench, f32 bench, reference arm
python -m pytest tests -m gpu -x -q > gpurun_out/gt35.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke35.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke35.log
python bench.py > gpurun_out/bench35.json 2> gpurun_out/bench35.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench35_ref.json 2>> gpurun_out/bench35.err
