# Lanczos: device span per step (CUPTI) vs wall time; per-kernel busy time
mkdir -p gpurun_out
python tools/lanczos_bench.py C3 200 > gpurun_out/lz58.jsonl 2> gpurun_out/lz58.err
python tools/lanczos_bench.py C5 50 >> gpurun_out/lz58.jsonl 2>> gpurun_out/lz58.err
tail -3 gpurun_out/lz58.err
