# Lanczos with more per-warp partials than the update pass's CTAs; memcheck
mkdir -p gpurun_out
python -m pytest tests/test_lanczos.py -m gpu -q > gpurun_out/t67.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/t67.txt
compute-sanitizer --tool memcheck python -m pytest tests/test_lanczos.py -m gpu -q -k many_product > gpurun_out/t67_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/t67_memcheck.txt
tail -n 3 gpurun_out/t67.txt gpurun_out/t67_memcheck.txt
