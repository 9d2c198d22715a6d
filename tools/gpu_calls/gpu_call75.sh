# y-store knob: every setting and variant bitwise = the FMA chain
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "y_store" > gpurun_out/t75.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/t75.txt
tail -n 3 gpurun_out/t75.txt
