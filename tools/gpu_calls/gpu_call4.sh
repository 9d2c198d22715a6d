python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/kbench.py --fmts pjds32,pjds32s --variants 2x4,2x20,4x2,4x18,4x4,4x20 > gpurun_out/kbench3.jsonl 2> gpurun_out/kbench3.err
tail -3 gpurun_out/kbench3.err
