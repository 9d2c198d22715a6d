python tools/kbench.py --configs C3,C5,C2 --fmts pjds32s,pjds32 --dtypes f64 --policies 1x2,1x0,0x0,1x1,3x2,0x2,1x3 > gpurun_out/kbench6.jsonl 2> gpurun_out/kbench6.err
tail -3 gpurun_out/kbench6.err
