# NEXT-2 sigma windows on the long-row matrices (DLR1-, DLR2-, UHBR-shaped): does a narrower jagged-column stride help?
timeout 1500 python tools/kbench.py --configs C4,W4,W5 --dtypes f64,f32 --fmts pjds32,pjds32s --sigmas 0,1024,4096,16384,65536,0 --reps 40 > gpurun_out/kbench54.jsonl 2> gpurun_out/kbench54.err
