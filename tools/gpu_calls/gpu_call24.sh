nvidia-smi --query-gpu=name,serial,clocks.sm,clocks.mem,clocks.max.sm,clocks.max.mem,temperature.gpu,power.draw,ecc.mode.current --format=csv
python tools/kbench.py --configs C2,C3,C5 --fmts pjds32s --dtypes f64 --variants 0x0 --reps 100 > gpurun_out/kbench24.jsonl 2> gpurun_out/kbench24.err
python tools/kbench.py --configs C2,C3 --fmts pjds32s --dtypes f64 --variants 0x0 --reps 100 >> gpurun_out/kbench24.jsonl 2>> gpurun_out/kbench24.err
python -c "import paper_1112_5588_b200 as pj; print(pj.bw_probe(4<<30, 5))"
tail -2 gpurun_out/kbench24.err
