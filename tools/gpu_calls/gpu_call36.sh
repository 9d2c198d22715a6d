# bench lines for the other configs with the current defaults (b_r = 32)
python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/b36_C5_f32.json 2> gpurun_out/b36.err
for c in C3 C2 C4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/b36_${c}_f64.json 2>> gpurun_out/b36.err; done
