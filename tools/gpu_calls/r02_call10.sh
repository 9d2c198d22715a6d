# round 2, call 10: CTA size A/B (256 default vs 128 vs 64 threads per CTA), all configs, same box
set -x
for T in 256 128 64 256; do
  PJDS_NVCC_DEFINES="-DPJDS_CTA_THREADS=$T" python -c "import build_native; build_native.build_pjds(force=True)" > /dev/null 2>&1
  python tools/kbench.py --configs C2,C4,C3,C5 --dtypes f64,f32 --fmts pjds32s,pjds32 --reps 40 > gpurun_out/r02c10_cta$T.jsonl 2>&1
  mv gpurun_out/r02c10_cta$T.jsonl gpurun_out/r02c10_cta${T}_$(date +%s).jsonl
done
