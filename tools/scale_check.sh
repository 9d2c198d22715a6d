#!/usr/bin/env bash
# Multi-GPU check for a box with >= 2 GPUs (not runnable in this round's one-GPU sandbox):
# C5 DP strong scaling at N = 1, 2, 4, 8 with every transport of the dist path, one JSON line per run
# under gpurun_out/scale/.  N = 1 is the single-GPU bench; efficiency = value_N / (N * value_1).
set -u
mkdir -p gpurun_out/scale
NG=$(python -c "import torch; print(torch.cuda.device_count())")
timeout 900 python bench.py --steps 100 --warmup 5 --no-compare --no-per-config > gpurun_out/scale/n1.json 2> gpurun_out/scale/n1.err
for N in 2 4 8; do
  [ "$N" -le "$NG" ] || continue
  # bench.py --gpus N launches its own N ranks (torchrun) and times the other transports as legs
  for TR in nccl direct; do
    timeout 1200 python bench.py --gpus "$N" --steps 100 --warmup 5 --transport "$TR" \
      > "gpurun_out/scale/n${N}_${TR}.json" 2> "gpurun_out/scale/n${N}_${TR}.err"
    echo "N=$N transport=$TR rc=$?"
  done
done
python - <<'PY'
import glob, json, os
v1 = json.loads(open("gpurun_out/scale/n1.json").read().strip().splitlines()[-1])["value"]
for f in sorted(glob.glob("gpurun_out/scale/n[248]_*.json")):
    t = open(f).read().strip()
    if not t:
        print(os.path.basename(f), "no output"); continue
    d = json.loads(t.splitlines()[-1])
    print(os.path.basename(f), d["value"], "GF/s", "eff", round(d["value"] / (d["n_gpus"] * v1), 3))
PY
