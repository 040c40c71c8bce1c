#!/bin/bash
# A/B of the advance kernels on the bench window (C2, t = 0.0005, 200 steps):
# k_advance_v2 (default) vs k_advance_tiled (VLBM_ADV=1), 2 runs each.
mkdir -p gpurun_out
for r in 1 2; do
  for v in 2 1; do
    VLBM_ADV=$v python bench.py --no-cpu-baseline --no-postproc --no-late --no-e2e \
      > gpurun_out/ab_adv_v${v}_r${r}.json 2>> gpurun_out/ab_adv.err
    python - "$v" "$r" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/ab_adv_v{sys.argv[1]}_r{sys.argv[2]}.json"))
k = d["kernel_ms_per_step"]
print(f"adv v{sys.argv[1]} run {sys.argv[2]}: value {d['glups']:.3f} G/s advance {k['ms_advance']:.4f} ms "
      f"frac {d['roofline']['frac']:.3f}  FO {d['first_order']['value']/1e9:.2f} G/s "
      f"FO adv {d['first_order']['advance_ms']:.4f} ms frac {d['first_order']['roofline']['frac']:.3f}")
PY
  done
done
