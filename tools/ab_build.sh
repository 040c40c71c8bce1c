#!/bin/bash
# A/B of compile-time variants on the bench's mid window (t = 5e-4) and a late
# window (t = 0.002), 200 steps of configs[1] each, two runs per variant:
#   tools/ab_build.sh "label1=flags1" "label2=flags2" ...   ("default=" for none)
# Each variant rebuilds the library in place; the default build is restored last.
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-postproc --no-late --no-e2e --no-first-order"
for spec in "$@"; do
  label=${spec%%=*}; flags=${spec#*=}
  VLBM_NVCC_EXTRA="$flags" python -m paper_2605_25282_b200.build -f > /dev/null || { echo "$label: build failed"; continue; }
  for r in 1 2; do
    for w in mid late; do
      ts=0.0005; [ $w = late ] && ts=0.002
      $B --t-start $ts > gpurun_out/ab_${label}_${w}_r$r.json 2>> gpurun_out/ab_build.err
      python -c "
import json; d = json.load(open('gpurun_out/ab_${label}_${w}_r$r.json'))
print('$label $w r$r', 'value %.3f G/s' % d['glups'], {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items() if k != 'note'})"
    done
  done
done
python -m paper_2605_25282_b200.build -f > /dev/null
