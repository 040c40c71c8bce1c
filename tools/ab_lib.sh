#!/bin/bash
# A/B of prebuilt libraries on the bench's mid (t = 5e-4) and late (t = 0.002)
# windows, 200 steps of configs[1] each, two runs per library:
#   tools/ab_lib.sh label1=path1.so label2=path2.so ...   (empty path = the in-tree build)
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-postproc --no-late --no-e2e --no-first-order"
for r in 1 2; do
  for spec in "$@"; do
    label=${spec%%=*}; lib=${spec#*=}
    for w in mid late; do
      ts=0.0005; [ $w = late ] && ts=0.002
      VLBM_LIB=$lib $B --t-start $ts > gpurun_out/abl_${label}_${w}_r$r.json 2>> gpurun_out/ab_lib.err
      python -c "
import json; d = json.load(open('gpurun_out/abl_${label}_${w}_r$r.json'))
print('$label $w r$r', 'value %.3f G/s' % d['glups'], {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items() if k != 'note'})"
    done
  done
done
