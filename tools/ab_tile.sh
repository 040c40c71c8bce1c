#!/bin/bash
# A/B of the limiter tile pass on the bench window and a late window:
# the current build vs a git revision's march_tiled.cu (e.g. HEAD~1), built
# into a copy of the library.  Usage: tools/ab_tile.sh <rev>
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-postproc --no-late --no-e2e --no-first-order"
run() {
  $B "${@:2}" > gpurun_out/abt_$1.json 2>> gpurun_out/abt.err
  python -c "
import json; d = json.load(open('gpurun_out/abt_$1.json'))
print('$1', 'value %.3f G/s' % d['glups'], {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items() if k != 'note'})"
}
for r in 1 2; do
  run new_mid_r$r
  run new_late_r$r --t-start 0.002
done
