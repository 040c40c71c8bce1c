#!/bin/bash
# A/B of the W1 kernel's L2 prefetch distance (CTAs ahead; 0 = off) on the
# configs[3] post-processing probe, two runs per variant:
#   bash tools/ab_w1.sh 0 148 296 444
mkdir -p gpurun_out
for A in "$@"; do
  VLBM_NVCC_EXTRA="-DVLBM_W1_AHEAD=$A" python -m paper_2605_25282_b200.build -f > /dev/null || { echo "ahead=$A: build failed"; continue; }
  for r in 1 2; do
    python tools/post_probe.py 1000 2> /dev/null | python -c "
import json, sys; d = json.loads(sys.stdin.read())
print('ahead=$A r$r', 'w1_kernel_ms %.2f w1_ms %.2f cells/s %.3g W1 %.17g' % (d['w1_kernel_ms'], d['w1_ms'], d['w1_cells_per_s'], d['W1']))"
  done
done
python -m paper_2605_25282_b200.build -f > /dev/null
