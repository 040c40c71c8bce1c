#!/bin/bash
# ncu --set full captures of the march kernels at late time (t = 0.002, C2, 64 samples, G=1).
set -x
mkdir -p gpurun_out
export VLBM_GROUPS=1
B="python bench.py --steps 20 --warmup 3 --t-start 0.002 --no-cpu-baseline --no-postproc --no-e2e --no-roofline"
for k in k_theta_tiled k_theta_hard k_bisect_unc k_bisect_cert k_bisect_tail k_advance_tiled; do
  ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 3000 -c 1 \
      -o gpurun_out/late_$k -f $B > gpurun_out/ncu_late_$k.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 12000 -c 400 --csv \
    --log-file gpurun_out/launches_late2.csv $B > gpurun_out/ncu_late_list.log 2>&1
