#!/bin/bash
# Round evidence (tag = $1, default r2) on one B200 (run under gpurun from the repo root):
#   1. the default bench line                       -> gpurun_out/${TAG}_bench.json
#   2. ncu launch list of the timed region           -> gpurun_out/${TAG}_launches.csv
#   3. ncu --set full of each march kernel at t=5e-4 (mid bench window, one
#      sample group) and of the W1/L1 post-processing kernels (configs[3])
#                                                    -> gpurun_out/${TAG}_<kernel>.ncu-rep
# tools/summarize_profiles.py turns these into profiles/${TAG}_*.
TAG=${1:-r2}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
B="python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-postproc --no-e2e --no-roofline --no-late"
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include timed/ -c 600 \
    --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include timed/ -c 600 \
    --csv --log-file gpurun_out/${TAG}_launches_late.csv $B --t-start 0.002 > gpurun_out/${TAG}_launches_late.log 2>&1
for k in k_theta_tiled k_theta_hard k_bisect_cert k_bisect_unc k_bisect_tail k_advance_tiled k_sched; do
  VLBM_GROUPS=1 ncu --set full --import-source on --clock-control none -k regex:"$k" --nvtx \
      --nvtx-include timed/ -c 1 -o gpurun_out/${TAG}_$k -f $B --t-start 0.0005 \
      > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
for k in ${POST_KERNELS-k_w1_tile k_ordered_sum k_strong_partials}; do
  ncu --set full --import-source on --clock-control none -k regex:"$k" -s 1 -c 1 \
      -o gpurun_out/${TAG}_$k -f python tools/post_probe.py 1000 > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
ls -la gpurun_out/${TAG}_*
