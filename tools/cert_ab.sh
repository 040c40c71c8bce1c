#!/bin/bash
# Limiter certificate A/B on a late window of configs[1] (t = 0.002):
# default (warp hint: a warp tries the theta = 1 certificate while its hint
# is >= 2) vs every warp always trying (VLBM_CERT_TRY=0): audited path rates
# (tools/cert_probe.py) and the timed kernel split (bench.py late window).
mkdir -p gpurun_out
B="python bench.py --t-start 0.002 --steps 100 --no-cpu-baseline --no-postproc --no-late --no-e2e --no-first-order"
python tools/cert_probe.py 0.002 50 > gpurun_out/cert_default.json
$B > gpurun_out/late_default.json
VLBM_NVCC_EXTRA="-DVLBM_CERT_TRY=0" python -m paper_2605_25282_b200.build -f > /dev/null
python tools/cert_probe.py 0.002 50 > gpurun_out/cert_try0.json
$B > gpurun_out/late_try0.json
python -m paper_2605_25282_b200.build -f > /dev/null
for v in default try0; do
  python -c "
import json; c = json.load(open('gpurun_out/cert_$v.json')); d = json.load(open('gpurun_out/late_$v.json'))
print('$v', 'cert/cell %.3f diag_ok %.3f unc_feasible %.3f warps_vchk %.3f' % (c['vertex_certified_at_1'], c['diag_ok_at_1'], c['unc_feasible'], c['warps_with_vertex_checks_per_warp']),
      'value %.3f G/s' % d['glups'], {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items() if k != 'note'})"
done
# upper bound of any vertex-check optimisation: the tile pass with the theta = 1
# vertex checks skipped (timing only; the results are NOT the reference's)
VLBM_NVCC_EXTRA="-DVLBM_EXP_NOVERTEX=1" python -m paper_2605_25282_b200.build -f > /dev/null
$B > gpurun_out/late_novertex.json
python -m paper_2605_25282_b200.build -f > /dev/null
python -c "
import json; d = json.load(open('gpurun_out/late_novertex.json'))
print('novertex (timing only)', 'value %.3f G/s' % d['glups'], {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items() if k != 'note'})"
