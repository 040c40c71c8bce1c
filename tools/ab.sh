# A/B timing of the march at early (t=0) and late (t=0.002) time, G=1 (kernel ms per step).
for t in 0 0.002; do
VLBM_GROUPS=1 python bench.py --steps 300 --warmup 5 --t-start $t --no-cpu-baseline --no-postproc --no-e2e --no-roofline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('t$t', round(d['glups'],3), {k:round(v,3) for k,v in d['kernel_ms_per_step'].items() if k != 'note'})"
done
