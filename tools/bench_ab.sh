# Full default-window march bench (2000 steps from t=0), A/B by env var prefix.
for cfg in "VLBM_CERT1=1" "VLBM_CERT1=0"; do
  env $cfg python bench.py --no-cpu-baseline --no-postproc --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['glups'],3), d['ms_per_step'])"
done
