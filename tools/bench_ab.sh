# Full default-window march bench (2000 steps from t=0), A/B over libraries:
# usage: bash tools/bench_ab.sh [lib.so ...]  ("" = the in-tree build)
for L in "" "$@"; do
  VLBM_LIB=$L python bench.py --no-cpu-baseline --no-postproc --no-e2e --no-roofline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${L:-base}', round(d['glups'],3), d['ms_per_step'])"
done
