# Full default-window march bench (2000 steps from t=0), A/B over libraries and
# sample-group counts:  bash tools/bench_ab.sh [lib.so ...]   ("" = in-tree build)
for L in "" "$@"; do for G in ${GROUPS_AB:-1}; do
  VLBM_GROUPS=$G VLBM_LIB=$L python bench.py --no-cpu-baseline --no-postproc --no-e2e --no-roofline --no-late 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${L:-base} G=$G', round(d['glups'],3), d['ms_per_step'])"
done; done
