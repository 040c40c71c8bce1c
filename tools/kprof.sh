#!/bin/bash
# Per-kernel device time (ncu gpu__time_duration, serialised launches) of 30
# late-time steps of the C2 march, summed by kernel; for A/B of kernel changes.
# usage: bash tools/kprof.sh [t_start] [tag]
T=${1:-0.002}; TAG=${2:-x}
mkdir -p gpurun_out
VLBM_GROUPS=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(theta|bisect|advance|sched)' \
  --nvtx --nvtx-include timed/ -c 180 --csv --log-file gpurun_out/kprof_$TAG.csv \
  python bench.py --steps 40 --warmup 3 --t-start $T --no-cpu-baseline --no-postproc --no-e2e --no-roofline > /dev/null 2>&1
python - "$TAG" <<'PY'
import csv, sys, collections
lines = open(f"gpurun_out/kprof_{sys.argv[1]}.csv").read().splitlines()
rows = list(csv.reader(lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(",", "")); u = r[ui]
    v = {"usecond": 1e-3, "nsecond": 1e-6, "ns": 1e-6, "us": 1e-3, "msecond": 1.0, "ms": 1.0}[u] * v
    name = r[ki].split("(")[0].split("<")[0].split("::")[-1]
    tot[name] += v; cnt[name] += 1
steps = max(cnt.values())
print(sys.argv[1], {k: round(tot[k] / cnt[k] * (cnt[k] / steps), 4) for k in sorted(tot)}, "ms/step over", steps, "launches")
PY
