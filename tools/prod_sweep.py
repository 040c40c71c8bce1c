"""BASELINE configs[4]: the grid-convergence sweep at production scale on one
B200 -- the jet at 500x100, 1000x200, 2000x400 (levels 3; 4 adds 4000x800),
M samples each to t = 0.003 at the reference config's snapshot times, L1
and W1 Cauchy rates between consecutive levels computed on the device
(sweep.production_sweep: bit-identical to grid_sweep / compute_metrics).

    python tools/prod_sweep.py [M=1000] [levels=3] [batch=125] > profiles/r2_prod_sweep.json
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25282_b200 import sweep  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 3
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 125
times = [0.0, 0.00075, 0.0015, 0.00225, 0.003]
t0 = time.perf_counter()


def progress(done, total, label):
    print(json.dumps({"progress": done, "of": total, "level": label,
                      "wall_s": round(time.perf_counter() - t0, 1)}), file=sys.stderr, flush=True)


rep = sweep.production_sweep(torch, 500, 100, levels, M, times, base_seed=42, batch=batch,
                             progress=progress)
upd = {lab: int(st.sum()) * int(lab.split("x")[0]) * int(lab.split("x")[1])
       for lab, st in rep.steps.items()}
out = {"what": "configs[4] production sweep", "M": M, "levels": list(rep.steps),
       "batch": batch, "times": times,
       "rows": [r.__dict__ for r in rep.rows], "rates": [r.__dict__ for r in rep.rates],
       "steps_min_max": {k: [int(v.min()), int(v.max())] for k, v in rep.steps.items()},
       "sample_cell_updates": upd, "march_seconds": rep.march_seconds,
       "march_rate": {k: upd[k] / rep.march_seconds[k] for k in upd},
       "metrics_seconds": rep.metrics_seconds, "wall_s": round(time.perf_counter() - t0, 1)}
print(json.dumps(out, indent=1))
