"""Limiter-certificate audit over a whole production horizon (run on a GPU box).

    python tools/audit_long.py c2   # configs[1] grid: 1000x200, 64 samples, to t = 0.003
    python tools/audit_long.py c3   # a configs[2] shard: 4000x800, 16 samples, to t = 0.003

With the audit on (vlbm_batch_set_audit) every decision the limiter takes
from a certificate instead of an exact evaluation -- the theta = 1 vertex
certificate, each certified bisection step and each replayed bisection step
(rlmp.cuh, rlmp_replay.cuh) -- is re-checked with the reference's full
16-check feasible() on the GPU, and disagreements are counted (counter 0,
must stay 0).  The march runs run_sample's loop through the reference
config's snapshot times (config.hpp:37); at each time one JSON line reports
the cumulative counters, the limiter-queue statistics and the wall time.  For
c2 the snapshots of samples 0, 21, 42, 63 are also hashed (they must equal
tests/golden/golden_long.json, i.e. the reference's own run_sample).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_25282_b200 as v  # noqa: E402

TIMES = [0.0, 0.00075, 0.0015, 0.00225, 0.003]


def digest(a) -> str:
    a = np.array(a, dtype="<f8")
    a[np.isnan(a)] = np.nan
    return hashlib.sha256(a.tobytes()).hexdigest()


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "c2"
    nx, ny, S = (1000, 200, 64) if case == "c2" else (4000, 800, 16)
    if len(sys.argv) > 2:
        S = int(sys.argv[2])
    g = v.Grid(nx, ny)
    golden = None
    gpath = os.path.join(ROOT, "tests", "golden", "golden_long.json")
    if case == "c2" and os.path.exists(gpath):
        with open(gpath) as f:
            golden = json.load(f)["t003"]["1000x200"]
    t0 = time.perf_counter()
    sim = v.BatchSimulation.jet(g, n_samples=S, base_seed=42)
    sim.set_audit(True)
    ok = True
    for k, t in enumerate(TIMES):
        sim.run_to(t)
        tt, steps, status = sim.scalars()
        line = {"case": case, "grid": f"{nx}x{ny}", "samples": S, "t": t,
                "wall_s": round(time.perf_counter() - t0, 2),
                "steps_min": int(steps.min()), "steps_max": int(steps.max()),
                "sample_cell_updates": int(steps.sum()) * nx * ny,
                "diverged": int((status == 2).sum()),
                "audit": sim.audit_counters(), "queues": sim.queue_stats()}
        if golden:
            match = {}
            for m in (0, 21, 42, 63):
                if m < S:
                    d = digest(sim.state(m))
                    match[m] = d == golden[str(m)]["snapshots"][k]
                    ok &= match[m]
            line["snapshot_matches_reference"] = match
        ok &= line["audit"]["mismatches"] == 0
        print(json.dumps(line), flush=True)
    print(json.dumps({"case": case, "ok": bool(ok)}), flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
