"""Long-horizon golden digests from the REFERENCE itself (oracle/_ref, the
unmodified headers compiled by oracle/Makefile).  Run once in the container
that has /root/reference (about an hour on 7 cores):

    python tests/golden/make_golden_long.py

Writes tests/golden/golden_long.json:

* ``c2``: BASELINE configs[1] -- the jet at 1000x200, samples m = 0..63
  (base_seed 42), run_sample (solver.hpp:625-669) with snapshot times
  {0, 0.001}: per-sample digest of the t = 0.001 field, time and step count,
  plus the 64-sample ensemble_moments (metrics.hpp:148-177) at t = 0.001 --
  digests of the mean density plane and of (mean, std) of all components.
* ``t003``: the reference config's snapshot times {0, 7.5e-4, 1.5e-3,
  2.25e-3, 3e-3} (config.hpp:37) on 200x40 (m = 0..7), 500x100 (m = 0..3)
  and 1000x200 (m = 0, 21, 42, 63): digests of every snapshot.

Per-task results are cached under /tmp/golden_long so an interrupted run
resumes.  Digests: SHA-256 of the raw little-endian float64 planes (NaNs
canonicalised), as in make_golden.py.
"""
from __future__ import annotations

import json
import os
import sys
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import digest, hexf  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_long.json")
CACHE = "/tmp/golden_long"
REF_TIMES = [0.0, 0.00075, 0.0015, 0.00225, 0.003]
C2_TIMES = [0.0, 0.001]
C2_SAMPLES = 64
T003 = {(200, 40): range(8), (500, 100): range(4), (1000, 200): (0, 21, 42, 63)}


def _task(args):
    kind, nx, ny, m, times = args
    path = os.path.join(CACHE, f"{kind}_{nx}x{ny}_{m}.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    from oracle.oracle import Oracle, make_grid, make_params, make_pert
    ref = Oracle("ref")
    r = ref.run_sample(make_grid(nx, ny), make_params(), make_pert(), 42, m, times)
    rec = {"kind": kind, "nx": nx, "ny": ny, "m": m, "steps": r["steps"],
           "admissible": r["admissible"], "diverged": [bool(d) for d in r["diverged"]],
           "times": [hexf(t) for t in r["time"]],
           "snapshots": [digest(f) for f in r["fields"]]}
    if kind == "c2":
        np.save(os.path.join(CACHE, f"c2_field_{m}.npy"), r["fields"][-1])
    with open(path + ".tmp", "w") as f:
        json.dump(rec, f)
    os.replace(path + ".tmp", path)
    print(f"done {kind} {nx}x{ny} m={m} steps={r['steps']}", flush=True)
    return rec


def main():
    from oracle import oracle
    oracle.build(ref=True)
    os.makedirs(CACHE, exist_ok=True)
    tasks = [("t003", 1000, 200, m, REF_TIMES) for m in T003[(1000, 200)]]
    tasks += [("c2", 1000, 200, m, C2_TIMES) for m in range(C2_SAMPLES)]
    tasks += [("t003", nx, ny, m, REF_TIMES) for (nx, ny), ms in T003.items() if nx < 1000
              for m in ms]
    nproc = int(os.environ.get("GOLDEN_PROCS", "7"))
    with Pool(nproc) as pool:
        recs = pool.map(_task, tasks, chunksize=1)
    G = {"generator": "oracle/_ref (unmodified reference headers), run_sample, base_seed 42",
         "ref_times": [hexf(t) for t in REF_TIMES], "c2_times": [hexf(t) for t in C2_TIMES],
         "c2": {"samples": {}}, "t003": {}}
    for r in recs:
        key = str(r["m"])
        if r["kind"] == "c2":
            G["c2"]["samples"][key] = r
        else:
            G["t003"].setdefault(f"{r['nx']}x{r['ny']}", {})[key] = r
    # the 64-sample ensemble mean at t = 0.001 (ensemble_moments, metrics.hpp:148-177)
    from oracle.oracle import Oracle
    x = np.stack([np.load(os.path.join(CACHE, f"c2_field_{m}.npy")) for m in range(C2_SAMPLES)])
    mean, sd = Oracle("ref").ensemble_moments(x)
    G["c2"]["mean_rho"] = digest(mean[0])
    G["c2"]["moments"] = digest(mean, sd)
    G["c2"]["mean_rho_sum"] = hexf(float(np.sum(mean[0])))
    with open(OUT, "w") as f:
        json.dump(G, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
