"""Generates tests/golden/golden.json from the REFERENCE itself (oracle/_ref:
the unmodified headers of /root/reference/proj/include compiled by
oracle/Makefile).  Run in the container that has /root/reference:

    python tests/golden/make_golden.py

Bit-exact fixtures are stored as SHA-256 digests of the raw little-endian
float64 bytes (fields in the .vlbm plane layout of include/vlbm_b200.h) and
as float.hex() strings for scalars, so a test can demand bit identity.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402
from oracle.oracle import (INLET, OUTFLOW, PERIODIC, WALL, FIRST_ORDER, SECOND_ORDER, RLMP,  # noqa: E402
                           make_grid, make_params, make_pert)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def digest(*arrays) -> str:
    """SHA-256 of the raw float64 bytes, NaNs canonicalised (NaN payload and
    sign bits are not reproducible across compilers and are not compared)."""
    h = hashlib.sha256()
    for a in arrays:
        a = np.array(a, dtype="<f8")
        a[np.isnan(a)] = np.nan
        h.update(a.tobytes())
    return h.hexdigest()


def hexf(x: float) -> str:
    return float(x).hex()


def smooth_field(nx, ny, x_max, gamma=1.4):
    """test_solver.cpp:31-48's smooth periodic field, plus a spike."""
    dx = x_max / nx
    x = (np.arange(nx) + 0.5) * dx
    y = -0.25 + (np.arange(ny) + 0.5) * dx
    X, Y = np.meshgrid(x, y)
    rho = 1.0 + 0.3 * np.sin(2 * np.pi * X / x_max) * np.cos(2 * np.pi * (Y + 0.25) / 0.5)
    v1 = 0.2 * np.cos(2 * np.pi * X / x_max)
    v2 = 0.1 * np.sin(2 * np.pi * (Y + 0.25) / 0.5)
    p = 1.0 + 0.2 * np.cos(2 * np.pi * X / x_max)
    E = p / (gamma - 1.0) + 0.5 * rho * (v1 * v1 + v2 * v2)
    f = np.stack([rho, rho * v1, rho * v2, E])
    f[0, ny // 2, nx // 3] *= 3.0
    f[3, ny // 2, nx // 3] *= 3.0
    return np.ascontiguousarray(f)


BC_CASES = {
    "all_periodic": ((PERIODIC, PERIODIC, PERIODIC, PERIODIC), 32, 32),
    "periodic_x_wall_y": ((PERIODIC, PERIODIC, WALL, WALL), 32, 16),
    "outflow_x_periodic_y": ((OUTFLOW, OUTFLOW, PERIODIC, PERIODIC), 40, 8),
    "outflow_x_wall_y": ((OUTFLOW, OUTFLOW, WALL, WALL), 24, 12),
}

STEPS_C1 = (1, 10, 50, 200)


def metrics_inputs(seed, M, ny, nx):
    rng = np.random.default_rng(seed)
    a = rng.lognormal(-0.125, 0.5, size=(M, 4, ny, nx))
    b = rng.lognormal(-0.125, 0.5, size=(M, 4, ny, nx))
    a[:, 1:3] = rng.normal(size=(M, 2, ny, nx))
    b[:, 1:3] = rng.normal(size=(M, 2, ny, nx))
    return a, b


def main():
    oracle.build(ref=True)
    ref = oracle.Oracle("ref")
    G = {"generator": "oracle/_ref (unmodified reference headers)", "ic": {}, "c1": {},
         "bc": {}, "run_sample": {}, "metrics": {}}

    # IC: draw_coefficients (perturbation.hpp:42-54) and inlet rows
    pp = make_pert()
    for base, m in [(42, 0), (42, 1), (42, 7), (42, 63), (1, 0), (99, 123), (7, 5)]:
        seed, y, z = ref.draw_coefficients(base, m, 10)
        rows = ref.inlet_rows(make_grid(200, 40), y, z, pp)
        init = ref.initial_field(make_grid(200, 40), y, z, pp, strip=0.02)
        G["ic"][f"{base}:{m}"] = {"seed": str(seed), "y": [hexf(v) for v in y],
                                  "z": [hexf(v) for v in z], "inlet_rows_200x40": digest(rows),
                                  "initial_field_200x40": digest(init)}

    # C1: 200x40, M=8, step(suggest_dt()) x 200, digests of u+pops after selected steps
    g = make_grid(200, 40)
    for m in range(8):
        s = ref.jet_sim(g, make_params(), pp, 42, m)
        rec = {}
        done = 0
        for k in STEPS_C1:
            while done < k:
                s.step(s.suggest_dt())
                done += 1
            u, p = s.get(pops=True)
            rec[str(k)] = {"state": digest(u, p), "time": hexf(s.time)}
        G["c1"][str(m)] = rec

    # Boundary variants x limiters: 20 steps of step(suggest_dt())
    for name, (bc, nx, ny) in BC_CASES.items():
        for lim in (RLMP, FIRST_ORDER, SECOND_ORDER):
            x_max = 0.5 * nx / ny
            init = smooth_field(nx, ny, x_max)
            s = ref.sim(make_grid(nx, ny, x_max), make_params(gamma=1.4, limiter=lim, bc=bc), init)
            for _ in range(20):
                s.step(s.suggest_dt())
            u, p = s.get(pops=True)
            G["bc"][f"{name}:{lim}"] = {"state": digest(u, p), "time": hexf(s.time),
                                         "init": digest(init)}

    # run_sample on the smoke grid 125x25, samples 0..2, reference snapshot times
    times = [0.0, 0.00075, 0.0015, 0.00225, 0.003]
    for m in range(3):
        r = ref.run_sample(make_grid(125, 25), make_params(), pp, 42, m, times)
        G["run_sample"][str(m)] = {"steps": r["steps"], "admissible": r["admissible"],
                                   "seed": str(r["seed"]),
                                   "times": [hexf(t) for t in r["time"]],
                                   "snapshots": [digest(f) for f in r["fields"]]}

    # metrics on seeded synthetic ensembles
    for (seed, M, ny, nx) in [(1, 1, 4, 4), (2, 7, 6, 8), (3, 64, 10, 12), (4, 1000, 2, 4)]:
        a, b = metrics_inputs(seed, M, ny, nx)
        es, pc = ref.strong_error(a, b)
        w1 = [ref.wasserstein1(a, b, var) for var in range(4)]
        rec = {"M": M, "ny": ny, "nx": nx, "strong": hexf(es), "strong_pc": [hexf(v) for v in pc],
               "w1": [hexf(v) for v in w1], "restrict0": digest(ref.restrict_field(a[0]))}
        if M >= 2:
            mean, sd = ref.ensemble_moments(a)
            rec["moments"] = digest(mean, sd)
        G["metrics"][f"{seed}"] = rec

    with open(OUT, "w") as f:
        json.dump(G, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
