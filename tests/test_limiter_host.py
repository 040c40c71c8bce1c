"""The device limiter's arithmetic (csrc/rlmp.cuh, csrc/rlmp_replay.cuh) on the
CPU (-m "not gpu"): tests/cpp/bin/limiter_check compiles those headers for the
host (g++, no FMA contraction: the same IEEE operations nvcc --fmad=false
emits) and runs every limiter path of the kernels on per-cell limiter inputs
dumped by the C oracle over a late-time jet march (rlmp_theta,
solver.hpp:437-487).  Every path -- the plain 30-step bisection, the queued
certified bisection (replay off) and the replayed bisection with its tail --
must return the reference's theta bit for bit, the theta = 1 quadratic-form
decision of the vertex floors must never contradict the exact checks, and the audit (the full
feasible() re-run at every bisection step) must count zero disagreements.
The GPU tests (test_gpu_march.py) check the same paths end to end on device.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import make_grid, make_params, make_pert

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "bin", "limiter_check")


@pytest.fixture(scope="module")
def limiter_check():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp"), "limiter"], check=True)
    return BIN


@pytest.mark.parametrize("m,steps,every", [(0, 900, 150), (5, 600, 200)])
def test_limiter_paths_bit_exact(vo, limiter_check, tmp_path, m, steps, every):
    g = make_grid(200, 40)
    p = make_params()
    sim = vo.jet_sim(g, p, make_pert(), 42, m)
    recs = []
    for k in range(steps):
        dt = sim.suggest_dt()
        if k % every == every - 1:
            recs.append(sim.limiter_cells(g.x_max / g.nx / dt))  # a = dx / dt of this step
        sim.step(dt)
    path = tmp_path / "cells.bin"
    np.concatenate(recs).tofile(path)
    out = subprocess.run([limiter_check, str(path), repr(p.gamma)], check=True,
                         capture_output=True, text=True).stdout
    r = json.loads(out)
    assert r["cells"] == len(recs) * g.nx * g.ny
    assert r["bisections"] > 1000  # late-time march: the bisection paths are exercised
    assert r["replay_stopped"] > 0  # ... including the tail resumption
    # the quadratic form decides nearly every theta = 1 vertex check (both ways)
    assert r["quadform_pass"] > 0.9 * r["theta_one"] and r["quadform_fail"] > 0
    assert r["quadform_open"] < 0.02 * r["cells"]
    assert r["hypot_checks"] > 100000  # hypot_ref (conservative bound) == this host's libm
    # synthetic cells sitting on the pressure floor (both sides, jet-core cancellation,
    # non-finite and non-positive densities): decided both ways, never wrongly
    assert r["fuzz_pass"] > 50000 and r["fuzz_fail"] > 50000 and r["fuzz_open"] > 1000
    for k in ("fuzz_errors", "quadform_errors", "mismatch_plain", "mismatch_queued", "mismatch_replay",
              "audit_errors", "margin_errors", "hypot_errors"):
        assert r[k] == 0, (k, r)
