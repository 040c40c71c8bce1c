"""Limiter certificate statistics on a late window of configs[1]'s grid
(GPU box): march 1000x200 x 64 samples to T (default 0.002) without audit,
then audit N steps and print per-cell rates of the limiter paths.
    python tools/cert_probe.py [T] [N]"""
import json
import sys

sys.path.insert(0, ".")
import paper_2605_25282_b200 as v  # noqa: E402

T = float(sys.argv[1]) if len(sys.argv) > 1 else 0.002
N = int(sys.argv[2]) if len(sys.argv) > 2 else 100
g = v.Grid(1000, 200)
sim = v.BatchSimulation.jet(g, n_samples=64, base_seed=42)
sim.run_to(T)
sim.set_audit(True)
sim.step(N)
a = sim.audit_counters()
cells = 64 * N * g.cells()
print(json.dumps({"T": T, "steps": N, **{k: a[k] / cells for k in a if k != "mismatches"},
                  "warps_with_vertex_checks_per_warp": a["warps_with_vertex_checks"] / (cells / 32),
                  "mismatches": a["mismatches"]}))
