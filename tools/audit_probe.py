"""Limiter statistics over a C2 march (audit mode): per-step cell counts of
each limiter path, the quadratic form's decision rate at theta = 1, and the disagreement count (must
be 0).  Run on a GPU box: python tools/audit_probe.py"""
import sys
sys.path.insert(0, '.')
import paper_2605_25282_b200 as v

S = 8
g = v.Grid(1000, 200)
sim = v.BatchSimulation.jet(g, n_samples=S, base_seed=42)
sim.set_audit(True)
prev, prev_steps = None, 0
for t in (0.0002, 0.0005, 0.001, 0.0015, 0.002, 0.0025):
    sim.run_to(t)
    c = sim.audit_counters()
    steps = int(sim.scalars()[1].sum())
    d = c if prev is None else {k: (c[k] - prev[k]) % (1 << 32) for k in c}
    n = max(steps - prev_steps, 1)  # sample-steps in this interval
    prev, prev_steps = c, steps
    cells = n * g.cells()
    per = lambda k: d[k] / n
    print(f"t={t}: mismatches={c['mismatches']} per sample-step of {g.cells()} cells: "
          f"diag_ok={per('diag_ok_at_1'):.0f} decided_by_form={per('vertex_decided_at_1'):.0f} open={per('vertex_open_at_1'):.0f} "
          f"feasible={per('feasible_at_1'):.0f} bisections={per('bisections'):.0f} "
          f"uncertified={per('uncertified'):.0f} unc_vertices_start={per('unc_vertices_start'):.0f} "
          f"vertex_evals={per('vertex_evals'):.0f}", flush=True)
