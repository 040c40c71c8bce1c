import sys
sys.path.insert(0, '.')
import paper_2605_25282_b200 as v
g = v.Grid(1000, 200)
sim = v.BatchSimulation.jet(g, n_samples=8, base_seed=42)
sim.set_audit(True)
prev = None
for t in (0.0001, 0.0003, 0.0005, 0.0008, 0.001):
    sim.run_to(t)
    c = sim.audit_counters()
    print(t, c, flush=True)
