"""BASELINE configs[2] on one B200: one GPU's shard of the production march --
the jet at 4000x800 (3.2 M cells), 125 samples (1000 / 8 GPUs), run_sample's
loop (solver.hpp:625-669) through the reference config's snapshot times
{0, 7.5e-4, 1.5e-3, 2.25e-3, 3e-3} (config.hpp:37) to t = 0.003.

    python tools/c3_shard.py [samples] [m0] > profiles/r2_c3_shard.jsonl

One JSON line per snapshot interval: sample-cell updates and device time of
the interval (CUDA events on the batch stream), hence the throughput of that
stretch of the run (the last interval, t in [2.25e-3, 3e-3], is the late
regime where ~28 % of the cells are limiter hard cells); step counts,
diverged samples, the limiter-queue statistics (serial sample groups,
capacity, overflows -- must be 0) and the SHA-256 of sample 0's snapshot.
The 128 GB of state is far larger than L2.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_25282_b200 as v  # noqa: E402

TIMES = [0.0, 0.00075, 0.0015, 0.00225, 0.003]


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 125
    m0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    g = v.Grid(4000, 800)
    torch.cuda.init()
    t0 = time.perf_counter()
    sim = v.BatchSimulation.jet(g, n_samples=S, base_seed=42, m0=m0)
    st = torch.cuda.ExternalStream(sim.stream())
    print(json.dumps({"what": "configs[2] shard", "grid": "4000x800", "samples": S, "m0": m0,
                      "create_s": round(time.perf_counter() - t0, 2),
                      "queues": sim.queue_stats(),
                      "device_mem_gb": round(torch.cuda.mem_get_info()[1] / 1e9, 1),
                      "free_gb_after_create": round(torch.cuda.mem_get_info()[0] / 1e9, 1)}),
          flush=True)
    prev_upd = 0
    total_ms = 0.0
    for t in TIMES:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record(st)
        sim.run_to(t)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        total_ms += ms
        tt, steps, status = sim.scalars()
        upd = int(steps.sum()) * g.cells()
        d = upd - prev_upd
        prev_upd = upd
        u0 = np.array(sim.state(0), dtype="<f8")
        print(json.dumps({
            "t": t, "interval_updates": d, "interval_ms": ms,
            "interval_wall_s": round(time.perf_counter() - w0, 2),
            "interval_rate": d / (ms * 1e-3) if ms > 0 else None,
            "steps_min": int(steps.min()), "steps_max": int(steps.max()),
            "diverged": int((status == 2).sum()),
            "queues": sim.queue_stats(),
            "sample0_sha256": hashlib.sha256(u0.tobytes()).hexdigest()}), flush=True)
    print(json.dumps({"total_updates": prev_upd, "total_device_s": total_ms / 1e3,
                      "mean_rate": prev_upd / (total_ms * 1e-3),
                      "wall_s": round(time.perf_counter() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
