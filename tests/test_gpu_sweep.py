"""BASELINE configs[4] on the device (paper_2605_25282_b200.sweep.grid_sweep):
march every grid level, keep the snapshots in GPU memory, then per
consecutive pair and time the joint validity, W1 and E_strong, and per time
the fitted rates -- against the reference itself (oracle/_ref: run_sample per
sample and grid, restrict_field, wasserstein1, strong_error, fit_rate),
bit for bit."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import make_grid, make_params, make_pert  # noqa: E402

def bits(x):
    return np.float64(x).view(np.uint64)


@pytest.mark.gpu
def test_grid_sweep_matches_reference_compute_metrics(vlbm, ref):
    from paper_2605_25282_b200 import sweep
    nx0, ny0, levels, M = 60, 12, 3, 6
    times = [0.0, 3e-4, 6e-4]
    rep = sweep.grid_sweep(torch, nx0, ny0, levels, M, times, base_seed=42)
    p, pp = make_params(), make_pert()
    runs = []
    for l in range(levels):
        g = make_grid(nx0 << l, ny0 << l)
        runs.append([ref.run_sample(g, p, pp, 42, m, times) for m in range(M)])
    for l in range(levels):
        assert [r["steps"] for r in runs[l]] == list(rep.steps[f"{nx0 << l}x{ny0 << l}"])
    rows = iter(rep.rows)
    w1s, ess = {}, {}
    for pi in range(levels - 1):
        mask = [runs[pi][m]["admissible"] and runs[pi + 1][m]["admissible"] for m in range(M)]
        keep = [m for m in range(M) if mask[m]]
        for ti, t in enumerate(times):
            A = np.stack([runs[pi][m]["fields"][ti] for m in keep])
            B = np.stack([ref.restrict_field(runs[pi + 1][m]["fields"][ti]) for m in keep])
            w1 = ref.wasserstein1(A, B, 0)
            es = ref.strong_error(A, B)[0]
            row = next(rows)
            assert row.pair == f"{nx0 << pi}->{nx0 << (pi + 1)}" and row.time == t
            assert row.m_star == len(keep)
            assert bits(row.w1) == bits(w1) and bits(row.e_strong) == bits(es), (pi, ti)
            w1s[pi, ti], ess[pi, ti] = w1, es
    dxs = [make_grid(nx0 << l, ny0 << l).x_max / (nx0 << l) for l in range(levels - 1)]
    for ti, rr in enumerate(rep.rates):
        for got, errs in ((rr.r_w1, w1s), (rr.r_strong, ess)):
            e = [errs[pi, ti] for pi in range(levels - 1)]
            want = ref.fit_rate(e, dxs) if all(x > 0 for x in e) else float("nan")
            assert (np.isnan(got) and np.isnan(want)) or bits(got) == bits(want), (ti, got, want)


@pytest.mark.parametrize("n", [2, 3, 4])
def test_fit_rate_restatement_bitwise(ref, n):
    """sweep.fit_rate (host scalars) == the reference's fit_rate bit for bit."""
    from paper_2605_25282_b200 import sweep
    rng = np.random.default_rng(n)
    for _ in range(200):
        e = list(rng.lognormal(-3.0, 1.0, size=n))
        dx = sorted(rng.uniform(1e-4, 1e-1, size=n), reverse=True)
        assert bits(sweep.fit_rate(e, dx)) == bits(ref.fit_rate(e, dx))



def _sweep_worker(rank, world, port, q):
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_25282_b200 import sweep
    rep = sweep.grid_sweep(torch, 40, 8, 3, 5, [0.0, 2e-4, 4e-4], base_seed=11, dist=dist)
    if rank == 0:
        q.put([(r.pair, r.time, r.m_star, float(r.w1).hex(), float(r.e_strong).hex())
               for r in rep.rows] + [(float(r.r_w1).hex(), float(r.r_strong).hex())
                                     for r in rep.rates] + [rep.steps["160x32"].tolist()])
    dist.destroy_process_group()


@pytest.mark.gpu
def test_grid_sweep_sharded_equals_single_process():
    """grid_sweep with the samples sharded over 2 processes (sharing the one
    GPU: real CUDA-IPC peer mappings, gloo for the host exchange) gives rank 0
    the single-process report bit for bit."""
    import socket
    import torch.multiprocessing as mp
    from paper_2605_25282_b200 import sweep
    rep = sweep.grid_sweep(torch, 40, 8, 3, 5, [0.0, 2e-4, 4e-4], base_seed=11)
    want = [(r.pair, r.time, r.m_star, float(r.w1).hex(), float(r.e_strong).hex())
            for r in rep.rows] + [(float(r.r_w1).hex(), float(r.r_strong).hex())
                                  for r in rep.rates] + [rep.steps["160x32"].tolist()]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [2, 4, 6])
def test_production_sweep_equals_grid_sweep(vlbm, batch):
    """The production sweep (sample-batch major, only the W1 planes and the
    strong_error partials kept) gives grid_sweep's rows, rates and step
    counts bit for bit -- grid_sweep being pinned to the reference's
    run_sample + compute_metrics above -- for several batch splits."""
    from paper_2605_25282_b200 import sweep
    nx0, ny0, levels, M = 60, 12, 3, 6
    times = [0.0, 3e-4, 6e-4]
    want = sweep.grid_sweep(torch, nx0, ny0, levels, M, times, base_seed=42)
    got = sweep.production_sweep(torch, nx0, ny0, levels, M, times, base_seed=42, batch=batch)
    assert len(got.rows) == len(want.rows)
    for a, b in zip(got.rows, want.rows):
        assert (a.time, a.pair, a.m_star) == (b.time, b.pair, b.m_star)
        assert bits(a.w1) == bits(b.w1) and bits(a.e_strong) == bits(b.e_strong), (a, b)
    for a, b in zip(got.rates, want.rates):
        for x, y in ((a.r_w1, b.r_w1), (a.r_strong, b.r_strong)):
            assert (np.isnan(x) and np.isnan(y)) or bits(x) == bits(y)
    for lab in want.steps:
        assert list(got.steps[lab]) == list(want.steps[lab])
