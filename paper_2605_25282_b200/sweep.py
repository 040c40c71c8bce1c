"""Grid-convergence sweep on the device (BASELINE configs[4]): the pipeline of
``vlbm run`` + ``vlbm metrics`` (run_ensemble, ensemble.hpp:235-342, then
compute_metrics, metrics.hpp:259-327) with the snapshots kept in GPU memory
instead of .vlbm files.

Every grid level marches the same M samples (one batch per level, or batches
of ``batch`` samples) to each snapshot time; the dense fields are copied
device-to-device into the level's snapshot store.  For every consecutive
pair and time: the joint validity mask (admissible on both grids,
ensemble.hpp:75-109), W1 of the metric variable with the restriction fused
(post.w1_cell_terms + ordered_mean) and E_strong from the per-sample
partials (vlbm_d_strong_partials) -- bit-identical to compute_metrics on the
reference's files.  Then the per-time rate fits (fit_rate, metrics.hpp:
180-219), restated here in the reference's operation order (host scalars).

torch provides the device buffers; every number comes from the CUDA library.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import post
from .vlbm import (BatchSimulation, GasParams, Grid, LatticeParams, PerturbationParams,
                   _check, lib)


@dataclass
class MetricsRow:  # metrics.hpp:237-243
    time: float
    pair: str
    m_star: int
    w1: float
    e_strong: float


@dataclass
class RateRow:  # metrics.hpp:245-249
    time: float
    r_w1: float
    r_strong: float


@dataclass
class SweepReport:  # MetricsReport, metrics.hpp:251-254
    rows: list = field(default_factory=list)
    rates: list = field(default_factory=list)
    steps: dict = field(default_factory=dict)  # grid label -> per-sample step counts


def fit_slope(x: Sequence[float], y: Sequence[float]) -> float:
    """metrics.hpp:179-197, same operation order."""
    if len(x) != len(y) or len(x) < 2:
        raise ValueError("fit_slope: need at least two matching points")
    n = float(len(x))
    xm = ym = 0.0
    for a, b in zip(x, y):
        xm += a
        ym += b
    xm /= n
    ym /= n
    sxy = sxx = 0.0
    for a, b in zip(x, y):
        sxy += (a - xm) * (b - ym)
        sxx += (a - xm) * (a - xm)
    return sxy / sxx


def fit_rate(errors: Sequence[float], dxs: Sequence[float]) -> float:
    """metrics.hpp:201-216: log-log least-squares slope (libm log)."""
    if len(errors) != len(dxs) or len(errors) < 2:
        raise ValueError("fit_rate: need at least two matching points")
    lx, ly = [], []
    for i, (e, d) in enumerate(zip(errors, dxs)):
        if not e > 0.0:
            raise ValueError("fit_rate: errors must be positive")
        if i > 0 and d >= dxs[i - 1]:
            raise ValueError("fit_rate: dxs must be strictly decreasing")
        lx.append(math.log(d))
        ly.append(math.log(e))
    return fit_slope(lx, ly)


def _positive(u: np.ndarray, gamma: float) -> bool:
    """admissible() over a field (euler.hpp:103-106): finite, rho > 0, p > 0."""
    r, mx, my, e = u
    p = (gamma - 1.0) * (e - (0.5 * (mx * mx + my * my)) / r)
    return bool(np.all(np.isfinite(u)) and np.all(r > 0.0) and np.all(p > 0.0))


def grid_sweep(torch, nx0: int, ny0: int, levels: int, n_samples: int,
               times: Sequence[float], base_seed: int = 42,
               lattice: LatticeParams = LatticeParams(), gas: GasParams = GasParams(),
               pp: PerturbationParams = PerturbationParams(), strip_width: float = 0.02,
               metric_variable: int = 0, require_positivity: bool = False, m0: int = 0,
               batch: Optional[int] = None, device: int = 0, dist=None,
               group=None) -> Optional[SweepReport]:
    """Grids nx0 x ny0 * 2^l (l = 0..levels-1), M = n_samples samples each,
    snapshots at ``times``; returns the rows and rates compute_metrics would
    write (metrics.csv / rates.csv).

    With ``dist`` (torch.distributed, one process per GPU) the samples are
    sharded: rank r marches its contiguous share on every level
    with no communication; per pair and time the joint validity masks are
    gathered, W1 runs as dist.peer_wasserstein1 (each rank's kernel reads the
    other ranks' snapshots through CUDA-IPC peer mappings, no re-shard) and
    E_strong from the ranks' per-sample partials gathered in sample order.
    Rank 0 returns the report (bit-identical to one process); the other ranks
    return None."""
    if levels < 2:
        raise RuntimeError("metrics: need >= 2 grids for Cauchy errors")
    times = list(times)
    M_total = n_samples
    if dist is not None:
        from .dist import shard_range
        s0, M = shard_range(M_total, dist.get_world_size(group), dist.get_rank(group))
        m0 += s0
    else:
        M = M_total
    batch = batch or max(M, 1)
    dev = torch.device("cuda", device)
    grids = [Grid(nx0 << l, ny0 << l) for l in range(levels)]
    store, valid = [], []  # store[l][ti]: (M, 4, ny, nx) device tensor; valid[l]: bool (M,)
    rep = SweepReport()
    for g in grids:
        snaps = [torch.empty((M, 4, g.ny, g.nx), dtype=torch.float64, device=dev) for _ in times]
        ok = np.ones(M, bool)
        steps = np.zeros(M, np.int64)
        for b0 in range(0, M, batch):
            nb = min(batch, M - b0)
            with BatchSimulation.jet(g, lattice, gas, pp, base_seed, m0 + b0, nb, strip_width,
                                     device) as sim:
                for ti, t in enumerate(times):
                    sim.run_to(t)
                    sim.fields_to_device(snaps[ti][b0:b0 + nb].data_ptr())
                    if require_positivity:
                        u = snaps[ti][b0:b0 + nb].cpu().numpy()
                        for s in range(nb):
                            ok[b0 + s] &= _positive(u[s], gas.gamma)
                _, st, status = sim.scalars()
                ok[b0:b0 + nb] &= status != 2  # diverged: placeholder snapshots, inadmissible
                steps[b0:b0 + nb] = st
        store.append(snaps)
        valid.append(ok)
        rep.steps[g.label()] = steps
    n_pairs = levels - 1
    w1s = [[0.0] * len(times) for _ in range(n_pairs)]
    strongs = [[0.0] * len(times) for _ in range(n_pairs)]
    if dist is not None:
        return _sharded_metrics(torch, dist, group, grids, times, store, valid, metric_variable,
                                rep, w1s, strongs)
    for p in range(n_pairs):
        cg, fg = grids[p], grids[p + 1]
        mask = valid[p] & valid[p + 1]
        m_star = int(mask.sum())
        if m_star < 1:
            raise RuntimeError("metrics: no jointly valid samples for pair")
        keep = torch.from_numpy(np.flatnonzero(mask)).to(dev)
        for ti, t in enumerate(times):
            c = store[p][ti].index_select(0, keep).contiguous()
            f = store[p + 1][ti].index_select(0, keep).contiguous()
            k = metric_variable
            w1 = float(post.ordered_mean(
                torch, post.w1_cell_terms(torch, c[:, k].contiguous(), f[:, k].contiguous()))
                .item())
            part = torch.empty((m_star, 10), dtype=torch.float64, device=dev)
            _check(lib().vlbm_d_strong_partials(m_star, cg.nx, cg.ny, c.data_ptr(), f.data_ptr(),
                                                part.data_ptr(),
                                                torch.cuda.current_stream(dev).cuda_stream))
            es = post.strong_finish(part.cpu().numpy())
            rep.rows.append(MetricsRow(float(t), f"{cg.nx}->{fg.nx}", m_star, w1, es))
            w1s[p][ti], strongs[p][ti] = w1, es
    return _finish_rates(rep, grids, times, w1s, strongs)


def _finish_rates(rep, grids, times, w1s, strongs):
    n_pairs = len(grids) - 1
    dxs = [g.dx() for g in grids[:-1]]

    def safe_fit(e):
        try:
            return fit_rate(e, dxs)
        except ValueError:
            return float("nan")

    for ti, t in enumerate(times):
        rep.rates.append(RateRow(float(t), safe_fit([w1s[p][ti] for p in range(n_pairs)]),
                                 safe_fit([strongs[p][ti] for p in range(n_pairs)])))
    return rep


def _sharded_metrics(torch, dist, group, grids, times, store, valid, k, rep, w1s, strongs):
    """The metrics of a sample-sharded sweep (see grid_sweep)."""
    from .dist import distributed_strong_error, peer_wasserstein1
    rank = dist.get_rank(group)
    host = dist.get_backend(group) == "gloo"
    for label in list(rep.steps):  # per-sample step counts of every rank, in sample order
        parts = [None] * dist.get_world_size(group)
        dist.all_gather_object(parts, rep.steps[label].tolist(), group=group)
        rep.steps[label] = np.array([x for q in parts for x in q], np.int64)
    for p in range(len(grids) - 1):
        cg, fg = grids[p], grids[p + 1]
        mask = valid[p] & valid[p + 1]
        counts = [None] * dist.get_world_size(group)
        dist.all_gather_object(counts, int(mask.sum()), group=group)
        m_star = sum(counts)
        if m_star < 1:
            raise RuntimeError("metrics: no jointly valid samples for pair")
        dev = store[p][0].device
        keep = torch.from_numpy(np.flatnonzero(mask)).to(dev)
        vmask = torch.from_numpy(mask)
        for ti, t in enumerate(times):
            c = store[p][ti]
            f = store[p + 1][ti]
            M = c.shape[0]
            w1 = peer_wasserstein1(torch, dist, c[:, k].reshape(M, -1).contiguous(),
                                   f[:, k].reshape(M, -1).contiguous(), vmask, cg.nx, group)
            cv = c.index_select(0, keep).contiguous()
            fv = f.index_select(0, keep).contiguous()
            part = torch.empty((cv.shape[0], 10), dtype=torch.float64, device=dev)
            if cv.shape[0]:
                _check(lib().vlbm_d_strong_partials(cv.shape[0], cg.nx, cg.ny, cv.data_ptr(),
                                                    fv.data_ptr(), part.data_ptr(),
                                                    torch.cuda.current_stream(dev).cuda_stream))
            es = distributed_strong_error(torch, dist, part.cpu() if host else part, group)
            if rank == 0:
                rep.rows.append(MetricsRow(float(t), f"{cg.nx}->{fg.nx}", m_star, w1, es))
                w1s[p][ti], strongs[p][ti] = w1, es
    if rank != 0:
        return None
    return _finish_rates(rep, grids, times, w1s, strongs)


def production_sweep(torch, nx0: int, ny0: int, levels: int, n_samples: int,
                     times: Sequence[float], base_seed: int = 42, batch: int = 125,
                     lattice: LatticeParams = LatticeParams(), gas: GasParams = GasParams(),
                     pp: PerturbationParams = PerturbationParams(), strip_width: float = 0.02,
                     metric_variable: int = 0, m0: int = 0, device: int = 0,
                     progress=None) -> SweepReport:
    """grid_sweep at production scale (BASELINE configs[4]: M = 1000, grids up
    to 2000x400 / 4000x800): the same rows and rates, bit for bit, without
    keeping every level's snapshots.

    Sample-batch major: each batch of samples is marched on every level in
    turn (level l's snapshots of the batch stay on the device only until
    level l + 1 of the batch has run).  As soon as a fine-level snapshot of
    the batch exists, the pair's per-sample strong_error partials are taken
    against the coarse snapshot (restriction fused, vlbm_d_strong_partials),
    and the metric variable is kept for W1 -- the coarse plane and the
    restricted fine plane (vlbm_d_restrict_var: the same arithmetic as the
    fused restriction).  After the last batch: joint validity per pair, W1 of
    the jointly valid samples per (pair, time) on the device (cell terms +
    storage-order mean), E_strong from their partials in sample order, and
    the rate fits.  Device memory: one level's batch state, the previous
    level's batch snapshots and the W1 planes (2 x M x coarse cells per
    pair and time)."""
    if levels < 2:
        raise RuntimeError("metrics: need >= 2 grids for Cauchy errors")
    import time as _time
    times = list(times)
    T, M = len(times), n_samples
    dev = torch.device("cuda", device)
    grids = [Grid(nx0 << l, ny0 << l) for l in range(levels)]
    k = metric_variable
    f64 = torch.float64
    # W1 planes [pair][time]: coarse plane (M, nc) and restricted fine plane (M, nc)
    w1c = [[torch.empty((M, grids[p].cells()), dtype=f64, device=dev) for _ in times]
           for p in range(levels - 1)]
    w1f = [[torch.empty((M, grids[p].cells()), dtype=f64, device=dev) for _ in times]
           for p in range(levels - 1)]
    part = [torch.empty((T, M, 10), dtype=f64, device=dev) for _ in range(levels - 1)]
    valid = [np.ones(M, bool) for _ in grids]
    steps = [np.zeros(M, np.int64) for _ in grids]
    march_s = [0.0] * levels
    rep = SweepReport()
    stream = torch.cuda.current_stream(dev)
    for b0 in range(0, M, batch):
        nb = min(batch, M - b0)
        prev = None  # level l-1 snapshots of this batch: (T, nb, 4, ny, nx)
        for l, g in enumerate(grids):
            keep = l < levels - 1
            cur = torch.empty((T if keep else 1, nb, 4, g.ny, g.nx), dtype=f64, device=dev)
            t0 = _time.perf_counter()
            with BatchSimulation.jet(g, lattice, gas, pp, base_seed, m0 + b0, nb, strip_width,
                                     device) as sim:
                for ti, t in enumerate(times):
                    sim.run_to(t)
                    buf = cur[ti if keep else 0]
                    sim.fields_to_device(buf.data_ptr())
                    torch.cuda.synchronize(dev)
                    s = stream.cuda_stream
                    if l > 0:
                        cg = grids[l - 1]
                        _check(lib().vlbm_d_strong_partials(
                            nb, cg.nx, cg.ny, prev[ti].data_ptr(), buf.data_ptr(),
                            part[l - 1][ti, b0:b0 + nb].data_ptr(), s))
                        _check(lib().vlbm_d_restrict_var(
                            nb, cg.nx, cg.ny, buf.data_ptr(), k,
                            w1f[l - 1][ti][b0:b0 + nb].data_ptr(), s))
                    if keep:
                        w1c[l][ti][b0:b0 + nb].copy_(buf[:, k].reshape(nb, -1))
                _, st, status = sim.scalars()
            torch.cuda.synchronize(dev)
            march_s[l] += _time.perf_counter() - t0
            valid[l][b0:b0 + nb] &= status != 2
            steps[l][b0:b0 + nb] = st
            prev = cur if keep else None
            if progress:
                progress(b0 + nb, M, g.label())
    for l, g in enumerate(grids):
        rep.steps[g.label()] = steps[l]
    rep.march_seconds = {g.label(): march_s[l] for l, g in enumerate(grids)}
    n_pairs = levels - 1
    w1s = [[0.0] * T for _ in range(n_pairs)]
    strongs = [[0.0] * T for _ in range(n_pairs)]
    t0 = _time.perf_counter()
    for p in range(n_pairs):
        cg, fg = grids[p], grids[p + 1]
        mask = valid[p] & valid[p + 1]
        m_star = int(mask.sum())
        if m_star < 1:
            raise RuntimeError("metrics: no jointly valid samples for pair")
        idx = torch.from_numpy(np.flatnonzero(mask)).to(dev)
        for ti, t in enumerate(times):
            a = w1c[p][ti].index_select(0, idx).contiguous()
            b = w1f[p][ti].index_select(0, idx).contiguous()
            terms = torch.empty(cg.cells(), dtype=f64, device=dev)
            _check(lib().vlbm_d_w1_cells_planes(m_star, cg.cells(), a.data_ptr(), b.data_ptr(),
                                                terms.data_ptr(), stream.cuda_stream))
            w1 = float(post.ordered_mean(torch, terms).item())
            es = post.strong_finish(part[p][ti].index_select(0, idx).cpu().numpy())
            rep.rows.append(MetricsRow(float(t), f"{cg.nx}->{fg.nx}", m_star, w1, es))
            w1s[p][ti], strongs[p][ti] = w1, es
    rep.metrics_seconds = _time.perf_counter() - t0
    return _finish_rates(rep, grids, times, w1s, strongs)
