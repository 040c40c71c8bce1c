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
               batch: Optional[int] = None, device: int = 0) -> SweepReport:
    """Grids nx0 x ny0 * 2^l (l = 0..levels-1), M = n_samples samples each,
    snapshots at ``times``; returns the rows and rates compute_metrics would
    write (metrics.csv / rates.csv)."""
    if levels < 2:
        raise RuntimeError("metrics: need >= 2 grids for Cauchy errors")
    times = list(times)
    M = n_samples
    batch = batch or M
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
