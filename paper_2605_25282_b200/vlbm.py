"""Python host mirror of the reference's VLBM hot-path interface, over the
C ABI of include/vlbm_b200.h (libvlbm_b200.so, sm_100a kernels).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/vlbm/):

* ``Grid``, ``LatticeParams``/``GasParams``, ``PerturbationParams``,
  ``BcType``, ``Limiter``              -> grid.hpp, lattice.hpp, euler.hpp,
                                          perturbation.hpp, solver.hpp:20
* ``draw_coefficients``, ``inlet_state`` -> perturbation.hpp:42-95
* ``BatchSimulation``                  -> many ``Simulation`` objects
                                          (solver.hpp:57-603) marching together
* ``run_samples``                      -> ``run_sample`` (solver.hpp:625-669)
                                          for a batch of samples
* ``restrict_field``, ``strong_error``, ``wasserstein1``,
  ``ensemble_moments``                 -> metrics.hpp:29-177

``std::invalid_argument`` maps to ``ValueError``, ``std::domain_error`` to
``ArithmeticError``, ``std::runtime_error`` to ``RuntimeError``.  There is no
CPU fallback: if the library or a CUDA device is missing, calls raise.
Fields use the .vlbm plane layout: arrays of shape (4, ny, nx).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VLBM_LIB") or os.path.join(_PKG, "lib", "libvlbm_b200.so")

D, I, U64, I64 = C.c_double, C.c_int, C.c_uint64, C.c_int64
DP = C.POINTER(C.c_double)


class BcType(enum.IntEnum):  # solver.hpp:20
    Inlet = 0
    Outflow = 1
    Wall = 2
    Periodic = 3


class Limiter(enum.IntEnum):  # lattice.hpp:10
    FirstOrder = 0
    SecondOrder = 1
    Rlmp = 2


class _Grid(C.Structure):
    _fields_ = [("nx", I), ("ny", I), ("x_max", D), ("y_min", D), ("y_max", D)]


class _Params(C.Structure):
    _fields_ = [("gamma", D), ("alpha", D), ("safety", D), ("rlmp_relaxation", D),
                ("positivity_floor", D), ("limiter", I), ("conservative_bound", I),
                ("rho_ref", D), ("p_ref", D), ("bc", I * 4)]


class _Pert(C.Structure):
    _fields_ = [("amplitude", D), ("modes", I), ("decay_exponent", D), ("r_jet", D),
                ("rho_jet_bar", D), ("rho_amb", D), ("p_amb", D), ("v_jet", D)]


@dataclass
class Grid:  # grid.hpp:14-38
    nx: int = 0
    ny: int = 0
    x_max: float = 2.5
    y_min: float = -0.25
    y_max: float = 0.25

    def dx(self) -> float:
        return self.x_max / self.nx

    def x_center(self, i: int) -> float:
        return (i + 0.5) * self.dx()

    def y_center(self, j: int) -> float:
        return self.y_min + (j + 0.5) * self.dx()

    def cells(self) -> int:
        return self.nx * self.ny

    def label(self) -> str:
        return f"{self.nx}x{self.ny}"

    def _c(self) -> _Grid:
        return _Grid(self.nx, self.ny, self.x_max, self.y_min, self.y_max)


@dataclass
class GasParams:  # euler.hpp:9-11
    gamma: float = 5.0 / 3.0


@dataclass
class LatticeParams:  # lattice.hpp:13-35
    alpha: float = 0.0
    safety: float = 2.0
    limiter: Limiter = Limiter.Rlmp
    rlmp_relaxation: float = 0.5
    positivity_floor: float = 1e-7
    conservative_bound: bool = False


@dataclass
class PerturbationParams:  # perturbation.hpp:16-31
    amplitude: float = 0.1
    modes: int = 10
    decay_exponent: float = 2.0
    r_jet: float = 0.05
    rho_jet_bar: float = 5.0
    rho_amb: float = 0.5
    p_amb: float = 0.4127
    v_jet: float = 800.0

    def _c(self) -> _Pert:
        return _Pert(self.amplitude, self.modes, self.decay_exponent, self.r_jet,
                     self.rho_jet_bar, self.rho_amb, self.p_amb, self.v_jet)


@dataclass
class Boundaries:  # solver.hpp:25-31 (the inlet profile is passed as rows)
    x_min: BcType = BcType.Inlet
    x_max: BcType = BcType.Outflow
    y_min: BcType = BcType.Wall
    y_max: BcType = BcType.Wall


def _params(lat: LatticeParams, gas: GasParams, bcs: Boundaries, rho_ref=0.5,
            p_ref=0.4127) -> _Params:
    p = _Params()
    p.gamma, p.alpha, p.safety = gas.gamma, lat.alpha, lat.safety
    p.rlmp_relaxation, p.positivity_floor = lat.rlmp_relaxation, lat.positivity_floor
    p.limiter, p.conservative_bound = int(lat.limiter), int(bool(lat.conservative_bound))
    p.rho_ref, p.p_ref = rho_ref, p_ref
    for k, b in enumerate((bcs.x_min, bcs.x_max, bcs.y_min, bcs.y_max)):
        p.bc[k] = int(b)
    return p


# ---- library loading ---------------------------------------------------------

_lib = None


def lib() -> C.CDLL:
    """Loads libvlbm_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (the VLBM path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    G, Pp, Pe, V = C.POINTER(_Grid), C.POINTER(_Params), C.POINTER(_Pert), C.c_void_p

    def sig(name, res, args):
        f = getattr(L, name)
        f.restype, f.argtypes = res, args

    sig("vlbm_abi_version", I, [])
    sig("vlbm_last_error", C.c_char_p, [])
    sig("vlbm_draw_coefficients", U64, [U64, U64, I, DP, DP])
    sig("vlbm_inlet_rows", I, [G, Pe, D, DP, DP, DP])
    sig("vlbm_batch_create", I, [G, Pp, Pe, U64, I64, I, D, I, C.POINTER(V)])
    sig("vlbm_batch_create_fields", I, [G, Pp, I, DP, DP, C.POINTER(U64), I, C.POINTER(V)])
    sig("vlbm_batch_destroy", None, [V])
    sig("vlbm_batch_size", I, [V])
    sig("vlbm_batch_run_to", I, [V, D])
    sig("vlbm_batch_step", I, [V, I, D])
    sig("vlbm_batch_step_with_blending", I, [V, D, DP, DP])
    sig("vlbm_batch_get", I, [V, I, DP, DP, DP, C.POINTER(I64), C.POINTER(I)])
    sig("vlbm_batch_get_fields", I, [V, DP])
    sig("vlbm_batch_copy_fields_device", I, [V, V])
    sig("vlbm_batch_get_scalars", I, [V, DP, C.POINTER(I64), C.POINTER(I)])
    sig("vlbm_batch_get_theta", I, [V, I, DP])
    sig("vlbm_batch_device_u", I, [V, I, C.POINTER(DP)])
    sig("vlbm_batch_stream", V, [V])
    sig("vlbm_batch_set_timing", I, [V, I])
    sig("vlbm_batch_stats", I, [V, C.POINTER(I64), DP, DP, DP, C.POINTER(I64)])
    sig("vlbm_batch_kernel_ms", I, [V, DP])
    sig("vlbm_batch_set_audit", I, [V, I])
    sig("vlbm_batch_audit", I, [V, C.POINTER(I64)])
    sig("vlbm_batch_queue_stats", I, [V, C.POINTER(I64)])
    sig("vlbm_metrics_begin", I, [I, I, I, I, I, C.POINTER(V)])
    sig("vlbm_metrics_add", I, [V, I, I, DP, DP])
    sig("vlbm_metrics_finish", I, [V, DP, DP, DP])
    sig("vlbm_metrics_destroy", None, [V])
    sig("vlbm_restrict_field", I, [I, I, DP, DP])
    sig("vlbm_strong_error", I, [I, I64, DP, DP, DP, DP])
    sig("vlbm_wasserstein1", I, [I, I64, DP, DP, I, DP])
    sig("vlbm_ensemble_moments", I, [I, I64, DP, DP, DP])
    sig("vlbm_d_strong_partials", I, [I, I, I, V, V, V, V])
    sig("vlbm_d_strong_partials_var", I, [I, I, I, V, I64, V, I64, V, V])
    sig("vlbm_strong_finish", I, [I, DP, DP, DP])
    sig("vlbm_d_w1_restrict", I, [I, I, I, V, I64, V, I64, V, V])
    sig("vlbm_d_restrict_var", I, [I, I, I, V, I, V, V])
    sig("vlbm_d_w1_cells", I, [I, I64, V, V, V, V])
    sig("vlbm_d_w1_cells_planes", I, [I, I64, V, V, V, V])
    sig("vlbm_d_ordered_mean", I, [I64, V, V, V])
    sig("vlbm_d_moments_planes", I, [I, I64, V, V, V, V])
    sig("vlbm_d_w1_rows", I, [I, I, I64, I64, V, V, V, V])
    sig("vlbm_d_w1_restrict_mean", I, [I, I, I, V, I64, V, I64, V, V, V, V])
    sig("vlbm_ipc_handle", I, [V, C.POINTER(C.c_ubyte), C.POINTER(U64)])
    sig("vlbm_ipc_open", I, [C.POINTER(C.c_ubyte), C.POINTER(V)])
    sig("vlbm_ipc_close", I, [V])
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().vlbm_last_error().decode()
    if rc == -1:
        raise ValueError(msg)
    if rc == -2:
        raise ArithmeticError(msg)
    if rc == -5:
        raise MemoryError(msg)
    raise RuntimeError(f"vlbm error {rc}: {msg}")


def _dp(a: np.ndarray):
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError("expected a C-contiguous float64 array")
    return a.ctypes.data_as(DP)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- initial conditions ------------------------------------------------------

@dataclass
class ModeCoefficients:  # perturbation.hpp:34-38
    y_coeffs: np.ndarray
    z_coeffs: np.ndarray
    seed: int = 0


def draw_coefficients(base_seed: int, m: int, K: int) -> ModeCoefficients:
    """draw_coefficients (perturbation.hpp:42-54): 2K splitmix64 uniforms."""
    if K < 1:
        raise ValueError("draw_coefficients: K must be >= 1")
    y, z = np.zeros(K), np.zeros(K)
    seed = lib().vlbm_draw_coefficients(base_seed, m, K, _dp(y), _dp(z))
    return ModeCoefficients(y, z, int(seed))


def inlet_rows(grid: Grid, coeffs: ModeCoefficients, pp: PerturbationParams,
               gas: GasParams = GasParams()) -> np.ndarray:
    """inlet_state at every y_center(j) (perturbation.hpp:87-95) -> (ny, 4)."""
    out = np.zeros((grid.ny, 4))
    p = pp._c()
    p.modes = len(coeffs.y_coeffs)
    _check(lib().vlbm_inlet_rows(C.byref(grid._c()), C.byref(p), gas.gamma,
                                 _dp(_f64(coeffs.y_coeffs)), _dp(_f64(coeffs.z_coeffs)),
                                 _dp(out)))
    return out


# ---- the march ---------------------------------------------------------------

class BatchSimulation:
    """S independent ``Simulation`` instances on one grid, marched together on
    one GPU (sample index folded into the launch grid).

    Construct either the jet case exactly as ``run_sample`` builds it
    (``BatchSimulation.jet``) or from explicit initial fields and boundaries
    (``BatchSimulation(grid, lattice, gas, bcs, fields, inlet_rows)``)."""

    def __init__(self, grid: Grid, lattice: LatticeParams, gas: GasParams, bcs: Boundaries,
                 fields, inlet_rows=None, rho_ref: float = 0.5, p_ref: float = 0.4127,
                 device: int = 0, _handle=None):
        self.grid = grid
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            f = _f64(fields)
            if f.ndim == 3:
                f = f[None]
            if f.shape[1:] != (4, grid.ny, grid.nx):
                raise ValueError("Simulation: initial field size mismatch")
            rows = None
            if inlet_rows is not None:
                rows = _f64(inlet_rows)
                if rows.ndim == 2:
                    rows = np.ascontiguousarray(np.broadcast_to(rows, (f.shape[0],) + rows.shape))
            p = _params(lattice, gas, bcs, rho_ref, p_ref)
            _check(lib().vlbm_batch_create_fields(C.byref(grid._c()), C.byref(p), f.shape[0],
                                                  _dp(f), None if rows is None else _dp(rows),
                                                  None, device, C.byref(self._h)))
        self.n = lib().vlbm_batch_size(self._h)

    @classmethod
    def jet(cls, grid: Grid, lattice: LatticeParams = LatticeParams(),
            gas: GasParams = GasParams(), pp: PerturbationParams = PerturbationParams(),
            base_seed: int = 42, m0: int = 0, n_samples: int = 1, strip_width: float = 0.02,
            device: int = 0) -> "BatchSimulation":
        """Samples m0..m0+n-1 built as run_sample builds them (solver.hpp:633-640)."""
        h = C.c_void_p()
        p = _params(lattice, gas, Boundaries())
        _check(lib().vlbm_batch_create(C.byref(grid._c()), C.byref(p), C.byref(pp._c()),
                                       base_seed, m0, n_samples, strip_width, device,
                                       C.byref(h)))
        return cls(grid, lattice, gas, Boundaries(), None, _handle=h)

    def close(self):
        if self._h:
            lib().vlbm_batch_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- marching --
    def run_to(self, target: float) -> None:
        """run_sample's inner loop to `target` for every running sample."""
        _check(lib().vlbm_batch_run_to(self._h, target))

    def step(self, n: int = 1, dt: float = 0.0) -> None:
        """n x step(suggest_dt()) per sample; dt > 0 uses step(dt)."""
        _check(lib().vlbm_batch_step(self._h, n, dt))

    def step_with_blending(self, theta_x, theta_y, dt: float = 0.0) -> None:
        tx, ty = _f64(theta_x), _f64(theta_y)
        g = self.grid
        tx = np.ascontiguousarray(np.broadcast_to(tx, (self.n, g.ny, g.nx + 1)))
        ty = np.ascontiguousarray(np.broadcast_to(ty, (self.n, g.ny + 1, g.nx)))
        _check(lib().vlbm_batch_step_with_blending(self._h, dt, _dp(tx), _dp(ty)))

    # -- readout --
    def state(self, s: int = 0) -> np.ndarray:
        u = np.zeros((4, self.grid.ny, self.grid.nx))
        _check(lib().vlbm_batch_get(self._h, s, _dp(u), None, None, None, None))
        return u

    def populations(self, s: int = 0) -> np.ndarray:
        p = np.zeros((4, 4, self.grid.ny, self.grid.nx))
        _check(lib().vlbm_batch_get(self._h, s, None, _dp(p), None, None, None))
        return p

    def fields(self) -> np.ndarray:
        u = np.zeros((self.n, 4, self.grid.ny, self.grid.nx))
        _check(lib().vlbm_batch_get_fields(self._h, _dp(u)))
        return u

    def fields_to_device(self, ptr: int) -> None:
        """Dense (n, 4, ny, nx) fields into device memory at ptr (same GPU)."""
        _check(lib().vlbm_batch_copy_fields_device(self._h, ptr))

    def scalars(self):
        t = np.zeros(self.n)
        st = (I64 * self.n)()
        stat = (I * self.n)()
        _check(lib().vlbm_batch_get_scalars(self._h, _dp(t), st, stat))
        return t, np.array(st[:], np.int64), np.array(stat[:], np.int32)

    def times(self) -> np.ndarray:
        return self.scalars()[0]

    def theta_cell(self, s: int = 0) -> np.ndarray:
        th = np.zeros((self.grid.ny, self.grid.nx))
        _check(lib().vlbm_batch_get_theta(self._h, s, _dp(th)))
        return th

    def set_timing(self, on: bool = True) -> None:
        _check(lib().vlbm_batch_set_timing(self._h, int(on)))

    def stats(self) -> dict:
        la, cu = I64(), I64()
        mt, ma, ms = D(), D(), D()
        _check(lib().vlbm_batch_stats(self._h, C.byref(la), C.byref(mt), C.byref(ma),
                                      C.byref(ms), C.byref(cu)))
        km = (D * 4)()
        _check(lib().vlbm_batch_kernel_ms(self._h, km))
        return dict(launches=la.value, ms_theta=mt.value, ms_advance=ma.value,
                    ms_sched=ms.value, cell_updates=cu.value, ms_theta_tiles=km[0],
                    ms_theta_hard=km[1])

    def queue_stats(self) -> dict:
        """Limiter-queue capacity, sample groups and overflow / hard-cell
        counters (cumulative since creation; vlbm_batch_queue_stats)."""
        n = (I64 * 6)()
        _check(lib().vlbm_batch_queue_stats(self._h, n))
        return dict(capacity=n[0], groups=n[1], overflow=n[2], peak_hard=n[3],
                    hard_total=n[4], passes=n[5])

    def set_audit(self, on: bool = True) -> None:
        """Re-check every certified bisection step with the full feasible()."""
        _check(lib().vlbm_batch_set_audit(self._h, int(on)))

    def audit_counters(self) -> dict:
        n = (I64 * 16)()
        _check(lib().vlbm_batch_audit(self._h, n))
        return dict(mismatches=n[0], bisections=n[1], certified_at_thc=n[2], uncertified=n[3],
                    not_certifiable=n[4], no_margin_at_0=n[5], unc_vertices_start=n[6],
                    vertex_evals=n[7], diag_ok_at_1=n[8], vertex_decided_at_1=n[9],
                    feasible_at_1=n[10], vertex_open_at_1=n[12],
                    stage_decided_by_form=n[13])

    def audit_mismatches(self) -> int:
        return self.audit_counters()["mismatches"]

    def device_u(self, s: int = 0) -> int:
        p = DP()
        _check(lib().vlbm_batch_device_u(self._h, s, C.byref(p)))
        return C.cast(p, C.c_void_p).value

    def stream(self) -> int:
        return lib().vlbm_batch_stream(self._h) or 0


# ---- run_sample ----------------------------------------------------------------

@dataclass
class FieldSnapshot:  # grid.hpp:41-52 (data in plane layout (4, ny, nx))
    grid: Grid
    time: float = 0.0
    sample_seed: int = 0
    diverged: bool = False
    data: np.ndarray = field(default_factory=lambda: np.zeros((4, 0, 0)))


@dataclass
class SampleResult:  # solver.hpp:605-609
    snapshots: list
    admissible: bool = True
    steps: int = 0


def run_samples(grid: Grid, lattice: LatticeParams, gas: GasParams, pp: PerturbationParams,
                base_seed: int, m0: int, n_samples: int, strip_width: float,
                snapshot_times: Sequence[float], device: int = 0) -> list[SampleResult]:
    """``run_sample`` (solver.hpp:625-669) for samples m0..m0+n-1 in one batch:
    every sample marches to each snapshot time with its own adaptive dt,
    clamped to hit the time exactly; divergence yields placeholder snapshots
    stamped with the sample's own time and the diverged flag."""
    times = list(snapshot_times)
    for a, b in zip(times, times[1:]):
        if b <= a:
            raise ValueError("run_sample: snapshot times must be strictly increasing")
    seeds = [draw_coefficients(base_seed, m0 + s, pp.modes).seed for s in range(n_samples)]
    results = [SampleResult([], True, 0) for _ in range(n_samples)]
    with BatchSimulation.jet(grid, lattice, gas, pp, base_seed, m0, n_samples, strip_width,
                             device) as sim:
        for target in times:
            sim.run_to(target)
            u = sim.fields()
            t, steps, status = sim.scalars()
            for s in range(n_samples):
                div = bool(status[s] == 2)
                results[s].snapshots.append(FieldSnapshot(
                    grid, float(t[s]) if div else float(target), seeds[s], div, u[s]))
        t, steps, status = sim.scalars()
        for s in range(n_samples):
            results[s].admissible = bool(status[s] != 2)
            results[s].steps = int(steps[s])
    return results


# ---- metrics -----------------------------------------------------------------

def restrict_field(fine) -> np.ndarray:
    """restrict_field (metrics.hpp:29-49) of one (4, ny, nx) field."""
    f = _f64(fine)
    _, ny, nx = f.shape
    if nx % 2 or ny % 2:
        raise ValueError("restrict_field: fine dimensions must be even")
    out = np.zeros((4, ny // 2, nx // 2))
    _check(lib().vlbm_restrict_field(nx, ny, _dp(f), _dp(out)))
    return out


def _ensemble(x) -> np.ndarray:
    x = _f64(x)
    if x.ndim < 2 or x.shape[1] != 4:
        raise ValueError("expected an ensemble of shape (M, 4, ...)")
    return x


def strong_error(coarse, restricted_fine, per_component: bool = False):
    """strong_error (metrics.hpp:55-90): mean over samples of the relative L1
    distance over all four components."""
    a, b = _ensemble(coarse), _ensemble(restricted_fine)
    if a.shape[0] == 0 or a.shape[0] != b.shape[0]:
        raise ValueError("strong_error: sample counts differ or are empty")
    if a.shape != b.shape:
        raise ValueError("strong_error: grid mismatch between coarse and restricted")
    r, pc = D(), np.zeros(4)
    _check(lib().vlbm_strong_error(a.shape[0], a[0].size // 4, _dp(a), _dp(b), C.byref(r),
                                   _dp(pc)))
    return (r.value, pc) if per_component else r.value


def wasserstein1(a, b, var: int = 0) -> float:
    """wasserstein1 (metrics.hpp:97-125): per-cell sorted-order W1, averaged
    over cells in storage order (bit-exact)."""
    a, b = _ensemble(a), _ensemble(b)
    if a.shape[0] == 0 or a.shape[0] != b.shape[0]:
        raise ValueError("wasserstein1: sample counts differ or are empty")
    if a.shape != b.shape:
        raise ValueError("wasserstein1: inconsistent field sizes")
    r = D()
    _check(lib().vlbm_wasserstein1(a.shape[0], a[0].size // 4, _dp(a), _dp(b), int(var),
                                   C.byref(r)))
    return r.value


def ensemble_moments(samples):
    """ensemble_moments (metrics.hpp:148-177) -> (mean, stddev)."""
    x = _ensemble(samples)
    if x.shape[0] == 0:
        raise ValueError("ensemble_moments: no samples")
    mean, sd = np.zeros(x.shape[1:]), np.zeros(x.shape[1:])
    _check(lib().vlbm_ensemble_moments(x.shape[0], x[0].size // 4, _dp(x), _dp(mean), _dp(sd)))
    return mean, sd
