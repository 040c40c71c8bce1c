"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers:

* ``Oracle("ref")``  -> oracle/_ref/libvlbm_ref.so, the UNMODIFIED reference
  headers (/root/reference/proj/include/vlbm/*.hpp) behind oracle/ref_shim.cpp;
* ``Oracle("vo")``   -> oracle/lib/libvlbm_oracle.so, our plain-C restatement
  (oracle/vlbm_oracle.c), pinned to "ref" by tests/test_oracle_pin.py.

Both expose the same calls with the same argument meaning, so every parity
test can be run against either.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module; the
product package (paper_2605_25282_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libvlbm_ref.so"),
    "vo": os.path.join(HERE, "lib", "libvlbm_oracle.so"),
}

D = C.c_double
I = C.c_int
L = C.c_long
U64 = C.c_uint64
I64 = C.c_int64
P = C.c_void_p
DP = C.POINTER(C.c_double)


class VGrid(C.Structure):
    _fields_ = [("nx", I), ("ny", I), ("x_max", D), ("y_min", D), ("y_max", D)]


class VParams(C.Structure):
    _fields_ = [
        ("gamma", D), ("alpha", D), ("safety", D), ("rlmp_relaxation", D),
        ("positivity_floor", D), ("limiter", I), ("conservative_bound", I),
        ("rho_ref", D), ("p_ref", D), ("bc", I * 4),
    ]


class VPert(C.Structure):
    _fields_ = [
        ("amplitude", D), ("modes", I), ("decay_exponent", D), ("r_jet", D),
        ("rho_jet_bar", D), ("rho_amb", D), ("p_amb", D), ("v_jet", D),
    ]


INLET, OUTFLOW, WALL, PERIODIC = 0, 1, 2, 3
FIRST_ORDER, SECOND_ORDER, RLMP = 0, 1, 2


def make_grid(nx, ny, x_max=2.5, y_min=-0.25, y_max=0.25) -> VGrid:
    return VGrid(nx, ny, x_max, y_min, y_max)


def make_params(gamma=5.0 / 3.0, alpha=0.0, safety=2.0, limiter=RLMP, kappa=0.5, floor=1e-7,
                conservative_bound=0, rho_ref=0.5, p_ref=0.4127,
                bc=(INLET, OUTFLOW, WALL, WALL)) -> VParams:
    p = VParams()
    p.gamma, p.alpha, p.safety, p.rlmp_relaxation = gamma, alpha, safety, kappa
    p.positivity_floor, p.limiter, p.conservative_bound = floor, limiter, conservative_bound
    p.rho_ref, p.p_ref = rho_ref, p_ref
    for k in range(4):
        p.bc[k] = bc[k]
    return p


def make_pert(amplitude=0.1, modes=10, decay_exponent=2.0, r_jet=0.05, rho_jet_bar=5.0,
              rho_amb=0.5, p_amb=0.4127, v_jet=800.0) -> VPert:
    return VPert(amplitude, modes, decay_exponent, r_jet, rho_jet_bar, rho_amb, p_amb, v_jet)


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(DP)


def build(ref: bool = True) -> None:
    """Compile the restatement (and the reference shim when the reference
    headers are present) with oracle/Makefile."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/include"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    def __init__(self, kind: str = "vo"):
        self.kind = kind
        self.pre = "ref_" if kind == "ref" else "vo_"
        self.lib = C.CDLL(LIBS[kind])
        self._sig()

    def _f(self, name, res, args):
        fn = getattr(self.lib, self.pre + name)
        fn.restype = res
        fn.argtypes = args
        return fn

    def _sig(self):
        G, Pp, Pe = C.POINTER(VGrid), C.POINTER(VParams), C.POINTER(VPert)
        f = self._f
        self.f_last_error = f("last_error", C.c_char_p, [])
        self.f_draw = f("draw_coefficients", U64, [U64, U64, I, DP, DP])
        self.f_mix64 = f("mix64", U64, [U64])
        self.f_sample_seed = f("sample_seed", U64, [U64, U64])
        self.f_dens = f("density_perturbation", D, [D, I, DP, DP, Pe])
        self.f_inlet = f("inlet_state", None, [D, I, DP, DP, Pe, D, DP])
        self.f_init = f("initial_field", I, [G, I, DP, DP, Pe, D, D, DP])
        self.f_pressure = f("pressure", D, [DP, D])
        self.f_maxw = f("maxwellians", None, [DP, D, D, D, DP])
        self.f_create = f("sim_create", I, [G, Pp, DP, DP, U64, C.POINTER(P)])
        self.f_destroy = f("sim_destroy", None, [P])
        self.f_step = f("sim_step", I, [P, D])
        self.f_suggest = f("sim_suggest_dt", D, [P])
        self.f_time = f("sim_time", D, [P])
        self.f_steps = f("sim_steps", L, [P])
        self.f_finite = f("sim_state_finite", I, [P])
        self.f_get = f("sim_get", None, [P, DP, DP])
        self.f_blend = f("sim_compute_blending", I, [P, D, DP, DP])
        self.f_swb = f("sim_step_with_blending", I, [P, D, DP, DP])
        self.f_run = f("run_sample", I, [G, Pp, Pe, I, DP, DP, U64, D, DP, I, DP, DP,
                                         C.POINTER(I), C.POINTER(L), C.POINTER(I)])
        self.f_restrict = f("restrict_field", I, [I, I, DP, DP])
        self.f_strong = f("strong_error", I, [I, I64, DP, DP, DP, DP])
        self.f_w1 = f("wasserstein1", I, [I, I64, DP, DP, I, DP])
        self.f_mom = f("ensemble_moments", I, [I, I64, DP, DP, DP])
        if self.kind == "vo":
            self.f_theta = f("sim_theta_cell", None, [P, DP])
            self.f_limcells = f("sim_limiter_cells", I, [P, D, DP])
        if self.kind == "ref":
            self.f_ot = f("ot_oracle", D, [I, DP, DP])
            self.f_fit = f("fit_rate", D, [I, DP, DP])
            self.f_march = f("march_timed", D, [G, Pp, Pe, U64, L, I, L, D, D, I, C.POINTER(L)])
            self.f_post = f("postproc_timed", D, [I, I, I, DP, DP, DP, DP])
            self.f_window = f("march_window", D, [G, Pp, Pe, U64, L, I, D, L, D, I,
                                                  C.POINTER(L), DP])

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.f_last_error().decode())

    # ---- IC -----------------------------------------------------------------
    def draw_coefficients(self, base, m, K=10):
        y, z = np.zeros(K), np.zeros(K)
        seed = self.f_draw(base, m, K, _dp(y), _dp(z))
        return int(seed), y, z

    def density_perturbation(self, y, yc, zc, pp):
        yc, zc = np.ascontiguousarray(yc, np.float64), np.ascontiguousarray(zc, np.float64)
        return self.f_dens(y, len(yc), _dp(yc), _dp(zc), C.byref(pp))

    def inlet_state(self, y, yc, zc, pp, gamma=5.0 / 3.0):
        yc, zc = np.ascontiguousarray(yc, np.float64), np.ascontiguousarray(zc, np.float64)
        out = np.zeros(4)
        self.f_inlet(y, len(yc), _dp(yc), _dp(zc), C.byref(pp), gamma, _dp(out))
        return out

    def inlet_rows(self, g: VGrid, yc, zc, pp, gamma=5.0 / 3.0):
        dx = g.x_max / g.nx
        return np.stack([self.inlet_state(g.y_min + (j + 0.5) * dx, yc, zc, pp, gamma)
                         for j in range(g.ny)])

    def initial_field(self, g, yc, zc, pp, gamma=5.0 / 3.0, strip=0.02):
        yc, zc = np.ascontiguousarray(yc, np.float64), np.ascontiguousarray(zc, np.float64)
        out = np.zeros((4, g.ny, g.nx))
        self._check(self.f_init(C.byref(g), len(yc), _dp(yc), _dp(zc), C.byref(pp), gamma, strip,
                                _dp(out)))
        return out

    def pressure(self, u, gamma):
        u = np.ascontiguousarray(u, np.float64)
        return self.f_pressure(_dp(u), gamma)

    def maxwellians(self, u, a, alpha, gamma):
        u = np.ascontiguousarray(u, np.float64)
        out = np.zeros((4, 4))
        self.f_maxw(_dp(u), a, alpha, gamma, _dp(out))
        return out

    # ---- Simulation ---------------------------------------------------------
    def sim(self, g, p, init, inlet_rows=None, seed=0) -> "Sim":
        init = np.ascontiguousarray(init, np.float64)
        rows = None if inlet_rows is None else np.ascontiguousarray(inlet_rows, np.float64)
        h = P()
        self._check(self.f_create(C.byref(g), C.byref(p), _dp(init),
                                  None if rows is None else _dp(rows), seed, C.byref(h)))
        return Sim(self, h, g)

    def jet_sim(self, g, p, pp, base_seed, m, strip=0.02) -> "Sim":
        """A sample built as run_sample builds it (solver.hpp:633-640)."""
        seed, yc, zc = self.draw_coefficients(base_seed, m, pp.modes)
        rows = self.inlet_rows(g, yc, zc, pp, p.gamma)
        init = self.initial_field(g, yc, zc, pp, p.gamma, strip)
        q = make_params(gamma=p.gamma, alpha=p.alpha, safety=p.safety, limiter=p.limiter,
                        kappa=p.rlmp_relaxation, floor=p.positivity_floor,
                        conservative_bound=p.conservative_bound, rho_ref=pp.rho_amb,
                        p_ref=pp.p_amb, bc=(INLET, OUTFLOW, WALL, WALL))
        return self.sim(g, q, init, rows, seed)

    def run_sample(self, g, p, pp, base_seed, m, times, strip=0.02):
        seed, yc, zc = self.draw_coefficients(base_seed, m, pp.modes)
        times = np.ascontiguousarray(times, np.float64)
        nt = len(times)
        fields = np.zeros((nt, 4, g.ny, g.nx))
        t_out = np.zeros(nt)
        div = (I * nt)()
        steps, adm = L(), I()
        self._check(self.f_run(C.byref(g), C.byref(p), C.byref(pp), len(yc), _dp(yc), _dp(zc),
                               seed, strip, _dp(times), nt, _dp(fields), _dp(t_out), div,
                               C.byref(steps), C.byref(adm)))
        return dict(fields=fields, time=t_out, diverged=np.array(list(div), bool),
                    steps=steps.value, admissible=bool(adm.value), seed=seed)

    # ---- metrics ------------------------------------------------------------
    def restrict_field(self, fine):
        fine = np.ascontiguousarray(fine, np.float64)
        _, ny, nx = fine.shape
        out = np.zeros((4, ny // 2, nx // 2))
        self._check(self.f_restrict(nx, ny, _dp(fine), _dp(out)))
        return out

    def strong_error(self, a, b):
        a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
        M = a.shape[0]
        n = a[0].size // 4
        r, pc = D(), np.zeros(4)
        self._check(self.f_strong(M, n, _dp(a), _dp(b), C.byref(r), _dp(pc)))
        return r.value, pc

    def wasserstein1(self, a, b, var=0):
        a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
        M = a.shape[0]
        n = a[0].size // 4
        r = D()
        self._check(self.f_w1(M, n, _dp(a), _dp(b), var, C.byref(r)))
        return r.value

    def ensemble_moments(self, x):
        x = np.ascontiguousarray(x, np.float64)
        M = x.shape[0]
        n = x[0].size // 4
        mean, sd = np.zeros(x.shape[1:]), np.zeros(x.shape[1:])
        self._check(self.f_mom(M, n, _dp(x), _dp(mean), _dp(sd)))
        return mean, sd

    def ot_oracle(self, a, b):
        a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
        return self.f_ot(len(a), _dp(a), _dp(b))

    def fit_rate(self, e, dx):
        e, dx = np.ascontiguousarray(e, np.float64), np.ascontiguousarray(dx, np.float64)
        return self.f_fit(len(e), _dp(e), _dp(dx))

    def march_timed(self, g, p, pp, base_seed, m0, n_samples, steps, t_target=0.0, strip=0.02,
                    threads=1):
        upd = L()
        sec = self.f_march(C.byref(g), C.byref(p), C.byref(pp), base_seed, m0, n_samples, steps,
                           t_target, strip, threads, C.byref(upd))
        return sec, upd.value

    def march_window(self, g, p, pp, base_seed, m0, n_samples, t_start, steps, strip=0.02,
                     threads=1):
        """Untimed run_sample loop to t_start, then `steps` timed steps of every
        sample (reference only).  Returns (timed seconds, updates, pre seconds)."""
        upd, pre = L(), D()
        sec = self.f_window(C.byref(g), C.byref(p), C.byref(pp), base_seed, m0, n_samples,
                            t_start, steps, strip, threads, C.byref(upd), C.byref(pre))
        return sec, upd.value, pre.value

    def postproc_timed(self, coarse, fine):
        """restrict_field + wasserstein1 + strong_error as compute_metrics runs
        them (single-threaded, reference only): (seconds, W1, E_strong)."""
        coarse = np.ascontiguousarray(coarse, np.float64)
        fine = np.ascontiguousarray(fine, np.float64)
        M, _, nyc, nxc = coarse.shape
        w1, es = D(), D()
        sec = self.f_post(M, nxc, nyc, _dp(coarse), _dp(fine), C.byref(w1), C.byref(es))
        return sec, w1.value, es.value


@dataclass
class Sim:
    o: Oracle
    h: P
    g: VGrid

    def __del__(self):
        try:
            self.o.f_destroy(self.h)
        except Exception:
            pass

    def step(self, dt):
        self.o._check(self.o.f_step(self.h, dt))

    def suggest_dt(self):
        return self.o.f_suggest(self.h)

    @property
    def time(self):
        return self.o.f_time(self.h)

    @property
    def steps(self):
        return self.o.f_steps(self.h)

    def state_finite(self):
        return bool(self.o.f_finite(self.h))

    def get(self, pops=False):
        u = np.zeros((4, self.g.ny, self.g.nx))
        pp = np.zeros((4, 4, self.g.ny, self.g.nx)) if pops else None
        self.o.f_get(self.h, _dp(u), None if pp is None else _dp(pp))
        return (u, pp) if pops else u

    def theta_cell(self):
        """Cell theta of the last limiter pass (restatement only)."""
        th = np.zeros((self.g.ny, self.g.nx))
        self.o.f_theta(self.h, _dp(th))
        return th

    def limiter_cells(self, a):
        """Per-cell limiter inputs and theta at speed a (restatement only):
        (ny*nx, 27) = u_FO, c_w, c_e, c_s, c_n, rho_lo, rho_hi, p_lo, p_hi,
        rho_floor, p_floor, theta."""
        out = np.zeros((self.g.ny * self.g.nx, 27))
        self.o._check(self.o.f_limcells(self.h, a, _dp(out)))
        return out

    def compute_blending(self, a):
        tx = np.zeros((self.g.ny, self.g.nx + 1))
        ty = np.zeros((self.g.ny + 1, self.g.nx))
        self.o._check(self.o.f_blend(self.h, a, _dp(tx), _dp(ty)))
        return tx, ty

    def step_with_blending(self, dt, tx, ty):
        tx, ty = np.ascontiguousarray(tx, np.float64), np.ascontiguousarray(ty, np.float64)
        self.o._check(self.o.f_swb(self.h, dt, _dp(tx), _dp(ty)))
