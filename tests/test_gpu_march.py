"""GPU parity of the batched VLBM march against the CPU oracle (-m gpu).

Every comparison is BIT-EXACT (uint64 views, so +-0 and NaN payloads count):
the limiter's discrete decisions amplify one ulp to O(1) within ~50 steps
(SURVEY.md §0 fact 4), so anything short of bit identity is a failure.  The
oracle is the reference itself (`orc`: oracle/_ref, the unmodified headers
compiled by oracle/Makefile, whose .so travels to the GPU box) whenever it is
built, else the C restatement (oracle/vlbm_oracle.c, pinned bit-for-bit to
the reference by tests/test_oracle_pin.py); the cell-theta checks use the
restatement (the reference does not expose its cell theta).
"""
import numpy as np
import pytest

from oracle.oracle import (INLET, OUTFLOW, PERIODIC, WALL, FIRST_ORDER, SECOND_ORDER, RLMP,
                           make_grid, make_params, make_pert)

pytestmark = pytest.mark.gpu


def bits(a):
    """uint64 view with NaNs canonicalised (NaN payload/sign bits are not
    reproducible across compilers or devices and are not compared)."""
    a = np.array(a, np.float64)
    a[np.isnan(a)] = np.nan
    return a.view(np.uint64)


def assert_bitwise(got, want, what):
    if not np.array_equal(bits(got), bits(want)):
        d = np.abs(np.asarray(got) - np.asarray(want))
        bad = np.argwhere(bits(got) != bits(want))
        raise AssertionError(f"{what}: {len(bad)} entries differ, first at {bad[0].tolist()}, "
                             f"max |d| = {np.nanmax(d):.3e}")


# ---- config 1: 200x40, M=8, 200 steps of step(suggest_dt()) -----------------

def test_config1_bitwise_per_step(vlbm, orc, vo):
    """BASELINE configs[0]: every sample's u, pops and cell theta bit-identical
    to the oracle after steps 1, 2, 5, 20, 50, 100 and 200."""
    g = vlbm.Grid(200, 40)
    M = 8
    sim = vlbm.BatchSimulation.jet(g, n_samples=M, base_seed=42)
    refs = [orc.jet_sim(make_grid(200, 40), make_params(), make_pert(), 42, m) for m in range(M)]
    th_refs = [vo.jet_sim(make_grid(200, 40), make_params(), make_pert(), 42, m) for m in (0, 5)]
    done = 0
    for target in (1, 2, 5, 20, 50, 100, 200):
        sim.step(target - done)
        for r in refs:
            for _ in range(target - done):
                r.step(r.suggest_dt())
        done = target
        t, steps, status = sim.scalars()
        for m, r in enumerate(refs):
            assert steps[m] == target and status[m] == 0
            assert bits(t[m]) == bits(r.time), (m, t[m], r.time)
            u, p = r.get(pops=True)
            assert_bitwise(sim.state(m), u, f"u sample {m} step {target}")
            assert_bitwise(sim.populations(m), p, f"pops sample {m} step {target}")
    # cell theta of the last step (the restatement keeps it after the step)
    for m, r in zip((0, 5), th_refs):
        for _ in range(200):
            r.step(r.suggest_dt())
        assert_bitwise(sim.theta_cell(m), r.theta_cell(), f"theta sample {m}")


@pytest.mark.parametrize("nx,ny", [(4, 4), (37, 11), (33, 17), (66, 9), (97, 23)])
def test_ragged_grids_bitwise(vlbm, vo, nx, ny):
    """Grids that are not multiples of the 32x8 tiles (partial tiles, tiles
    touching several boundaries, the minimum 4x4 grid): the jet with square
    cells (x_max = 0.5 nx / ny), 30 steps, u, pops and cell theta
    bit-identical to the oracle."""
    x_max = 0.5 * nx / ny
    g = vlbm.Grid(nx, ny, x_max)
    sim = vlbm.BatchSimulation.jet(g, n_samples=2, base_seed=7)
    sim.step(30)
    for m in range(2):
        r = vo.jet_sim(make_grid(nx, ny, x_max), make_params(), make_pert(), 7, m)
        for _ in range(30):
            r.step(r.suggest_dt())
        u, p = r.get(pops=True)
        assert_bitwise(sim.state(m), u, f"u {nx}x{ny} sample {m}")
        assert_bitwise(sim.populations(m), p, f"pops {nx}x{ny} sample {m}")
        assert_bitwise(sim.theta_cell(m), r.theta_cell(), f"theta {nx}x{ny} sample {m}")


def test_run_samples_matches_run_sample(vlbm, orc):
    """run_samples == run_sample for every snapshot of 3 samples on the smoke
    grid 125x25 to t_end = 0.003 (times, diverged flags, steps, fields)."""
    times = [0.0, 0.00075, 0.0015, 0.00225, 0.003]
    g = vlbm.Grid(125, 25)
    res = vlbm.run_samples(g, vlbm.LatticeParams(), vlbm.GasParams(), vlbm.PerturbationParams(),
                           42, 0, 3, 0.02, times)
    for m in range(3):
        want = orc.run_sample(make_grid(125, 25), make_params(), make_pert(), 42, m, times)
        r = res[m]
        assert r.steps == want["steps"] and r.admissible == want["admissible"]
        for ti in range(len(times)):
            s = r.snapshots[ti]
            assert s.time == want["time"][ti] and s.diverged == want["diverged"][ti]
            assert s.sample_seed == want["seed"]
            assert_bitwise(s.data, want["fields"][ti], f"snapshot m={m} t={ti}")


def test_samples_not_in_lockstep(vlbm, orc):
    """Samples keep their own dt: a batch that starts at m0=5 reproduces the
    oracle's samples 5..8 (different step counts to the same target)."""
    g = vlbm.Grid(100, 20)
    sim = vlbm.BatchSimulation.jet(g, n_samples=4, base_seed=7, m0=5)
    sim.run_to(0.0004)
    t, steps, status = sim.scalars()
    for s in range(4):
        r = orc.jet_sim(make_grid(100, 20), make_params(), make_pert(), 7, 5 + s)
        n = 0
        while r.time < 0.0004 - 1e-12:
            r.step(min(r.suggest_dt(), 0.0004 - r.time))
            n += 1
        assert steps[s] == n
        assert bits(t[s]) == bits(r.time)
        assert_bitwise(sim.state(s), r.get(), f"sample {5 + s}")


# ---- boundary variants and limiter modes -------------------------------------

def smooth_field(nx, ny, x_max, gamma=1.4):
    """test_solver.cpp:31-48's smooth periodic field (conserved variables)."""
    dx = x_max / nx
    ly = 0.5
    x = (np.arange(nx) + 0.5) * dx
    y = -0.25 + (np.arange(ny) + 0.5) * dx
    X, Y = np.meshgrid(x, y)
    rho = 1.0 + 0.3 * np.sin(2 * np.pi * X / x_max) * np.cos(2 * np.pi * (Y + 0.25) / ly)
    v1 = 0.2 * np.cos(2 * np.pi * X / x_max)
    v2 = 0.1 * np.sin(2 * np.pi * (Y + 0.25) / ly)
    p = 1.0 + 0.2 * np.cos(2 * np.pi * X / x_max)
    E = p / (gamma - 1.0) + 0.5 * rho * (v1 * v1 + v2 * v2)
    return np.stack([rho, rho * v1, rho * v2, E])


BC_CASES = {
    "all_periodic": ((PERIODIC, PERIODIC, PERIODIC, PERIODIC), 32, 32),
    "periodic_x_wall_y": ((PERIODIC, PERIODIC, WALL, WALL), 32, 16),
    "outflow_x_periodic_y": ((OUTFLOW, OUTFLOW, PERIODIC, PERIODIC), 40, 8),
    "outflow_x_wall_y": ((OUTFLOW, OUTFLOW, WALL, WALL), 24, 12),
}


@pytest.mark.parametrize("case", list(BC_CASES))
@pytest.mark.parametrize("limiter", [RLMP, FIRST_ORDER, SECOND_ORDER])
def test_boundary_variants_bitwise(vlbm, orc, case, limiter):
    bc, nx, ny = BC_CASES[case]
    x_max = 0.5 * nx / ny
    init = smooth_field(nx, ny, x_max)
    # a spike so the limiter engages
    init[0, ny // 2, nx // 3] *= 3.0
    init[3, ny // 2, nx // 3] *= 3.0
    gamma = 1.4
    g = vlbm.Grid(nx, ny, x_max)
    lat = vlbm.LatticeParams(limiter=vlbm.Limiter(limiter))
    bcs = vlbm.Boundaries(*[vlbm.BcType(b) for b in bc])
    sim = vlbm.BatchSimulation(g, lat, vlbm.GasParams(gamma), bcs, init)
    r = orc.sim(make_grid(nx, ny, x_max), make_params(gamma=gamma, limiter=limiter, bc=bc), init)
    for n in (1, 4, 15):
        sim.step(n)
        for _ in range(n):
            r.step(r.suggest_dt())
        u, p = r.get(pops=True)
        assert_bitwise(sim.state(0), u, f"{case} u")
        assert_bitwise(sim.populations(0), p, f"{case} pops")


def test_inlet_generic_fields_and_alpha(vlbm, orc):
    """Generic construction with inlet rows and alpha = 0.25 (M5 = alpha u)."""
    nx, ny = 60, 12
    g = vlbm.Grid(nx, ny)
    pp = make_pert()
    seed, yc, zc = orc.draw_coefficients(3, 1, 10)
    rows = orc.inlet_rows(make_grid(nx, ny), yc, zc, pp)
    init = orc.initial_field(make_grid(nx, ny), yc, zc, pp, strip=0.1)
    lat = vlbm.LatticeParams(alpha=0.25)
    sim = vlbm.BatchSimulation(g, lat, vlbm.GasParams(), vlbm.Boundaries(), init, rows)
    r = orc.sim(make_grid(nx, ny), make_params(alpha=0.25), init, rows)
    sim.step(30)
    for _ in range(30):
        r.step(r.suggest_dt())
    u, p = r.get(pops=True)
    assert_bitwise(sim.state(0), u, "alpha u")
    assert_bitwise(sim.populations(0), p, "alpha pops")


def test_fixed_dt_steps(vlbm, orc):
    nx, ny = 40, 8
    init = smooth_field(nx, ny, 0.5 * nx / ny)
    g = vlbm.Grid(nx, ny, 0.5 * nx / ny)
    bcs = vlbm.Boundaries(*[vlbm.BcType.Periodic] * 4)
    sim = vlbm.BatchSimulation(g, vlbm.LatticeParams(), vlbm.GasParams(1.4), bcs, init)
    r = orc.sim(make_grid(nx, ny, 0.5 * nx / ny), make_params(gamma=1.4, bc=(3, 3, 3, 3)), init)
    dt = 0.7 * r.suggest_dt()
    sim.step(10, dt=dt)
    for _ in range(10):
        r.step(dt)
    assert_bitwise(sim.state(0), r.get(), "fixed dt")


def test_step_with_blending_random(vlbm, orc):
    """step_with_blending (solver.hpp:173-181) with random interface thetas."""
    nx, ny = 16, 16
    x_max = 0.5
    init = smooth_field(nx, ny, x_max)
    g = vlbm.Grid(nx, ny, x_max)
    bcs = vlbm.Boundaries(*[vlbm.BcType.Periodic] * 4)
    sim = vlbm.BatchSimulation(g, vlbm.LatticeParams(), vlbm.GasParams(1.4), bcs, init)
    r = orc.sim(make_grid(nx, ny, x_max), make_params(gamma=1.4, bc=(3, 3, 3, 3)), init)
    rng = np.random.default_rng(5)
    for _ in range(5):
        tx = rng.random((ny, nx + 1))
        ty = rng.random((ny + 1, nx))
        tx[:, nx] = tx[:, 0]
        ty[ny, :] = ty[0, :]
        dt = r.suggest_dt()
        sim.step_with_blending(tx, ty)
        r.step_with_blending(dt, tx, ty)
    assert_bitwise(sim.state(0), r.get(), "blended")


# ---- reference solver invariants, replayed on the kernel (test_solver.cpp) ----

def test_uniform_state_fixed_point(vlbm):
    """test_solver.cpp:75-95: a uniform state is invariant for any blending."""
    gamma = 1.4
    rho, v1, v2, p = 1.3, 0.4, -0.2, 0.9
    u0 = np.array([rho, rho * v1, rho * v2, p / (gamma - 1) + 0.5 * rho * (v1 * v1 + v2 * v2)])
    nx = ny = 16
    init = np.broadcast_to(u0[:, None, None], (4, ny, nx)).copy()
    g = vlbm.Grid(nx, ny, 0.5)
    bcs = vlbm.Boundaries(*[vlbm.BcType.Periodic] * 4)
    for alpha in (0.0, 0.25):
        sim = vlbm.BatchSimulation(g, vlbm.LatticeParams(alpha=alpha), vlbm.GasParams(gamma), bcs,
                                   init)
        rng = np.random.default_rng(5)
        for _ in range(10):
            tx = rng.random((ny, nx + 1))
            ty = rng.random((ny + 1, nx))
            tx[:, nx] = tx[:, 0]
            ty[ny, :] = ty[0, :]
            sim.step_with_blending(tx, ty)
        np.testing.assert_allclose(sim.state(0), init, rtol=1e-13)


def test_periodic_conservation(vlbm):
    """test_solver.cpp:97-112: periodic RLMP run conserves all four totals."""
    nx = ny = 32
    init = smooth_field(nx, ny, 0.5)
    g = vlbm.Grid(nx, ny, 0.5)
    bcs = vlbm.Boundaries(*[vlbm.BcType.Periodic] * 4)
    sim = vlbm.BatchSimulation(g, vlbm.LatticeParams(), vlbm.GasParams(1.4), bcs, init)
    before = init.reshape(4, -1).sum(1)
    sim.step(50)
    after = sim.state(0).reshape(4, -1).sum(1)
    scale = np.maximum(np.abs(before), 1.0)
    assert np.all(np.abs(after - before) / scale <= 1e-12)


def test_mirror_symmetry_unperturbed_jet(vlbm):
    """test_solver.cpp:228-263: amplitude 0 jet stays mirror symmetric."""
    g = vlbm.Grid(100, 20)
    pp = vlbm.PerturbationParams(amplitude=0.0)
    res = vlbm.run_samples(g, vlbm.LatticeParams(), vlbm.GasParams(), pp, 1, 0, 1, 0.0, [0.0005])
    s = res[0].snapshots[0].data
    assert res[0].admissible
    scale = np.abs(s).reshape(4, -1).max(1)
    m = s[:, ::-1, :]
    assert np.all(np.abs(s[0] - m[0]) <= 1e-10 * scale[0])
    assert np.all(np.abs(s[1] - m[1]) <= 1e-10 * scale[1])
    assert np.all(np.abs(s[2] + m[2]) <= 1e-10 * scale[1])
    assert np.all(np.abs(s[3] - m[3]) <= 1e-10 * scale[3])
    assert np.abs(s[0] - 0.5).sum() > 1.0


def test_divergence_flags_like_run_sample(vlbm, orc):
    """A blow-up (tiny safety factor, no limiter) is an outcome, not an error:
    the sample stops, later snapshots are placeholders with the sample's own
    time, exactly as run_sample (solver.hpp:645-666)."""
    times = [0.0, 0.0002, 0.0004]
    g = vlbm.Grid(60, 12)
    lat = vlbm.LatticeParams(limiter=vlbm.Limiter.SecondOrder, safety=1.0)
    res = vlbm.run_samples(g, lat, vlbm.GasParams(), vlbm.PerturbationParams(), 42, 0, 2, 0.02,
                           times)
    for m in range(2):
        want = orc.run_sample(make_grid(60, 12), make_params(limiter=SECOND_ORDER, safety=1.0),
                             make_pert(), 42, m, times)
        assert res[m].admissible == want["admissible"]
        assert res[m].steps == want["steps"]
        for ti in range(3):
            s = res[m].snapshots[ti]
            assert bits(s.time) == bits(want["time"][ti])
            assert s.diverged == want["diverged"][ti]
            assert_bitwise(s.data, want["fields"][ti], f"diverging sample {m} t{ti}")


def test_certified_bisection_audit_and_late_time_parity(vlbm, orc):
    """The limiter's certified bisection (rlmp.cuh) skips the vertex floors
    only where a rigorous rounding bound proves they pass.  With the audit on,
    every certified step is re-run in full on the GPU: zero disagreements over
    a whole late-time run, and the fields stay bit-identical to the oracle."""
    g = vlbm.Grid(300, 60)
    sim = vlbm.BatchSimulation.jet(g, n_samples=6, base_seed=42)
    sim.set_audit(True)
    sim.run_to(0.0009)
    assert sim.audit_mismatches() == 0
    t, steps, status = sim.scalars()
    for m in (0, 5):
        r = orc.jet_sim(make_grid(300, 60), make_params(), make_pert(), 42, m)
        while r.time < 0.0009 - 1e-12:
            r.step(min(r.suggest_dt(), 0.0009 - r.time))
        assert steps[m] == r.steps
        assert_bitwise(sim.state(m), r.get(), f"late-time sample {m}")


@pytest.mark.parametrize("cap", ["1536", "0"])
def test_limiter_queue_overflow_paths_bitwise(vlbm, orc, monkeypatch, cap):
    """A limiter queue far smaller than the hard cells (VLBM_HQ_CAP test hook):
    CTAs whose cells do not fit finish them in place (tile pass, stage,
    bisection tail) -- and with no queue at all (cap 0) every hard cell is
    finished by its tile thread.  Fields bit-identical to the oracle at late
    time."""
    monkeypatch.setenv("VLBM_HQ_CAP", cap)
    g = vlbm.Grid(200, 40)
    sim = vlbm.BatchSimulation.jet(g, n_samples=4, base_seed=42)
    sim.run_to(0.0008)
    t, steps, status = sim.scalars()
    for m in (0, 3):
        r = orc.jet_sim(make_grid(200, 40), make_params(), make_pert(), 42, m)
        while r.time < 0.0008 - 1e-12:
            r.step(min(r.suggest_dt(), 0.0008 - r.time))
        assert steps[m] == r.steps
        assert_bitwise(sim.state(m), r.get(), f"overflow cap {cap} sample {m}")
    q = sim.queue_stats()
    if cap != "0":  # the overflow counter sees the cells finished in place
        assert q["capacity"] == int(cap) and q["overflow"] > 0 and q["peak_hard"] > int(cap)


@pytest.mark.parametrize("groups,cap", [(3, None), (8, None), (3, "1536")])
def test_serial_sample_groups_bitwise(vlbm, orc, monkeypatch, groups, cap):
    """Serial sample groups (the configs[2] layout: groups of samples marched
    one after another on one stream, sharing one set of limiter queues that
    covers every cell of a group): fields, times and step counts
    bit-identical to the reference at late time; no overflow when the queue
    covers a group (the overflow counter counts the cells finished in place
    when it does not)."""
    monkeypatch.setenv("VLBM_SERIAL_GROUPS", str(groups))
    if cap:
        monkeypatch.setenv("VLBM_HQ_CAP", cap)
    g = vlbm.Grid(200, 40)
    sim = vlbm.BatchSimulation.jet(g, n_samples=8, base_seed=42)
    sim.run_to(0.0008)
    t, steps, status = sim.scalars()
    q = sim.queue_stats()
    assert q["groups"] == groups and q["passes"] > 0 and q["peak_hard"] > 0
    if cap:
        assert q["overflow"] > 0
    else:
        assert q["overflow"] == 0 and q["capacity"] >= 8 // groups * 8000
    for m in (0, 4, 7):
        r = orc.jet_sim(make_grid(200, 40), make_params(), make_pert(), 42, m)
        while r.time < 0.0008 - 1e-12:
            r.step(min(r.suggest_dt(), 0.0008 - r.time))
        assert steps[m] == r.steps and bits(t[m]) == bits(r.time)
        assert_bitwise(sim.state(m), r.get(), f"serial groups {groups} sample {m}")


@pytest.mark.parametrize("limiter", [RLMP, FIRST_ORDER])
def test_sod_tube_bitwise(vlbm, orc, limiter):
    """test_riemann.cpp's Sod tube (gamma 1.4; left rho 1, p 1, right rho
    0.125, p 0.1, at rest) on a 400x4 strip with outflow x and periodic y:
    shock, contact and rarefaction through the limiter; fields bit-identical
    to the oracle after 300 steps, density positive."""
    nx, ny = 400, 4
    x_max = 0.5 * nx / ny
    gamma = 1.4
    x = (np.arange(nx) + 0.5) * (x_max / nx)
    left = x < 0.5 * x_max
    rho = np.where(left, 1.0, 0.125)
    p = np.where(left, 1.0, 0.1)
    init = np.zeros((4, ny, nx))
    init[0] = rho[None, :]
    init[3] = (p / (gamma - 1.0))[None, :]
    bc = (OUTFLOW, OUTFLOW, PERIODIC, PERIODIC)
    g = vlbm.Grid(nx, ny, x_max)
    lat = vlbm.LatticeParams(limiter=vlbm.Limiter(limiter))
    bcs = vlbm.Boundaries(*[vlbm.BcType(b) for b in bc])
    sim = vlbm.BatchSimulation(g, lat, vlbm.GasParams(gamma), bcs, init)
    r = orc.sim(make_grid(nx, ny, x_max), make_params(gamma=gamma, limiter=limiter, bc=bc), init)
    sim.step(300)
    for _ in range(300):
        r.step(r.suggest_dt())
    u, pops = r.get(pops=True)
    assert_bitwise(sim.state(0), u, "sod u")
    assert_bitwise(sim.populations(0), pops, "sod pops")
    assert sim.state(0)[0].min() > 0.0


@pytest.mark.parametrize("kappa,safety,floor,cons", [(0.25, 2.5, 1e-6, 1), (0.9, 3.0, 1e-9, 0),
                                                      (0.0, 2.0, 1e-7, 1)])
def test_jet_lattice_parameters_bitwise(vlbm, orc, kappa, safety, floor, cons):
    """Non-default lattice parameters of the jet (lattice.hpp:13-35): RLMP
    relaxation kappa, the dt safety factor, the positivity floor and the
    conservative (hypot) signal-speed bound; 60 steps of 2 samples, fields
    and times bit-identical to the oracle."""
    g = vlbm.Grid(200, 40)
    lat = vlbm.LatticeParams(safety=safety, rlmp_relaxation=kappa, positivity_floor=floor,
                             conservative_bound=bool(cons))
    sim = vlbm.BatchSimulation.jet(g, lat, n_samples=2, base_seed=3)
    sim.step(60)
    t, _, _ = sim.scalars()
    p = make_params(safety=safety, kappa=kappa, floor=floor, conservative_bound=cons)
    for m in range(2):
        r = orc.jet_sim(make_grid(200, 40), p, make_pert(), 3, m)
        for _ in range(60):
            r.step(r.suggest_dt())
        assert bits(t[m]) == bits(r.time)
        u, pops = r.get(pops=True)
        assert_bitwise(sim.state(m), u, f"u sample {m}")
        assert_bitwise(sim.populations(m), pops, f"pops sample {m}")


def test_jet_perturbation_parameters_bitwise(vlbm, orc):
    """Non-default jet / perturbation parameters (perturbation.hpp:16-31:
    amplitude, modes, decay, jet radius, density and speed, ambient state)
    and inlet strip width: 50 steps of 3 samples, fields and times
    bit-identical to the oracle."""
    kw = dict(amplitude=0.3, modes=5, decay_exponent=1.5, r_jet=0.08, rho_jet_bar=3.0,
              rho_amb=0.7, p_amb=0.5, v_jet=500.0)
    g = vlbm.Grid(160, 32)
    pp = vlbm.PerturbationParams(**kw)
    sim = vlbm.BatchSimulation.jet(g, vlbm.LatticeParams(), vlbm.GasParams(), pp, base_seed=9,
                                   m0=4, n_samples=3, strip_width=0.05)
    sim.step(50)
    t, _, _ = sim.scalars()
    for s in range(3):
        r = orc.jet_sim(make_grid(160, 32), make_params(), make_pert(**kw), 9, 4 + s, strip=0.05)
        for _ in range(50):
            r.step(r.suggest_dt())
        assert bits(t[s]) == bits(r.time)
        u, pops = r.get(pops=True)
        assert_bitwise(sim.state(s), u, f"u sample {4 + s}")
        assert_bitwise(sim.populations(s), pops, f"pops sample {4 + s}")


def test_config2_first_50_steps_bitwise(vlbm, orc):
    """BASELINE configs[1]'s parity statement: per-sample fields of the
    1000x200 jet equal the CPU oracle for the first 50 steps (here every bit,
    4 of the 64 samples: 0, 21, 42, 63 of a 64-sample batch)."""
    g = vlbm.Grid(1000, 200)
    sim = vlbm.BatchSimulation.jet(g, n_samples=64, base_seed=42)
    sim.step(50)
    t, steps, _ = sim.scalars()
    for m in (0, 21, 42, 63):
        r = orc.jet_sim(make_grid(1000, 200), make_params(), make_pert(), 42, m)
        for _ in range(50):
            r.step(r.suggest_dt())
        assert steps[m] == 50 and bits(t[m]) == bits(r.time)
        u, pops = r.get(pops=True)
        assert_bitwise(sim.state(m), u, f"u sample {m}")
        assert_bitwise(sim.populations(m), pops, f"pops sample {m}")


MIXED_BCS = {
    "inlet_outflow_x_inlet_as_wrap_y": (INLET, OUTFLOW, INLET, INLET),
    "outflow_x_outflow_wrap_wall_y": (OUTFLOW, OUTFLOW, OUTFLOW, WALL),
    "inlet_outflow_x_wall_inlet_wrap_y": (INLET, OUTFLOW, WALL, INLET),
    "periodic_x_outflow_wrap_y": (PERIODIC, PERIODIC, OUTFLOW, OUTFLOW),
}


@pytest.mark.parametrize("case", list(MIXED_BCS))
def test_mixed_boundaries_bitwise_vs_reference(vlbm, ref, case):
    """Boundary combinations the reference accepts beyond the jet's: a y side
    that is neither wall nor periodic wraps its ghosts (solver.hpp:274-285)
    while its boundary faces stay non-periodic for interface_theta (:513),
    also next to a wall on the other y side (fill_ghosts' corner order).
    Checked against the reference itself (oracle/_ref), 25 steps."""
    bc = MIXED_BCS[case]
    nx, ny = 60, 12
    pp = make_pert()
    seed, yc, zc = ref.draw_coefficients(5, 2, 10)
    rows = ref.inlet_rows(make_grid(nx, ny), yc, zc, pp)
    init = ref.initial_field(make_grid(nx, ny), yc, zc, pp, strip=0.1)
    init[0, 3, 50] *= 2.0  # something for the wraps and mirrors to carry
    g = vlbm.Grid(nx, ny)
    bcs = vlbm.Boundaries(*[vlbm.BcType(b) for b in bc])
    sim = vlbm.BatchSimulation(g, vlbm.LatticeParams(), vlbm.GasParams(), bcs, init, rows)
    r = ref.sim(make_grid(nx, ny), make_params(bc=bc), init, rows)
    for n in (1, 24):
        sim.step(n)
        for _ in range(n):
            r.step(r.suggest_dt())
        u, p = r.get(pops=True)
        assert_bitwise(sim.state(0), u, f"{case} u")
        assert_bitwise(sim.populations(0), p, f"{case} pops")


@pytest.mark.parametrize("bc", [(WALL, OUTFLOW, WALL, WALL), (INLET, INLET, WALL, WALL),
                                (INLET, WALL, WALL, WALL)])
def test_unsupported_x_boundaries_rejected(vlbm, bc):
    """x walls and an x_max inlet are rejected as the reference rejects them
    (std::invalid_argument -> ValueError), before any march."""
    g = vlbm.Grid(16, 4)
    init = np.zeros((4, 4, 16))
    init[0], init[3] = 1.0, 1.0
    bcs = vlbm.Boundaries(*[vlbm.BcType(b) for b in bc])
    with pytest.raises(ValueError):
        vlbm.BatchSimulation(g, vlbm.LatticeParams(), vlbm.GasParams(), bcs, init,
                             np.ones((4, 4)))


@pytest.mark.parametrize("alpha", [0.5, 0.9])
def test_rest_population_weight_bitwise(vlbm, orc, alpha):
    """alpha in (0, 1) (test_lattice.cpp:31-49: M5 = alpha u, w = (1 - alpha)/4):
    periodic smooth field with a spike, RLMP, 10 steps bit-identical to the
    oracle.  (With this spike alpha = 0.9 becomes inadmissible at step 14 and
    alpha = 1 at step 11; the batch then stops the sample as run_sample does,
    while a bare Simulation::step keeps stepping NaNs.)"""
    nx, ny = 32, 16
    x_max = 0.5 * nx / ny
    init = smooth_field(nx, ny, x_max)
    init[0, 5, 7] *= 2.5
    bc = (PERIODIC, PERIODIC, PERIODIC, PERIODIC)
    g = vlbm.Grid(nx, ny, x_max)
    lat = vlbm.LatticeParams(alpha=alpha)
    bcs = vlbm.Boundaries(*[vlbm.BcType(b) for b in bc])
    sim = vlbm.BatchSimulation(g, lat, vlbm.GasParams(1.4), bcs, init)
    r = orc.sim(make_grid(nx, ny, x_max), make_params(gamma=1.4, alpha=alpha, bc=bc), init)
    sim.step(10)
    for _ in range(10):
        r.step(r.suggest_dt())
    u, p = r.get(pops=True)
    assert_bitwise(sim.state(0), u, f"alpha {alpha} u")
    assert_bitwise(sim.populations(0), p, f"alpha {alpha} pops")


@pytest.mark.parametrize("limiter", [RLMP, FIRST_ORDER])
def test_graph_replay_matches_direct_launches(vlbm, orc, monkeypatch, limiter):
    """Chunks after a call's first replay as one captured CUDA graph
    (capi.cu march_loop).  With graphs off (VLBM_GRAPHS=0) the same calls --
    run_to over many chunks, two targets, then step(n) -- give identical
    bits, step counts and launch counts; both match the oracle."""
    g = vlbm.Grid(200, 40)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("VLBM_GRAPHS", flag)
        sim = vlbm.BatchSimulation.jet(g, vlbm.LatticeParams(limiter=vlbm.Limiter(limiter)),
                                       n_samples=3, base_seed=42)
        sim.run_to(0.0003)
        sim.run_to(0.0005)
        sim.step(37)
        out[flag] = ([sim.state(m) for m in range(3)], sim.scalars()[1].copy(),
                     sim.stats()["launches"])
        sim.close()
    for m in range(3):
        assert_bitwise(out["1"][0][m], out["0"][0][m], f"graph vs direct sample {m}")
    assert list(out["1"][1]) == list(out["0"][1])
    assert out["1"][2] == out["0"][2]
    r = orc.jet_sim(make_grid(200, 40), make_params(limiter=limiter), make_pert(), 42, 2)
    for target in (0.0003, 0.0005):
        while r.time < target - 1e-12:
            r.step(min(r.suggest_dt(), target - r.time))
    for _ in range(37):
        r.step(r.suggest_dt())
    assert out["1"][1][2] == r.steps
    assert_bitwise(out["1"][0][2], r.get(), "graph replay vs oracle")


def test_cert_side_stream_matches_in_line(vlbm, orc, monkeypatch):
    """k_bisect_cert on its side stream (default) and in line on the main
    stream (VLBM_CERT_SIDE=0) give the same bits at late time, where all
    three bisection kernels have work; both match the oracle."""
    g = vlbm.Grid(200, 40)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("VLBM_CERT_SIDE", flag)
        sim = vlbm.BatchSimulation.jet(g, n_samples=4, base_seed=42)
        sim.run_to(0.0008)
        out[flag] = ([sim.state(m) for m in range(4)], sim.scalars()[1].copy())
        sim.close()
    for m in range(4):
        assert_bitwise(out["1"][0][m], out["0"][0][m], f"side vs in-line sample {m}")
    assert list(out["1"][1]) == list(out["0"][1])
    r = orc.jet_sim(make_grid(200, 40), make_params(), make_pert(), 42, 1)
    while r.time < 0.0008 - 1e-12:
        r.step(min(r.suggest_dt(), 0.0008 - r.time))
    assert out["1"][1][1] == r.steps
    assert_bitwise(out["1"][0][1], r.get(), "side stream vs oracle")


@pytest.mark.parametrize("nx,ny,strip", [(200, 40, 0.02), (37, 11, 0.3), (1000, 200, 0.02),
                                         (64, 16, 0.0), (50, 10, 5.0)])
def test_device_initial_field_bitwise(vlbm, orc, nx, ny, strip):
    """The batch's initial field (inlet rows on the host, ambient + wedge laid
    out on the device) and its equilibrium populations equal the reference's
    initial_field + Simulation ctor (perturbation.hpp:106-122, solver.hpp:61-100)
    bit for bit: thin, wide (strip 5: every row entirely wedge) and empty
    (strip 0) wedges, ragged grids, several samples."""
    x_max = 0.5 * nx / ny  # square cells (2.5 on the 5:1 jet grids)
    g = vlbm.Grid(nx, ny, x_max)
    S = 3
    sim = vlbm.BatchSimulation.jet(g, n_samples=S, base_seed=42, m0=5, strip_width=strip)
    for s in range(S):
        r = orc.jet_sim(make_grid(nx, ny, x_max), make_params(), make_pert(), 42, 5 + s,
                        strip=strip)
        u, p = r.get(pops=True)
        assert_bitwise(sim.state(s), u, f"initial u {nx}x{ny} strip {strip} sample {s}")
        assert_bitwise(sim.populations(s), p, f"initial pops {nx}x{ny} strip {strip} sample {s}")
