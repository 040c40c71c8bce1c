"""The C-ABI boundary without a GPU (-m "not gpu"): libvlbm_b200.so loads,
exports every entry point include/vlbm_b200.h declares, its host-side IC
(splitmix64 + host libm) is bit-identical to the oracle, and the march fails
loudly -- there is no CPU fallback -- when no CUDA device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vlbm_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vlbm_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import paper_2605_25282_b200 as v
    return v.lib()


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump), not PTX for a JIT."""
    import shutil
    import subprocess
    from paper_2605_25282_b200.vlbm import LIB_PATH
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_abi_version_and_defaults(lib):
    import paper_2605_25282_b200 as v
    assert lib.vlbm_abi_version() == 1
    p = v.vlbm._Params()
    lib.vlbm_default_params.argtypes = [C.POINTER(v.vlbm._Params)]
    lib.vlbm_default_params(C.byref(p))
    # lattice.hpp:13-25, euler.hpp:10, solver.hpp:585-586, 25-28
    assert (p.gamma, p.alpha, p.safety, p.rlmp_relaxation, p.positivity_floor) == \
        (5.0 / 3.0, 0.0, 2.0, 0.5, 1e-7)
    assert p.limiter == 2 and (p.rho_ref, p.p_ref) == (0.5, 0.4127)
    assert list(p.bc) == [0, 1, 2, 2]


def test_host_ic_matches_oracle_bitwise(vo):
    import paper_2605_25282_b200 as v
    g = v.Grid(200, 40)
    pp = v.PerturbationParams()
    for base, m in [(42, 0), (42, 5), (1, 999), (12345, 77)]:
        c = v.draw_coefficients(base, m, 10)
        seed, y, z = vo.draw_coefficients(base, m, 10)
        assert c.seed == seed
        assert np.array_equal(c.y_coeffs.view(np.uint64), y.view(np.uint64))
        assert np.array_equal(c.z_coeffs.view(np.uint64), z.view(np.uint64))
        rows = v.inlet_rows(g, c, pp)
        from oracle.oracle import make_grid, make_pert
        want = vo.inlet_rows(make_grid(200, 40), y, z, make_pert())
        assert np.array_equal(rows.view(np.uint64), want.view(np.uint64))


def test_inlet_rows_many_y_values_bitwise(vo):
    """The inlet profile goes through host libm cos/sin/pow: identical bits to
    the oracle (and hence the reference) on many grids."""
    import paper_2605_25282_b200 as v
    from oracle.oracle import make_grid, make_pert
    for nx, ny in [(125, 25), (250, 50), (500, 100), (1000, 200), (2000, 400), (4000, 800)]:
        c = v.draw_coefficients(42, nx, 10)
        got = v.inlet_rows(v.Grid(nx, ny), c, v.PerturbationParams())
        want = vo.inlet_rows(make_grid(nx, ny), c.y_coeffs, c.z_coeffs, make_pert())
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (nx, ny)


def test_validation_mirrors_reference_errors():
    import paper_2605_25282_b200 as v
    with pytest.raises(ValueError):
        v.draw_coefficients(1, 0, 0)  # draw_coefficients: K must be >= 1
    with pytest.raises(ValueError):
        v.restrict_field(np.zeros((4, 3, 4)))  # fine dimensions must be even
    with pytest.raises(ValueError):
        v.strong_error(np.zeros((2, 4, 2, 2)), np.zeros((3, 4, 2, 2)))
    with pytest.raises(ValueError):
        v.wasserstein1(np.zeros((0, 4, 2, 2)), np.zeros((0, 4, 2, 2)))
    with pytest.raises(ValueError):
        v.run_samples(v.Grid(8, 8), v.LatticeParams(), v.GasParams(), v.PerturbationParams(),
                      1, 0, 1, 0.0, [0.1, 0.05])


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device behaviour")
def test_march_fails_loudly_without_a_device():
    import paper_2605_25282_b200 as v
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        v.BatchSimulation.jet(v.Grid(40, 8))
    with pytest.raises(RuntimeError):
        v.wasserstein1(np.ones((2, 4, 2, 2)), np.ones((2, 4, 2, 2)))
