"""B200-native probabilistic VLBM hot path (arXiv 2605.25282).

The Monte-Carlo VLBM march of the Mach-2000 jet and its W1/L1
post-processing as hand-written sm_100a kernels behind the C ABI of
include/vlbm_b200.h.  See DESIGN.md.
"""
from .vlbm import (  # noqa: F401
    BatchSimulation, BcType, Boundaries, FieldSnapshot, GasParams, Grid, LatticeParams, Limiter,
    ModeCoefficients, PerturbationParams, SampleResult, draw_coefficients, ensemble_moments,
    inlet_rows, lib, restrict_field, run_samples, strong_error, wasserstein1,
)
