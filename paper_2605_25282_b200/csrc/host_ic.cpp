// host_ic.cpp — per-sample initial conditions on the host (integer-exact
// splitmix64 coefficients + the inlet profile through the host libm).
//
// The inlet profile uses cos/sin/pow; evaluating it on the host with the same
// glibc as the reference keeps every inlet row bit-identical to the
// reference's inlet_state (a 1-ulp device-libm difference would diverge the
// march within ~5 steps).  Built with g++ -O2
// -ffp-contract=off (no FMA), like the reference's default x86-64 build.
#include <cmath>
#include <cstring>

#include "internal.h"

namespace vlbm_impl {

double grid_dx(const vlbm_grid& g) { return g.x_max / g.nx; }                       // grid.hpp:21
double y_center(const vlbm_grid& g, int j) { return g.y_min + (j + 0.5) * grid_dx(g); }  // :23
static double x_center(const vlbm_grid& g, int i) { return (i + 0.5) * grid_dx(g); }  // :22

// Grid::validate, grid.hpp:28-35
int validate_grid(const vlbm_grid& g) {
  if (g.nx < 4 || g.ny < 4) return set_error(VLBM_E_INVALID, "Grid: nx, ny must be >= 4");
  const double dxx = g.x_max / g.nx;
  const double dxy = (g.y_max - g.y_min) / g.ny;
  if (std::abs(dxx - dxy) > 1e-12 * dxx)
    return set_error(VLBM_E_INVALID, "Grid: cells are not square (dx mismatch between x and y)");
  return VLBM_OK;
}

// LatticeParams::validate (lattice.hpp:28-33) + Simulation ctor checks
// (solver.hpp:69-75, 253-267).
int validate_params(const vlbm_params& p) {
  if (p.alpha < 0.0 || p.alpha > 1.0) return set_error(VLBM_E_INVALID, "alpha must be in [0,1]");
  if (p.safety < 1.0) return set_error(VLBM_E_INVALID, "safety must be >= 1");
  if (p.rlmp_relaxation < 0.0) return set_error(VLBM_E_INVALID, "rlmp_relaxation must be >= 0");
  if (!(p.positivity_floor > 0.0))
    return set_error(VLBM_E_INVALID, "positivity_floor must be > 0");
  if (p.limiter < 0 || p.limiter > 2) return set_error(VLBM_E_INVALID, "unknown limiter");
  for (int k = 0; k < 4; ++k)
    if (p.bc[k] < 0 || p.bc[k] > 3) return set_error(VLBM_E_INVALID, "unknown boundary type");
  if ((p.bc[0] == VLBM_BC_PERIODIC) != (p.bc[1] == VLBM_BC_PERIODIC) ||
      (p.bc[2] == VLBM_BC_PERIODIC) != (p.bc[3] == VLBM_BC_PERIODIC))
    return set_error(VLBM_E_INVALID, "Simulation: periodic sides must be paired");
  if (p.bc[0] == VLBM_BC_WALL)
    return set_error(VLBM_E_INVALID, "Simulation: walls are supported on y sides only");
  if (p.bc[1] == VLBM_BC_INLET || p.bc[1] == VLBM_BC_WALL)
    return set_error(VLBM_E_INVALID, "Simulation: unsupported x_max boundary");
  // y sides: a wall mirrors; any other type wraps (fill_ghosts, solver.hpp:
  // 270-285), while only a Periodic pair makes the boundary faces periodic for
  // interface_theta (:513) -- the reference accepts Inlet / Outflow there.
  // The x-side rejections above surface in the reference at the first
  // fill_ghosts (:254, :268); here already when the batch is created.
  return VLBM_OK;
}

// PerturbationParams::validate, perturbation.hpp:26-30
int validate_perturbation(const vlbm_perturbation& pp) {
  if (pp.amplitude < 0) return set_error(VLBM_E_INVALID, "amplitude must be >= 0");
  if (pp.modes < 1) return set_error(VLBM_E_INVALID, "modes must be >= 1");
  if (pp.decay_exponent <= 0) return set_error(VLBM_E_INVALID, "decay_exponent must be > 0");
  return VLBM_OK;
}

// splitmix64 (random.hpp:10-38): output n of the stream seeded with `seed`
// is the finalizer of seed + (n + 1) * 0x9E3779B97F4A7C15.
static inline uint64_t finalize(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline uint64_t mix64(uint64_t z) { return finalize(z + 0x9E3779B97F4A7C15ull); }

// taper_window (perturbation.hpp:57-61) and density_perturbation (:65-77).
static double taper(double ybar) {
  if (std::abs(ybar) >= 1.0) return 0.0;
  const double c = std::cos(0.5 * M_PI * ybar);
  return c * c;
}

static double density(double y, int K, const double* yc, const double* zc,
                      const vlbm_perturbation& pp) {
  const double ybar = y / pp.r_jet;
  const double w = taper(ybar);
  double sum = 0.0;
  for (int k = 1; k <= K; ++k) {
    const double weight = std::pow(static_cast<double>(k), -pp.decay_exponent);
    sum += weight * (yc[k - 1] * std::cos(k * M_PI * ybar) + zc[k - 1] * std::sin(k * M_PI * ybar));
  }
  return pp.rho_jet_bar * (1.0 + pp.amplitude * sum * w);
}

// inlet_state, perturbation.hpp:87-95
void inlet_state(double y, int K, const double* yc, const double* zc,
                 const vlbm_perturbation& pp, double gamma, double* out) {
  if (std::abs(y) <= pp.r_jet) {
    const double rho = density(y, K, yc, zc, pp);
    out[0] = rho;
    out[1] = rho * pp.v_jet;
    out[2] = 0.0;
    out[3] = pp.p_amb / (gamma - 1.0) + 0.5 * rho * pp.v_jet * pp.v_jet;
  } else {
    out[0] = pp.rho_amb;
    out[1] = 0.0;
    out[2] = 0.0;
    out[3] = pp.p_amb / (gamma - 1.0);
  }
}

// initial_field, perturbation.hpp:106-122 (ambient plus the inlet wedge).
void initial_field(const vlbm_grid& g, int K, const double* yc, const double* zc,
                   const vlbm_perturbation& pp, double gamma, double strip, double* out) {
  const size_t n = static_cast<size_t>(g.nx) * g.ny;
  const double amb[4] = {pp.rho_amb, 0.0, 0.0, pp.p_amb / (gamma - 1.0)};
  for (int k = 0; k < 4; ++k)
    for (size_t c = 0; c < n; ++c) out[k * n + c] = amb[k];
  const double height = g.y_max - g.y_min;
  for (int j = 0; j < g.ny; ++j) {
    const double y = y_center(g, j);
    double u_in[4];
    inlet_state(y, K, yc, zc, pp, gamma, u_in);
    const double w = strip * (0.5 + 5.0 * (y - g.y_min) / height);
    for (int i = 0; i < g.nx && x_center(g, i) < w; ++i)
      for (int k = 0; k < 4; ++k) out[k * n + static_cast<size_t>(j) * g.nx + i] = u_in[k];
  }
}

// The wedge of initial_field row by row: counts[j] = the number of leading
// cells with x_center(i) < w(y_j) (perturbation.hpp:116-119, the same
// expressions), so the device can lay out ambient + wedge without libm.
void wedge_counts(const vlbm_grid& g, double strip, int* counts) {
  const double height = g.y_max - g.y_min;
  for (int j = 0; j < g.ny; ++j) {
    const double y = y_center(g, j);
    const double w = strip * (0.5 + 5.0 * (y - g.y_min) / height);
    int n = 0;
    while (n < g.nx && x_center(g, n) < w) ++n;
    counts[j] = n;
  }
}

}  // namespace vlbm_impl

extern "C" {

// draw_coefficients, perturbation.hpp:42-54; sample_seed, random.hpp:42-44.
uint64_t vlbm_draw_coefficients(uint64_t base_seed, uint64_t m, int K, double* y, double* z) {
  using vlbm_impl::finalize;
  using vlbm_impl::mix64;
  const uint64_t seed = mix64(base_seed ^ mix64(m + 1));
  uint64_t state = seed;
  for (int k = 0; k < 2 * K; ++k) {
    state += 0x9E3779B97F4A7C15ull;
    const double unit = static_cast<double>(finalize(state) >> 11) * 0x1.0p-53;
    const double v = 2.0 * unit - 1.0;
    if (k & 1)
      z[k >> 1] = v;
    else
      y[k >> 1] = v;
  }
  return seed;
}

int vlbm_inlet_rows(const vlbm_grid* g, const vlbm_perturbation* pp, double gamma,
                    const double* yc, const double* zc, double* out) {
  if (int rc = vlbm_impl::validate_perturbation(*pp)) return rc;
  for (int j = 0; j < g->ny; ++j)
    vlbm_impl::inlet_state(vlbm_impl::y_center(*g, j), pp->modes, yc, zc, *pp, gamma, out + 4 * j);
  return VLBM_OK;
}

// Reference defaults: euler.hpp:10, lattice.hpp:13-25, solver.hpp:25-28,585-586.
void vlbm_default_params(vlbm_params* p) {
  p->gamma = 5.0 / 3.0;
  p->alpha = 0.0;
  p->safety = 2.0;
  p->rlmp_relaxation = 0.5;
  p->positivity_floor = 1e-7;
  p->limiter = VLBM_LIMITER_RLMP;
  p->conservative_bound = 0;
  p->rho_ref = 0.5;
  p->p_ref = 0.4127;
  p->bc[0] = VLBM_BC_INLET;
  p->bc[1] = VLBM_BC_OUTFLOW;
  p->bc[2] = VLBM_BC_WALL;
  p->bc[3] = VLBM_BC_WALL;
}

// perturbation.hpp:16-24
void vlbm_default_perturbation(vlbm_perturbation* pp) {
  pp->amplitude = 0.1;
  pp->modes = 10;
  pp->decay_exponent = 2.0;
  pp->r_jet = 0.05;
  pp->rho_jet_bar = 5.0;
  pp->rho_amb = 0.5;
  pp->p_amb = 0.4127;
  pp->v_jet = 800.0;
}

// config.hpp:27-29
void vlbm_default_grid(vlbm_grid* g, int nx, int ny) {
  g->nx = nx;
  g->ny = ny;
  g->x_max = 2.5;
  g->y_min = -0.25;
  g->y_max = 0.25;
}

}  // extern "C"
