/* oracle/vlbm_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never shipped).
 *
 * Plain-C restatement of the reference's VLBM march and W1/L1 metrics, written
 * from the reference's published algorithm.  Every function cites the
 * reference file:line it follows (paths under /root/reference/proj/include/
 * vlbm/).  It reproduces the reference's exact IEEE operation sequence
 * (association order, std::min/std::max tie semantics, the +0 of the alpha*u
 * term) so that it is bit-identical to the reference; tests/test_oracle_pin.py
 * proves that against oracle/_ref (the unmodified reference compiled here)
 * and against the reference tests' known answers.  Compile with
 * -ffp-contract=off (no FMA), never -ffast-math.
 */
#define _GNU_SOURCE
#include "vlbm_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static _Thread_local char g_err[256];
static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* vo_last_error(void) { return g_err; }

/* std::min / std::max / std::clamp semantics (ties and signed zeros keep the
 * first argument, exactly as <algorithm>). */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

/* ---- random.hpp --------------------------------------------------------- */

/* mix64, random.hpp:10-15 */
uint64_t vo_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* sample_seed, random.hpp:42-44 */
uint64_t vo_sample_seed(uint64_t base, uint64_t m) { return vo_mix64(base ^ vo_mix64(m + 1)); }

/* SplitMix64::next_u64/next_unit/next_sym, random.hpp:22-34: output n is
 * the finalizer of seed + (n+1) * golden gamma. */
static double sm_sym(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  const double unit = (double)(z >> 11) * 0x1.0p-53;
  return 2.0 * unit - 1.0;
}

/* draw_coefficients, perturbation.hpp:42-54: Y1,Z1,Y2,Z2,... */
uint64_t vo_draw_coefficients(uint64_t base, uint64_t m, int K, double* y, double* z) {
  const uint64_t seed = vo_sample_seed(base, m);
  uint64_t st = seed;
  for (int k = 0; k < K; ++k) {
    y[k] = sm_sym(&st);
    z[k] = sm_sym(&st);
  }
  return seed;
}

/* ---- perturbation.hpp --------------------------------------------------- */

/* taper_window, perturbation.hpp:57-61 */
static double taper(double ybar) {
  if (fabs(ybar) >= 1.0) return 0.0;
  const double c = cos(0.5 * M_PI * ybar);
  return c * c;
}

/* density_perturbation, perturbation.hpp:65-77 */
double vo_density_perturbation(double y, int K, const double* yc, const double* zc,
                               const vlbm_perturbation* pp) {
  const double ybar = y / pp->r_jet;
  const double w = taper(ybar);
  double sum = 0.0;
  for (int k = 1; k <= K; ++k) {
    const double weight = pow((double)k, -pp->decay_exponent);
    sum += weight * (yc[k - 1] * cos(k * M_PI * ybar) + zc[k - 1] * sin(k * M_PI * ybar));
  }
  return pp->rho_jet_bar * (1.0 + pp->amplitude * sum * w);
}

/* inlet_state, perturbation.hpp:87-95 (ambient_state :80-82) */
void vo_inlet_state(double y, int K, const double* yc, const double* zc,
                    const vlbm_perturbation* pp, double gamma, double* out) {
  if (fabs(y) <= pp->r_jet) {
    const double rho = vo_density_perturbation(y, K, yc, zc, pp);
    out[0] = rho;
    out[1] = rho * pp->v_jet;
    out[2] = 0.0;
    out[3] = pp->p_amb / (gamma - 1.0) + 0.5 * rho * pp->v_jet * pp->v_jet;
    return;
  }
  out[0] = pp->rho_amb;
  out[1] = 0.0;
  out[2] = 0.0;
  out[3] = pp->p_amb / (gamma - 1.0);
}

static double grid_dx(const vlbm_grid* g) { return g->x_max / g->nx; }
static double y_center(const vlbm_grid* g, int j) { return g->y_min + (j + 0.5) * grid_dx(g); }
static double x_center(const vlbm_grid* g, int i) { return (i + 0.5) * grid_dx(g); }

/* Grid::validate, grid.hpp:28-35 */
static int grid_validate(const vlbm_grid* g) {
  if (g->nx < 4 || g->ny < 4) return set_err(VLBM_E_INVALID, "Grid: nx, ny must be >= 4");
  const double dxx = g->x_max / g->nx;
  const double dxy = (g->y_max - g->y_min) / g->ny;
  if (fabs(dxx - dxy) > 1e-12 * dxx)
    return set_err(VLBM_E_INVALID, "Grid: cells are not square (dx mismatch between x and y)");
  return VLBM_OK;
}

/* initial_field, perturbation.hpp:106-122 */
int vo_initial_field(const vlbm_grid* g, int K, const double* yc, const double* zc,
                     const vlbm_perturbation* pp, double gamma, double strip, double* out) {
  int rc = grid_validate(g);
  if (rc) return rc;
  const size_t n = (size_t)g->nx * g->ny;
  const double amb[4] = {pp->rho_amb, 0.0, 0.0, pp->p_amb / (gamma - 1.0)};
  for (int k = 0; k < 4; ++k)
    for (size_t c = 0; c < n; ++c) out[k * n + c] = amb[k];
  const double height = g->y_max - g->y_min;
  for (int j = 0; j < g->ny; ++j) {
    const double y = y_center(g, j);
    double u_in[4];
    vo_inlet_state(y, K, yc, zc, pp, gamma, u_in);
    const double w = strip * (0.5 + 5.0 * (y - g->y_min) / height);
    for (int i = 0; i < g->nx && x_center(g, i) < w; ++i)
      for (int k = 0; k < 4; ++k) out[k * n + (size_t)j * g->nx + i] = u_in[k];
  }
  return VLBM_OK;
}

/* ---- euler.hpp / lattice.hpp --------------------------------------------- */

typedef struct {
  double v[4];
} cs; /* ConservedState, euler.hpp:16-46 */

static inline cs cs_add(cs a, cs b) {
  for (int k = 0; k < 4; ++k) a.v[k] = a.v[k] + b.v[k];
  return a;
}
static inline cs cs_sub(cs a, cs b) {
  for (int k = 0; k < 4; ++k) a.v[k] = a.v[k] - b.v[k];
  return a;
}
/* operator*(double s, ConservedState a): a *= s, euler.hpp:39-50 */
static inline cs cs_scale(double s, cs a) {
  for (int k = 0; k < 4; ++k) a.v[k] = a.v[k] * s;
  return a;
}

/* pressure, euler.hpp:62-65 (no clamp) */
static inline double pres(cs u, double gamma) {
  const double kinetic = 0.5 * (u.v[1] * u.v[1] + u.v[2] * u.v[2]) / u.v[0];
  return (gamma - 1.0) * (u.v[3] - kinetic);
}
double vo_pressure(const double* u, double gamma) {
  cs s = {{u[0], u[1], u[2], u[3]}};
  return pres(s, gamma);
}

/* flux_x / flux_y, euler.hpp:86-97 */
static inline cs fx(cs u, double gamma) {
  const double v1 = u.v[1] / u.v[0];
  const double p = pres(u, gamma);
  cs f = {{u.v[1], u.v[1] * v1 + p, u.v[2] * v1, (u.v[3] + p) * v1}};
  return f;
}
static inline cs fy(cs u, double gamma) {
  const double v2 = u.v[2] / u.v[0];
  const double p = pres(u, gamma);
  cs f = {{u.v[2], u.v[1] * v2, u.v[2] * v2 + p, (u.v[3] + p) * v2}};
  return f;
}

/* maxwellians, lattice.hpp:43-55 */
static inline void maxw(cs u, double a, double alpha, double gamma, cs m[4]) {
  const cs f = fx(u, gamma);
  const cs g = fy(u, gamma);
  const double w = 0.25 * (1.0 - alpha);
  const double inv2a = 0.5 / a;
  const cs wu = cs_scale(w, u);
  m[0] = cs_add(wu, cs_scale(inv2a, f));
  m[1] = cs_sub(wu, cs_scale(inv2a, f));
  m[2] = cs_add(wu, cs_scale(inv2a, g));
  m[3] = cs_sub(wu, cs_scale(inv2a, g));
}
void vo_maxwellians(const double* u, double a, double alpha, double gamma, double* out16) {
  cs s = {{u[0], u[1], u[2], u[3]}}, m[4];
  maxw(s, a, alpha, gamma, m);
  for (int k = 0; k < 4; ++k)
    for (int c = 0; c < 4; ++c) out16[4 * k + c] = m[k].v[c];
}

/* ---- solver.hpp: Simulation ---------------------------------------------- */

enum { G = 2 }; /* kGhost, solver.hpp:59 */

struct vo_sim {
  vlbm_grid g;
  vlbm_params p;
  int stride, rows;
  double time;
  long steps;
  uint64_t seed;
  cs *u, *un, *pops[4], *popsn[4], *mw[4], *ufo;
  double *pfo, *thc;
  double *tx, *ty; /* BlendingField, solver.hpp:35-51 */
  double* inlet;   /* inlet profile rows, ny x 4 (Boundaries::inlet_profile) */
};

#define CELL(arr, i, j) (arr)[(size_t)((j) + G) * s->stride + ((i) + G)]
#define TX(I, j) s->tx[(size_t)(j) * (s->g.nx + 1) + (I)]
#define TY(i, J) s->ty[(size_t)(J) * s->g.nx + (i)]

static cs inlet_row(const vo_sim* s, int j) {
  cs r = {{s->inlet[4 * j], s->inlet[4 * j + 1], s->inlet[4 * j + 2], s->inlet[4 * j + 3]}};
  return r;
}

/* signal_speed, solver.hpp:203-209 */
static double signal_speed(const vo_sim* s, cs u) {
  const double p = pres(u, s->p.gamma);
  if (!(u.v[0] > 0.0) || !(p > 0.0)) return NAN;
  const double c = sqrt(s->p.gamma * p / u.v[0]);
  if (s->p.conservative_bound) return hypot(u.v[1], u.v[2]) / u.v[0] + c;
  return smax(fabs(u.v[1]), fabs(u.v[2])) / u.v[0] + c;
}

/* kinetic_speed, solver.hpp:137-154 */
static double kinetic_speed(const vo_sim* s) {
  double sm = 0.0;
  for (int j = 0; j < s->g.ny; ++j)
    for (int i = 0; i < s->g.nx; ++i) {
      const double v = signal_speed(s, CELL(s->u, i, j));
      if (!isfinite(v)) return NAN;
      sm = smax(sm, v);
    }
  if (s->p.bc[0] == VLBM_BC_INLET) {
    for (int j = 0; j < s->g.ny; ++j) {
      const double v = signal_speed(s, inlet_row(s, j));
      if (!isfinite(v)) return NAN;
      sm = smax(sm, v);
    }
  }
  return s->p.safety * sm;
}

/* suggest_dt, solver.hpp:157 */
double vo_sim_suggest_dt(vo_sim* s) { return grid_dx(&s->g) / kinetic_speed(s); }

/* set_ghost_from / set_wall_ghost, solver.hpp:211-228 */
static void ghost_copy(vo_sim* s, int gi, int gj, int si, int sj) {
  CELL(s->u, gi, gj) = CELL(s->u, si, sj);
  for (int k = 0; k < 4; ++k) CELL(s->pops[k], gi, gj) = CELL(s->pops[k], si, sj);
}
static void ghost_wall(vo_sim* s, int gi, int gj, int si, int sj) {
  static const int swap_k[4] = {0, 1, 3, 2};
  cs m = CELL(s->u, si, sj);
  m.v[2] = -m.v[2];
  CELL(s->u, gi, gj) = m;
  for (int k = 0; k < 4; ++k) {
    cs f = CELL(s->pops[swap_k[k]], si, sj);
    f.v[2] = -f.v[2];
    CELL(s->pops[k], gi, gj) = f;
  }
}

/* fill_ghosts, solver.hpp:230-286: x sides on interior rows, then y sides
 * over the full padded width (corners inherit the x-side values). */
static void fill_ghosts(vo_sim* s, double a) {
  const int nx = s->g.nx, ny = s->g.ny;
  for (int j = 0; j < ny; ++j) {
    switch (s->p.bc[0]) {
      case VLBM_BC_INLET: {
        const cs u_in = inlet_row(s, j);
        cs m[4];
        maxw(u_in, a, s->p.alpha, s->p.gamma, m);
        for (int gi = -1; gi >= -2; --gi) {
          CELL(s->u, gi, j) = u_in;
          for (int k = 0; k < 4; ++k) CELL(s->pops[k], gi, j) = m[k];
        }
        break;
      }
      case VLBM_BC_OUTFLOW:
        ghost_copy(s, -1, j, 0, j);
        ghost_copy(s, -2, j, 0, j);
        break;
      default: /* periodic */
        ghost_copy(s, -1, j, nx - 1, j);
        ghost_copy(s, -2, j, nx - 2, j);
    }
    if (s->p.bc[1] == VLBM_BC_OUTFLOW) {
      ghost_copy(s, nx, j, nx - 1, j);
      ghost_copy(s, nx + 1, j, nx - 1, j);
    } else {
      ghost_copy(s, nx, j, 0, j);
      ghost_copy(s, nx + 1, j, 1, j);
    }
  }
  for (int i = -G; i < nx + G; ++i) {
    if (s->p.bc[2] == VLBM_BC_WALL) {
      ghost_wall(s, i, -1, i, 0);
      ghost_wall(s, i, -2, i, 1);
    } else {
      ghost_copy(s, i, -1, i, ny - 1);
      ghost_copy(s, i, -2, i, ny - 2);
    }
    if (s->p.bc[3] == VLBM_BC_WALL) {
      ghost_wall(s, i, ny, i, ny - 1);
      ghost_wall(s, i, ny + 1, i, ny - 2);
    } else {
      ghost_copy(s, i, ny, i, 0);
      ghost_copy(s, i, ny + 1, i, 1);
    }
  }
}

/* compute_maxwellians, solver.hpp:288-297 */
static void compute_maxwellians(vo_sim* s, double a) {
  for (int j = -G; j < s->g.ny + G; ++j)
    for (int i = -G; i < s->g.nx + G; ++i) {
      cs m[4];
      maxw(CELL(s->u, i, j), a, s->p.alpha, s->p.gamma, m);
      for (int k = 0; k < 4; ++k) CELL(s->mw[k], i, j) = m[k];
    }
}

/* compute_candidates, solver.hpp:301-316 */
static void compute_candidates(vo_sim* s) {
  for (int j = -1; j <= s->g.ny; ++j)
    for (int i = -1; i <= s->g.nx; ++i) {
      const cs x = cs_add(CELL(s->mw[0], i - 1, j), CELL(s->mw[1], i + 1, j));
      const cs y = cs_add(CELL(s->mw[2], i, j - 1), CELL(s->mw[3], i, j + 1));
      const cs fo = cs_add(cs_add(x, y), cs_scale(s->p.alpha, CELL(s->u, i, j)));
      CELL(s->ufo, i, j) = fo;
      CELL(s->pfo, i, j) = pres(fo, s->p.gamma);
    }
}

/* face_corrections, solver.hpp:321-329 */
static void face_corrections(const vo_sim* s, int i, int j, cs c[4]) {
#define CORR(k, ii, jj) cs_sub(CELL(s->mw[k], ii, jj), CELL(s->pops[k], ii, jj))
  c[0] = cs_sub(CORR(0, i - 1, j), CORR(1, i, j));
  c[1] = cs_sub(CORR(1, i + 1, j), CORR(0, i, j));
  c[2] = cs_sub(CORR(2, i, j - 1), CORR(3, i, j));
  c[3] = cs_sub(CORR(3, i, j + 1), CORR(2, i, j));
#undef CORR
}

/* allowance lambda, solver.hpp:389-397 */
static double allowance(double um2, double um1, double u0, double up1, double up2) {
  const double d2m = (um2 + u0) - 2.0 * um1;
  const double d2c = (um1 + up1) - 2.0 * u0;
  const double d2p = (u0 + up2) - 2.0 * up1;
  if (d2m * d2c < 0.0 || d2p * d2c < 0.0) return 0.0;
  return 0.5 * fabs(d2c);
}

typedef struct {
  double rho_lo, rho_hi, p_lo, p_hi, rho_floor, p_floor;
} bounds;

/* rlmp_bounds, solver.hpp:364-435 */
static bounds rlmp_bounds(const vo_sim* s, int i, int j) {
  const double gm = s->p.gamma;
  double rho_min = CELL(s->ufo, i, j).v[0], rho_max = rho_min;
  double p_min = CELL(s->pfo, i, j), p_max = p_min;
  double rho_prev[5], p_prev[5];
  static const int di[5] = {0, -1, 1, 0, 0};
  static const int dj[5] = {0, 0, 0, -1, 1};
  for (int n = 0; n < 5; ++n) {
    const int ii = i + di[n], jj = j + dj[n];
    const cs prev = CELL(s->u, ii, jj);
    rho_prev[n] = prev.v[0];
    p_prev[n] = pres(prev, gm);
    if (n > 0) {
      const double r = CELL(s->ufo, ii, jj).v[0];
      const double p = CELL(s->pfo, ii, jj);
      rho_min = smin(rho_min, r);
      rho_max = smax(rho_max, r);
      p_min = smin(p_min, p);
      p_max = smax(p_max, p);
    }
  }
  const double rho_head =
      allowance(CELL(s->u, i - 2, j).v[0], rho_prev[1], rho_prev[0], rho_prev[2],
                CELL(s->u, i + 2, j).v[0]) +
      allowance(CELL(s->u, i, j - 2).v[0], rho_prev[3], rho_prev[0], rho_prev[4],
                CELL(s->u, i, j + 2).v[0]);
  const double p_head =
      allowance(pres(CELL(s->u, i - 2, j), gm), p_prev[1], p_prev[0], p_prev[2],
                pres(CELL(s->u, i + 2, j), gm)) +
      allowance(pres(CELL(s->u, i, j - 2), gm), p_prev[3], p_prev[0], p_prev[4],
                pres(CELL(s->u, i, j + 2), gm));
  /* std::min_element / std::max_element: first extremum wins */
  double rmn = rho_prev[0], rmx = rho_prev[0], pmn = p_prev[0], pmx = p_prev[0];
  for (int n = 1; n < 5; ++n) {
    if (rho_prev[n] < rmn) rmn = rho_prev[n];
    if (rmx < rho_prev[n]) rmx = rho_prev[n];
    if (p_prev[n] < pmn) pmn = p_prev[n];
    if (pmx < p_prev[n]) pmx = p_prev[n];
  }
  const double rho_min_prev = rmn - rho_head;
  const double rho_max_prev = rmx + rho_head;
  const double p_min_prev = pmn - p_head;
  const double p_max_prev = pmx + p_head;
  const double kappa = s->p.rlmp_relaxation;
  bounds b;
  b.rho_floor = s->p.positivity_floor * s->p.rho_ref;
  b.p_floor = s->p.positivity_floor * s->p.p_ref;
  const double rho_eps = 1e-12 * (fabs(rho_max) + fabs(rho_min));
  const double p_eps = 1e-12 * (fabs(p_max) + fabs(p_min));
  const double frac = 1.0 - smin(kappa, 0.9);
  /* std::max({a, b, c}) == max(max(a, b), c) with first-wins ties */
  b.rho_lo = smax(smax(smin(rho_min - kappa * (rho_max - rho_min), rho_min_prev) - rho_eps,
                       frac * smin(rho_min, rho_min_prev)),
                  b.rho_floor);
  b.rho_hi = smax(rho_max + kappa * (rho_max - rho_min), rho_max_prev) + rho_eps;
  b.p_lo = smax(smax(smin(p_min - kappa * (p_max - p_min), p_min_prev) - p_eps,
                     frac * smin(p_min, p_min_prev)),
                b.p_floor);
  b.p_hi = smax(p_max + kappa * (p_max - p_min), p_max_prev) + p_eps;
  return b;
}

/* feasible lambda, solver.hpp:444-459 */
static int feasible(double th, cs fo, cs delta, const cs c[4], const bounds* b, double gm) {
  const cs u = cs_add(fo, cs_scale(th, delta));
  if (!(u.v[0] >= b->rho_lo) || !(u.v[0] <= b->rho_hi)) return 0;
  const double p = pres(u, gm);
  if (!(p >= b->p_lo) || !(p <= b->p_hi)) return 0;
  for (int mask = 1; mask < 16; ++mask) {
    cs cx = {{0.0, 0.0, 0.0, 0.0}}, cy = {{0.0, 0.0, 0.0, 0.0}};
    if (mask & 1) cx = cs_add(cx, cs_scale(th, c[0]));
    if (mask & 2) cx = cs_add(cx, cs_scale(th, c[1]));
    if (mask & 4) cy = cs_add(cy, cs_scale(th, c[2]));
    if (mask & 8) cy = cs_add(cy, cs_scale(th, c[3]));
    const cs v = cs_add(cs_add(fo, cx), cy);
    if (!(v.v[0] >= b->rho_floor) || !(pres(v, gm) >= b->p_floor)) return 0;
  }
  return 1;
}

/* rlmp_theta, solver.hpp:437-487 */
static double rlmp_theta(const vo_sim* s, int i, int j) {
  const double gm = s->p.gamma;
  const cs fo = CELL(s->ufo, i, j);
  cs c[4];
  face_corrections(s, i, j, c);
  const cs delta = cs_add(cs_add(c[0], c[1]), cs_add(c[2], c[3]));
  const bounds b = rlmp_bounds(s, i, j);
  if (feasible(1.0, fo, delta, c, &b, gm)) return 1.0;
  if (!feasible(0.0, fo, delta, c, &b, gm)) return 0.0;
  double theta = 1.0;
  if (delta.v[0] > 0.0) theta = smin(theta, (b.rho_hi - fo.v[0]) / delta.v[0]);
  if (delta.v[0] < 0.0) theta = smin(theta, (fo.v[0] - b.rho_lo) / (-delta.v[0]));
  const double dneg = (smin(c[0].v[0], 0.0) + smin(c[1].v[0], 0.0)) +
                      (smin(c[2].v[0], 0.0) + smin(c[3].v[0], 0.0));
  if (dneg < 0.0) theta = smin(theta, (fo.v[0] - b.rho_floor) / (-dneg));
  theta = theta < 0.0 ? 0.0 : (1.0 < theta ? 1.0 : theta); /* std::clamp */
  if (feasible(theta, fo, delta, c, &b, gm)) return theta;
  double lo = 0.0, hi = theta;
  for (int it = 0; it < 30; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (feasible(mid, fo, delta, c, &b, gm))
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

/* compute_theta, solver.hpp:489-505 */
static void compute_theta(vo_sim* s) {
  for (int j = 0; j < s->g.ny; ++j)
    for (int i = 0; i < s->g.nx; ++i) {
      double t;
      switch (s->p.limiter) {
        case VLBM_LIMITER_FIRST_ORDER: t = 0.0; break;
        case VLBM_LIMITER_SECOND_ORDER: t = 1.0; break;
        default: t = rlmp_theta(s, i, j);
      }
      CELL(s->thc, i, j) = t;
    }
}

/* interface_theta, solver.hpp:510-534 */
static void interface_theta(vo_sim* s) {
  const int nx = s->g.nx, ny = s->g.ny;
  const int per_x = s->p.bc[0] == VLBM_BC_PERIODIC;
  const int per_y = s->p.bc[2] == VLBM_BC_PERIODIC;
  for (int j = 0; j < ny; ++j) {
    for (int I = 1; I < nx; ++I) TX(I, j) = smin(CELL(s->thc, I - 1, j), CELL(s->thc, I, j));
    const double edge = per_x ? smin(CELL(s->thc, 0, j), CELL(s->thc, nx - 1, j)) : 0.0;
    TX(0, j) = per_x ? edge : CELL(s->thc, 0, j);
    TX(nx, j) = per_x ? edge : CELL(s->thc, nx - 1, j);
  }
  for (int i = 0; i < nx; ++i) {
    for (int J = 1; J < ny; ++J) TY(i, J) = smin(CELL(s->thc, i, J - 1), CELL(s->thc, i, J));
    const double edge = per_y ? smin(CELL(s->thc, i, 0), CELL(s->thc, i, ny - 1)) : 0.0;
    TY(i, 0) = per_y ? edge : CELL(s->thc, i, 0);
    TY(i, ny) = per_y ? edge : CELL(s->thc, i, ny - 1);
  }
}

/* advance, solver.hpp:536-575 */
static void advance(vo_sim* s) {
  const int nx = s->g.nx, ny = s->g.ny;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const double tw = TX(i, j), te = TX(i + 1, j), ts = TY(i, j), tn = TY(i, j + 1);
#define PULL(k, ii, jj, th)                                                              \
  cs_add(CELL(s->mw[k], ii, jj),                                                         \
         cs_scale(th, cs_sub(CELL(s->mw[k], ii, jj), CELL(s->pops[k], ii, jj))))
      const cs n1 = PULL(0, i - 1, j, tw);
      const cs n2 = PULL(1, i + 1, j, te);
      const cs n3 = PULL(2, i, j - 1, ts);
      const cs n4 = PULL(3, i, j + 1, tn);
#undef PULL
      CELL(s->popsn[0], i, j) = n1;
      CELL(s->popsn[1], i, j) = n2;
      CELL(s->popsn[2], i, j) = n3;
      CELL(s->popsn[3], i, j) = n4;
#define NEQ(k) cs_sub(CELL(s->mw[k], i, j), CELL(s->pops[k], i, j))
      cs un = cs_add(cs_add(cs_add(n1, n2), cs_add(n3, n4)), cs_scale(s->p.alpha, CELL(s->u, i, j)));
      const cs out = cs_add(cs_add(cs_scale(tw, NEQ(1)), cs_scale(te, NEQ(0))),
                            cs_add(cs_scale(ts, NEQ(3)), cs_scale(tn, NEQ(2))));
#undef NEQ
      un = cs_sub(un, out);
      CELL(s->un, i, j) = un;
    }
  cs* t = s->u;
  s->u = s->un;
  s->un = t;
  for (int k = 0; k < 4; ++k) {
    t = s->pops[k];
    s->pops[k] = s->popsn[k];
    s->popsn[k] = t;
  }
}

/* Simulation::Simulation, solver.hpp:61-100 */
int vo_sim_create(const vlbm_grid* g, const vlbm_params* p, const double* init,
                  const double* inlet_rows, uint64_t seed, vo_sim** out) {
  int rc = grid_validate(g);
  if (rc) return rc;
  if (p->alpha < 0.0 || p->alpha > 1.0) return set_err(VLBM_E_INVALID, "alpha must be in [0,1]");
  if (p->safety < 1.0) return set_err(VLBM_E_INVALID, "safety must be >= 1");
  if (p->rlmp_relaxation < 0.0) return set_err(VLBM_E_INVALID, "rlmp_relaxation must be >= 0");
  if (!(p->positivity_floor > 0.0))
    return set_err(VLBM_E_INVALID, "positivity_floor must be > 0");
  if ((p->bc[0] == VLBM_BC_PERIODIC) != (p->bc[1] == VLBM_BC_PERIODIC) ||
      (p->bc[2] == VLBM_BC_PERIODIC) != (p->bc[3] == VLBM_BC_PERIODIC))
    return set_err(VLBM_E_INVALID, "Simulation: periodic sides must be paired");
  if (p->bc[0] == VLBM_BC_INLET && !inlet_rows)
    return set_err(VLBM_E_INVALID, "Simulation: inlet boundary requires a profile");
  if (p->bc[0] == VLBM_BC_WALL)
    return set_err(VLBM_E_INVALID, "Simulation: walls are supported on y sides only");
  if (p->bc[1] == VLBM_BC_INLET || p->bc[1] == VLBM_BC_WALL)
    return set_err(VLBM_E_INVALID, "Simulation: unsupported x_max boundary");
  vo_sim* s = calloc(1, sizeof *s);
  s->g = *g;
  s->p = *p;
  s->seed = seed;
  s->stride = g->nx + 2 * G;
  s->rows = g->ny + 2 * G;
  const size_t n = (size_t)s->stride * s->rows;
  s->u = calloc(n, sizeof(cs));
  s->un = calloc(n, sizeof(cs));
  for (int k = 0; k < 4; ++k) {
    s->pops[k] = calloc(n, sizeof(cs));
    s->popsn[k] = calloc(n, sizeof(cs));
    s->mw[k] = calloc(n, sizeof(cs));
  }
  s->ufo = calloc(n, sizeof(cs));
  s->pfo = calloc(n, sizeof(double));
  s->thc = malloc(n * sizeof(double));
  for (size_t c = 0; c < n; ++c) s->thc[c] = 1.0;
  s->tx = calloc((size_t)(g->nx + 1) * g->ny, sizeof(double));
  s->ty = calloc((size_t)g->nx * (g->ny + 1), sizeof(double));
  if (inlet_rows) {
    s->inlet = malloc(sizeof(double) * 4 * g->ny);
    memcpy(s->inlet, inlet_rows, sizeof(double) * 4 * g->ny);
  }
  const size_t nc = (size_t)g->nx * g->ny;
  for (int j = 0; j < g->ny; ++j)
    for (int i = 0; i < g->nx; ++i)
      for (int k = 0; k < 4; ++k) CELL(s->u, i, j).v[k] = init[k * nc + (size_t)j * g->nx + i];
  const double a0 = grid_dx(g) / vo_sim_suggest_dt(s);
  for (int j = 0; j < g->ny; ++j)
    for (int i = 0; i < g->nx; ++i) {
      cs m[4];
      maxw(CELL(s->u, i, j), a0, p->alpha, p->gamma, m);
      for (int k = 0; k < 4; ++k) CELL(s->pops[k], i, j) = m[k];
    }
  *out = s;
  return VLBM_OK;
}

void vo_sim_destroy(vo_sim* s) {
  if (!s) return;
  free(s->u);
  free(s->un);
  for (int k = 0; k < 4; ++k) {
    free(s->pops[k]);
    free(s->popsn[k]);
    free(s->mw[k]);
  }
  free(s->ufo);
  free(s->pfo);
  free(s->thc);
  free(s->tx);
  free(s->ty);
  free(s->inlet);
  free(s);
}

/* Simulation::step, solver.hpp:160-170 */
int vo_sim_step(vo_sim* s, double dt) {
  const double a = grid_dx(&s->g) / dt;
  fill_ghosts(s, a);
  compute_maxwellians(s, a);
  compute_candidates(s);
  compute_theta(s);
  interface_theta(s);
  advance(s);
  s->time += dt;
  ++s->steps;
  return VLBM_OK;
}

/* step_with_blending, solver.hpp:173-181 */
int vo_sim_step_with_blending(vo_sim* s, double dt, const double* tx, const double* ty) {
  const double a = grid_dx(&s->g) / dt;
  fill_ghosts(s, a);
  compute_maxwellians(s, a);
  memcpy(s->tx, tx, sizeof(double) * (size_t)(s->g.nx + 1) * s->g.ny);
  memcpy(s->ty, ty, sizeof(double) * (size_t)s->g.nx * (s->g.ny + 1));
  advance(s);
  s->time += dt;
  ++s->steps;
  return VLBM_OK;
}

/* compute_blending, solver.hpp:184-191 */
int vo_sim_compute_blending(vo_sim* s, double a, double* tx, double* ty) {
  fill_ghosts(s, a);
  compute_maxwellians(s, a);
  compute_candidates(s);
  compute_theta(s);
  interface_theta(s);
  memcpy(tx, s->tx, sizeof(double) * (size_t)(s->g.nx + 1) * s->g.ny);
  memcpy(ty, s->ty, sizeof(double) * (size_t)s->g.nx * (s->g.ny + 1));
  return VLBM_OK;
}

/* The limiter's per-cell inputs at the step with speed a (the pipeline of
 * compute_blending, solver.hpp:184-191): per interior cell u_FO (4), the face
 * corrections c_w, c_e, c_s, c_n (16), rho_lo, rho_hi, p_lo, p_hi, rho_floor,
 * p_floor (rlmp_bounds) and the limiter's theta -- 27 doubles, row-major.
 * Test hook for the device limiter restatement (tests/cpp/limiter_check). */
int vo_sim_limiter_cells(vo_sim* s, double a, double* out) {
  fill_ghosts(s, a);
  compute_maxwellians(s, a);
  compute_candidates(s);
  for (int j = 0; j < s->g.ny; ++j)
    for (int i = 0; i < s->g.nx; ++i) {
      double* r = out + 27 * ((size_t)j * s->g.nx + i);
      const cs fo = CELL(s->ufo, i, j);
      cs c[4];
      face_corrections(s, i, j, c);
      const bounds b = rlmp_bounds(s, i, j);
      for (int k = 0; k < 4; ++k) r[k] = fo.v[k];
      for (int f = 0; f < 4; ++f)
        for (int k = 0; k < 4; ++k) r[4 + 4 * f + k] = c[f].v[k];
      r[20] = b.rho_lo;
      r[21] = b.rho_hi;
      r[22] = b.p_lo;
      r[23] = b.p_hi;
      r[24] = b.rho_floor;
      r[25] = b.p_floor;
      r[26] = rlmp_theta(s, i, j);
    }
  return VLBM_OK;
}

void vo_sim_theta_cell(vo_sim* s, double* theta) {
  for (int j = 0; j < s->g.ny; ++j)
    for (int i = 0; i < s->g.nx; ++i) theta[(size_t)j * s->g.nx + i] = CELL(s->thc, i, j);
}

double vo_sim_time(vo_sim* s) { return s->time; }
long vo_sim_steps(vo_sim* s) { return s->steps; }

/* state_finite, solver.hpp:122-133 */
int vo_sim_state_finite(vo_sim* s) {
  for (int j = 0; j < s->g.ny; ++j)
    for (int i = 0; i < s->g.nx; ++i)
      for (int k = 0; k < 4; ++k)
        if (!isfinite(CELL(s->u, i, j).v[k])) return 0;
  return 1;
}

void vo_sim_get(vo_sim* s, double* u, double* pops) {
  const size_t n = (size_t)s->g.nx * s->g.ny;
  for (int j = 0; j < s->g.ny; ++j)
    for (int i = 0; i < s->g.nx; ++i) {
      const size_t c = (size_t)j * s->g.nx + i;
      for (int k = 0; k < 4; ++k) {
        if (u) u[k * n + c] = CELL(s->u, i, j).v[k];
        if (pops)
          for (int q = 0; q < 4; ++q) pops[(4 * q + k) * n + c] = CELL(s->pops[q], i, j).v[k];
      }
    }
}

/* run_sample, solver.hpp:625-669 */
int vo_run_sample(const vlbm_grid* g, const vlbm_params* p, const vlbm_perturbation* pp, int K,
                  const double* yc, const double* zc, uint64_t seed, double strip,
                  const double* times, int n_times, double* out_fields, double* out_time,
                  int* out_div, long* out_steps, int* out_admissible) {
  if (pp->amplitude < 0) return set_err(VLBM_E_INVALID, "amplitude must be >= 0");
  if (pp->modes < 1) return set_err(VLBM_E_INVALID, "modes must be >= 1");
  if (pp->decay_exponent <= 0) return set_err(VLBM_E_INVALID, "decay_exponent must be > 0");
  for (int i = 1; i < n_times; ++i)
    if (times[i] <= times[i - 1])
      return set_err(VLBM_E_INVALID, "run_sample: snapshot times must be strictly increasing");
  const size_t n = (size_t)g->nx * g->ny;
  double* rows = malloc(sizeof(double) * 4 * g->ny);
  double* init = malloc(sizeof(double) * 4 * n);
  for (int j = 0; j < g->ny; ++j) vo_inlet_state(y_center(g, j), K, yc, zc, pp, p->gamma, rows + 4 * j);
  int rc = vo_initial_field(g, K, yc, zc, pp, p->gamma, strip, init);
  vlbm_params q = *p;
  q.bc[0] = VLBM_BC_INLET;
  q.bc[1] = VLBM_BC_OUTFLOW;
  q.bc[2] = VLBM_BC_WALL;
  q.bc[3] = VLBM_BC_WALL;
  q.rho_ref = pp->rho_amb; /* set_reference, solver.hpp:640 */
  q.p_ref = pp->p_amb;
  vo_sim* s = NULL;
  if (!rc) rc = vo_sim_create(g, &q, init, rows, seed, &s);
  free(rows);
  free(init);
  if (rc) return rc;
  const double t_eps = 1e-12;
  int diverged = 0;
  for (int t = 0; t < n_times; ++t) {
    const double target = times[t];
    if (!diverged) {
      while (s->time < target - t_eps) {
        const double dt_stable = vo_sim_suggest_dt(s);
        if (!isfinite(dt_stable) || dt_stable <= 0.0) {
          diverged = 1;
          break;
        }
        vo_sim_step(s, smin(dt_stable, target - s->time));
        if (!vo_sim_state_finite(s)) {
          diverged = 1;
          break;
        }
      }
    }
    if (out_fields) vo_sim_get(s, out_fields + 4 * n * t, NULL);
    if (out_time) out_time[t] = diverged ? s->time : target;
    if (out_div) out_div[t] = diverged;
  }
  if (out_steps) *out_steps = s->steps;
  if (out_admissible) *out_admissible = !diverged;
  vo_sim_destroy(s);
  return VLBM_OK;
}

/* ---- metrics.hpp --------------------------------------------------------- */

/* restrict_field, metrics.hpp:29-49 */
int vo_restrict_field(int nx, int ny, const double* fine, double* coarse) {
  if (nx % 2 != 0 || ny % 2 != 0)
    return set_err(VLBM_E_INVALID, "restrict_field: fine dimensions must be even");
  const int cx = nx / 2, cy = ny / 2;
  const size_t nf = (size_t)nx * ny, nc = (size_t)cx * cy;
  for (int k = 0; k < 4; ++k)
    for (int j = 0; j < cy; ++j)
      for (int i = 0; i < cx; ++i) {
        const double* f = fine + k * nf;
        const double sum = ((f[(size_t)(2 * j) * nx + 2 * i] + f[(size_t)(2 * j) * nx + 2 * i + 1]) +
                            f[(size_t)(2 * j + 1) * nx + 2 * i]) +
                           f[(size_t)(2 * j + 1) * nx + 2 * i + 1];
        coarse[k * nc + (size_t)j * cx + i] = sum * 0.25;
      }
  return VLBM_OK;
}

/* strong_error, metrics.hpp:55-90 */
int vo_strong_error(int M, int64_t n, const double* a, const double* b, double* result,
                    double* per_comp) {
  if (M < 1) return set_err(VLBM_E_INVALID, "strong_error: sample counts differ or are empty");
  double acc = 0.0, comp_acc[4] = {0, 0, 0, 0};
  for (int m = 0; m < M; ++m) {
    const double* A = a + (size_t)4 * n * m;
    const double* B = b + (size_t)4 * n * m;
    double num = 0.0, den = 0.0, cnum[4] = {0, 0, 0, 0}, cden[4] = {0, 0, 0, 0};
    for (int64_t c = 0; c < n; ++c)
      for (int k = 0; k < 4; ++k) {
        const double d = fabs(A[k * n + c] - B[k * n + c]);
        const double r = fabs(B[k * n + c]);
        num += d;
        den += r;
        cnum[k] += d;
        cden[k] += r;
      }
    if (den == 0.0) return set_err(VLBM_E_DOMAIN, "strong_error: zero reference norm");
    acc += num / den;
    for (int k = 0; k < 4; ++k) comp_acc[k] += cden[k] > 0.0 ? cnum[k] / cden[k] : 0.0;
  }
  if (per_comp)
    for (int k = 0; k < 4; ++k) per_comp[k] = comp_acc[k] / M;
  *result = acc / M;
  return VLBM_OK;
}

static int cmp_double(const void* x, const void* y) {
  const double a = *(const double*)x, b = *(const double*)y;
  return (a < b) ? -1 : (b < a) ? 1 : 0;
}

/* wasserstein1, metrics.hpp:97-125 */
int vo_wasserstein1(int M, int64_t n, const double* a, const double* b, int var, double* result) {
  if (M < 1) return set_err(VLBM_E_INVALID, "wasserstein1: sample counts differ or are empty");
  double* ca = malloc(sizeof(double) * M);
  double* cb = malloc(sizeof(double) * M);
  double acc = 0.0;
  for (int64_t c = 0; c < n; ++c) {
    for (int m = 0; m < M; ++m) {
      ca[m] = a[(size_t)4 * n * m + (size_t)var * n + c];
      cb[m] = b[(size_t)4 * n * m + (size_t)var * n + c];
    }
    qsort(ca, M, sizeof(double), cmp_double);
    qsort(cb, M, sizeof(double), cmp_double);
    double cell = 0.0;
    for (int m = 0; m < M; ++m) cell += fabs(ca[m] - cb[m]);
    acc += cell / (double)M;
  }
  free(ca);
  free(cb);
  *result = acc / (double)n;
  return VLBM_OK;
}

/* ensemble_moments, metrics.hpp:148-177 */
int vo_ensemble_moments(int M, int64_t n, const double* x, double* mean, double* stddev) {
  if (M < 1) return set_err(VLBM_E_INVALID, "ensemble_moments: no samples");
  if (M < 2) return set_err(VLBM_E_INVALID, "ensemble_moments: std requires at least 2 samples");
  const size_t N = (size_t)4 * n;
  for (size_t c = 0; c < N; ++c) mean[c] = 0.0;
  for (int m = 0; m < M; ++m)
    for (size_t c = 0; c < N; ++c) mean[c] += x[N * m + c];
  const double inv_m = 1.0 / M;
  for (size_t c = 0; c < N; ++c) mean[c] *= inv_m;
  for (size_t c = 0; c < N; ++c) stddev[c] = 0.0;
  for (int m = 0; m < M; ++m)
    for (size_t c = 0; c < N; ++c) {
      const double d = x[N * m + c] - mean[c];
      stddev[c] += d * d;
    }
  const double inv_m1 = 1.0 / (M - 1.0);
  for (size_t c = 0; c < N; ++c) stddev[c] = sqrt(stddev[c] * inv_m1);
  return VLBM_OK;
}
