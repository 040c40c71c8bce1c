// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" shim that compiles the UNMODIFIED reference headers from
// /root/reference/proj/include (header-only C++20, STL only) into
// oracle/_ref/libvlbm_ref.so.  Nothing here re-implements the reference: every
// numeric result comes from the reference's own Simulation / run_sample /
// metrics functions.  Used by tests/ (parity pins, golden generation) and by
// bench.py --impl reference (the reference CPU path on all host cores).
//
// Field layout crossing this shim: the .vlbm plane order of
// include/vlbm_b200.h (4 planes of ny x nx, x fastest).

#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "vlbm/metrics.hpp"
#include "vlbm/solver.hpp"
#include "vlbm_b200.h"

using namespace vlbm;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define SHIM_TRY try {
#define SHIM_CATCH                                          \
  }                                                         \
  catch (const std::invalid_argument& e) {                  \
    return fail(e, VLBM_E_INVALID);                         \
  }                                                         \
  catch (const std::domain_error& e) {                      \
    return fail(e, VLBM_E_DOMAIN);                          \
  }                                                         \
  catch (const std::exception& e) {                         \
    return fail(e, VLBM_E_RUNTIME);                         \
  }                                                         \
  return VLBM_OK;

Grid to_grid(const vlbm_grid* g) {
  Grid r;
  r.nx = g->nx;
  r.ny = g->ny;
  r.x_max = g->x_max;
  r.y_min = g->y_min;
  r.y_max = g->y_max;
  return r;
}

LatticeParams to_lattice(const vlbm_params* p) {
  LatticeParams l;
  l.alpha = p->alpha;
  l.safety = p->safety;
  l.limiter = static_cast<Limiter>(p->limiter);
  l.rlmp_relaxation = p->rlmp_relaxation;
  l.positivity_floor = p->positivity_floor;
  l.conservative_bound = p->conservative_bound != 0;
  return l;
}

PerturbationParams to_pert(const vlbm_perturbation* pp) {
  PerturbationParams r;
  r.amplitude = pp->amplitude;
  r.modes = pp->modes;
  r.decay_exponent = pp->decay_exponent;
  r.r_jet = pp->r_jet;
  r.rho_jet_bar = pp->rho_jet_bar;
  r.rho_amb = pp->rho_amb;
  r.p_amb = pp->p_amb;
  r.v_jet = pp->v_jet;
  return r;
}

ModeCoefficients to_coeffs(int K, const double* y, const double* z, uint64_t seed) {
  ModeCoefficients c;
  c.y_coeffs.assign(y, y + K);
  c.z_coeffs.assign(z, z + K);
  c.seed = seed;
  return c;
}

FieldSnapshot field_from_planes(const Grid& g, const double* f) {
  FieldSnapshot s;
  s.grid = g;
  const std::size_t n = g.cells();
  s.data.resize(n);
  for (int k = 0; k < 4; ++k)
    for (std::size_t c = 0; c < n; ++c) s.data[c][k] = f[k * n + c];
  return s;
}

void planes_from_field(const FieldSnapshot& s, double* f) {
  const std::size_t n = s.data.size();
  for (int k = 0; k < 4; ++k)
    for (std::size_t c = 0; c < n; ++c) f[k * n + c] = s.data[c][k];
}

struct RefSim {
  Grid grid;
  std::vector<double> inlet;  // ny x 4 (generic construction only)
  std::unique_ptr<Simulation> sim;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_draw_coefficients(uint64_t base, uint64_t m, int K, double* y, double* z) {
  const ModeCoefficients c = draw_coefficients(base, m, K);
  std::memcpy(y, c.y_coeffs.data(), sizeof(double) * K);
  std::memcpy(z, c.z_coeffs.data(), sizeof(double) * K);
  return c.seed;
}

uint64_t ref_mix64(uint64_t z) { return mix64(z); }
uint64_t ref_sample_seed(uint64_t b, uint64_t m) { return sample_seed(b, m); }

double ref_density_perturbation(double y, int K, const double* yc, const double* zc,
                                const vlbm_perturbation* pp) {
  return density_perturbation(y, to_coeffs(K, yc, zc, 0), to_pert(pp));
}

void ref_inlet_state(double y, int K, const double* yc, const double* zc,
                     const vlbm_perturbation* pp, double gamma, double* out) {
  GasParams g{gamma};
  const ConservedState u = inlet_state(y, to_coeffs(K, yc, zc, 0), to_pert(pp), g);
  for (int k = 0; k < 4; ++k) out[k] = u[k];
}

int ref_initial_field(const vlbm_grid* gg, int K, const double* yc, const double* zc,
                      const vlbm_perturbation* pp, double gamma, double strip, double* out) {
  SHIM_TRY
  GasParams g{gamma};
  const FieldSnapshot s = initial_field(to_grid(gg), to_coeffs(K, yc, zc, 0), to_pert(pp), g, strip);
  planes_from_field(s, out);
  SHIM_CATCH
}

double ref_pressure(const double* u, double gamma) {
  ConservedState s{u[0], u[1], u[2], u[3]};
  return pressure(s, GasParams{gamma});
}

void ref_maxwellians(const double* u, double a, double alpha, double gamma, double* out16) {
  ConservedState s{u[0], u[1], u[2], u[3]};
  const Maxwellians m = maxwellians(s, a, alpha, GasParams{gamma});
  for (int k = 0; k < 4; ++k)
    for (int c = 0; c < 4; ++c) out16[4 * k + c] = m.m[k][c];
}

// ---- Simulation -----------------------------------------------------------

// Jet sample built exactly as run_sample builds it (solver.hpp:633-640).
int ref_sim_create_jet(const vlbm_grid* gg, const vlbm_params* p, const vlbm_perturbation* pp,
                       int K, const double* yc, const double* zc, uint64_t seed, double strip,
                       void** out) {
  SHIM_TRY
  auto* r = new RefSim;
  r->grid = to_grid(gg);
  const PerturbationParams pert = to_pert(pp);
  const GasParams gas{p->gamma};
  const ModeCoefficients coeffs = to_coeffs(K, yc, zc, seed);
  Boundaries bcs;
  bcs.inlet_profile = [pert, coeffs, gas](double y) { return inlet_state(y, coeffs, pert, gas); };
  FieldSnapshot init = initial_field(r->grid, coeffs, pert, gas, strip);
  r->sim = std::make_unique<Simulation>(r->grid, to_lattice(p), gas, std::move(bcs), init);
  r->sim->set_reference(pert.rho_amb, pert.p_amb);
  *out = r;
  SHIM_CATCH
}

// Generic construction on a caller field with explicit boundary types.
// inlet_rows (ny x 4) backs the inlet profile when bc[0] is Inlet.
int ref_sim_create(const vlbm_grid* gg, const vlbm_params* p, const double* init,
                   const double* inlet_rows, uint64_t seed, void** out) {
  SHIM_TRY
  auto* r = new RefSim;
  r->grid = to_grid(gg);
  Boundaries bcs;
  bcs.x_min = static_cast<BcType>(p->bc[0]);
  bcs.x_max = static_cast<BcType>(p->bc[1]);
  bcs.y_min = static_cast<BcType>(p->bc[2]);
  bcs.y_max = static_cast<BcType>(p->bc[3]);
  if (inlet_rows) {
    r->inlet.assign(inlet_rows, inlet_rows + 4 * static_cast<std::size_t>(gg->ny));
    const Grid g = r->grid;
    const std::vector<double>* rows = &r->inlet;
    bcs.inlet_profile = [g, rows](double y) {
      const long j = std::lround((y - g.y_min) / g.dx() - 0.5);
      const double* q = rows->data() + 4 * j;
      return ConservedState{q[0], q[1], q[2], q[3]};
    };
  }
  FieldSnapshot init_f = field_from_planes(r->grid, init);
  init_f.sample_seed = seed;
  r->sim = std::make_unique<Simulation>(r->grid, to_lattice(p), GasParams{p->gamma},
                                        std::move(bcs), init_f);
  r->sim->set_reference(p->rho_ref, p->p_ref);
  *out = r;
  SHIM_CATCH
}

void ref_sim_destroy(void* h) { delete static_cast<RefSim*>(h); }

int ref_sim_step(void* h, double dt) {
  SHIM_TRY static_cast<RefSim*>(h)->sim->step(dt);
  SHIM_CATCH
}

double ref_sim_suggest_dt(void* h) { return static_cast<RefSim*>(h)->sim->suggest_dt(); }
double ref_sim_time(void* h) { return static_cast<RefSim*>(h)->sim->time(); }
long ref_sim_steps(void* h) { return static_cast<RefSim*>(h)->sim->steps(); }
int ref_sim_state_finite(void* h) { return static_cast<RefSim*>(h)->sim->state_finite() ? 1 : 0; }

void ref_sim_get(void* h, double* u, double* pops) {
  RefSim* r = static_cast<RefSim*>(h);
  const int nx = r->grid.nx, ny = r->grid.ny;
  const std::size_t n = r->grid.cells();
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const std::size_t c = static_cast<std::size_t>(j) * nx + i;
      if (u) {
        const ConservedState& s = r->sim->state(i, j);
        for (int k = 0; k < 4; ++k) u[k * n + c] = s[k];
      }
      if (pops) {
        for (int q = 0; q < 4; ++q) {
          const ConservedState& s = r->sim->population(q, i, j);
          for (int k = 0; k < 4; ++k) pops[(4 * q + k) * n + c] = s[k];
        }
      }
    }
}

void ref_sim_set_state(void* h, const double* u) {
  RefSim* r = static_cast<RefSim*>(h);
  const int nx = r->grid.nx, ny = r->grid.ny;
  const std::size_t n = r->grid.cells();
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const std::size_t c = static_cast<std::size_t>(j) * nx + i;
      ConservedState& s = r->sim->state(i, j);
      for (int k = 0; k < 4; ++k) s[k] = u[k * n + c];
    }
}

int ref_sim_compute_blending(void* h, double a, double* tx, double* ty) {
  SHIM_TRY
  RefSim* r = static_cast<RefSim*>(h);
  const BlendingField b = r->sim->compute_blending(a);
  std::memcpy(tx, b.theta_x.data(), sizeof(double) * b.theta_x.size());
  std::memcpy(ty, b.theta_y.data(), sizeof(double) * b.theta_y.size());
  SHIM_CATCH
}

int ref_sim_step_with_blending(void* h, double dt, const double* tx, const double* ty) {
  SHIM_TRY
  RefSim* r = static_cast<RefSim*>(h);
  BlendingField b;
  b.resize(r->grid.nx, r->grid.ny);
  std::memcpy(b.theta_x.data(), tx, sizeof(double) * b.theta_x.size());
  std::memcpy(b.theta_y.data(), ty, sizeof(double) * b.theta_y.size());
  r->sim->step_with_blending(dt, b);
  SHIM_CATCH
}

// ---- run_sample -------------------------------------------------------------

// out_fields: n_times field blocks; out_time/out_div: n_times.
int ref_run_sample(const vlbm_grid* gg, const vlbm_params* p, const vlbm_perturbation* pp, int K,
                   const double* yc, const double* zc, uint64_t seed, double strip,
                   const double* times, int n_times, double* out_fields, double* out_time,
                   int* out_div, long* out_steps, int* out_admissible) {
  SHIM_TRY
  SampleSpec spec;
  spec.grid = to_grid(gg);
  spec.lattice = to_lattice(p);
  spec.gas = GasParams{p->gamma};
  spec.perturbation = to_pert(pp);
  spec.coeffs = to_coeffs(K, yc, zc, seed);
  spec.inlet_strip_width = strip;
  spec.snapshot_times.assign(times, times + n_times);
  const SampleResult res = run_sample(spec);
  const std::size_t n = spec.grid.cells();
  for (int t = 0; t < n_times; ++t) {
    if (out_fields) planes_from_field(res.snapshots[t], out_fields + 4 * n * t);
    if (out_time) out_time[t] = res.snapshots[t].time;
    if (out_div) out_div[t] = res.snapshots[t].diverged ? 1 : 0;
  }
  if (out_steps) *out_steps = res.steps;
  if (out_admissible) *out_admissible = res.admissible ? 1 : 0;
  SHIM_CATCH
}

// ---- metrics ----------------------------------------------------------------

int ref_restrict_field(int nx, int ny, const double* fine, double* coarse) {
  SHIM_TRY
  Grid g;
  g.nx = nx;
  g.ny = ny;
  const FieldSnapshot r = restrict_field(field_from_planes(g, fine));
  planes_from_field(r, coarse);
  SHIM_CATCH
}

static std::vector<FieldSnapshot> ensemble(int M, int64_t n, const double* f) {
  Grid g;
  g.nx = static_cast<int>(n);
  g.ny = 1;
  std::vector<FieldSnapshot> v;
  v.reserve(M);
  for (int m = 0; m < M; ++m) v.push_back(field_from_planes(g, f + 4 * n * m));
  return v;
}

int ref_strong_error(int M, int64_t n, const double* a, const double* b, double* result,
                     double* per_comp) {
  SHIM_TRY
  const auto ea = ensemble(M, n, a), eb = ensemble(M, n, b);
  std::vector<double> comp;
  *result = strong_error(ea, eb, per_comp ? &comp : nullptr);
  if (per_comp)
    for (int k = 0; k < 4; ++k) per_comp[k] = comp[k];
  SHIM_CATCH
}

int ref_wasserstein1(int M, int64_t n, const double* a, const double* b, int var,
                     double* result) {
  SHIM_TRY
  const auto ea = ensemble(M, n, a), eb = ensemble(M, n, b);
  std::vector<const FieldSnapshot*> pa, pb;
  for (const auto& s : ea) pa.push_back(&s);
  for (const auto& s : eb) pb.push_back(&s);
  *result = wasserstein1(pa, pb, static_cast<Variable>(var));
  SHIM_CATCH
}

int ref_ensemble_moments(int M, int64_t n, const double* x, double* mean, double* stddev) {
  SHIM_TRY
  const auto e = ensemble(M, n, x);
  std::vector<const FieldSnapshot*> pe;
  for (const auto& s : e) pe.push_back(&s);
  const auto [mu, sd] = ensemble_moments(pe);
  planes_from_field(mu, mean);
  planes_from_field(sd, stddev);
  SHIM_CATCH
}

double ref_ot_oracle(int n, const double* a, const double* b) {
  return ot_oracle(std::vector<double>(a, a + n), std::vector<double>(b, b + n));
}

double ref_fit_rate(int n, const double* e, const double* dx) {
  return fit_rate(std::vector<double>(e, e + n), std::vector<double>(dx, dx + n));
}

// ---- CPU baseline timing ------------------------------------------------------

// The reference CPU march on `threads` std::threads, one (sample) task at a
// time from an atomic counter exactly like run_ensemble's worker
// (ensemble.hpp:294-332), file I/O excluded.  Each task builds the sample as
// run_sample does and takes `steps` iterations of its loop body
// (suggest_dt -> step -> state_finite, solver.hpp:647-657) with no clamp, or
// (steps < 0) runs run_sample to t_target.  Returns wall seconds; the
// sample-cell-update count goes to *updates.
double ref_march_timed(const vlbm_grid* gg, const vlbm_params* p, const vlbm_perturbation* pp,
                       uint64_t base_seed, long m0, int n_samples, long steps, double t_target,
                       double strip, int threads, long* updates) {
  const Grid grid = to_grid(gg);
  const PerturbationParams pert = to_pert(pp);
  const GasParams gas{p->gamma};
  const LatticeParams lat = to_lattice(p);
  std::atomic<int> next{0};
  std::atomic<long> total{0};
  auto worker = [&]() {
    for (;;) {
      const int t = next.fetch_add(1);
      if (t >= n_samples) return;
      const ModeCoefficients coeffs = draw_coefficients(base_seed, m0 + t, pert.modes);
      long done = 0;
      if (steps < 0) {
        SampleSpec spec;
        spec.grid = grid;
        spec.lattice = lat;
        spec.gas = gas;
        spec.perturbation = pert;
        spec.coeffs = coeffs;
        spec.inlet_strip_width = strip;
        spec.snapshot_times = {t_target};
        done = run_sample(spec).steps;
      } else {
        Boundaries bcs;
        bcs.inlet_profile = [&pert, coeffs, gas](double y) {
          return inlet_state(y, coeffs, pert, gas);
        };
        FieldSnapshot init = initial_field(grid, coeffs, pert, gas, strip);
        Simulation sim(grid, lat, gas, std::move(bcs), init);
        sim.set_reference(pert.rho_amb, pert.p_amb);
        for (long s = 0; s < steps; ++s) {
          const double dt = sim.suggest_dt();
          if (!std::isfinite(dt) || dt <= 0.0) break;
          sim.step(dt);
          ++done;
          if (!sim.state_finite()) break;
        }
      }
      total += done * static_cast<long>(grid.cells());
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  const int nt = std::max(1, std::min(threads, n_samples));
  for (int w = 0; w < nt; ++w) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  if (updates) *updates = total.load();
  return std::chrono::duration<double>(t1 - t0).count();
}

// The reference CPU march over a mid-run window, in two phases on `threads`
// std::threads: (1, untimed) every sample is built as run_sample builds it
// and marched with run_sample's loop body to t_start (dt clamped to hit it,
// solver.hpp:645-657); (2, timed) each sample takes `steps` more iterations of
// suggest_dt -> step -> state_finite (no clamp) -- the same trajectory the
// GPU bench times after run_to(t_start).  Returns the wall seconds of phase
// 2; the sample-cell updates of phase 2 go to *updates, phase 1's wall to
// *pre_seconds.
double ref_march_window(const vlbm_grid* gg, const vlbm_params* p, const vlbm_perturbation* pp,
                        uint64_t base_seed, long m0, int n_samples, double t_start, long steps,
                        double strip, int threads, long* updates, double* pre_seconds) {
  const Grid grid = to_grid(gg);
  const PerturbationParams pert = to_pert(pp);
  const GasParams gas{p->gamma};
  const LatticeParams lat = to_lattice(p);
  std::vector<std::unique_ptr<Simulation>> sims(n_samples);
  std::vector<char> alive(n_samples, 1);
  const int nt = std::max(1, std::min(threads, n_samples));
  auto pool_run = [&](auto&& body) {
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w)
      pool.emplace_back([&]() {
        for (int t; (t = next.fetch_add(1)) < n_samples;) body(t);
      });
    for (auto& th : pool) th.join();
  };
  const auto t0 = std::chrono::steady_clock::now();
  pool_run([&](int t) {
    const ModeCoefficients coeffs = draw_coefficients(base_seed, m0 + t, pert.modes);
    Boundaries bcs;
    bcs.inlet_profile = [&pert, coeffs, gas](double y) { return inlet_state(y, coeffs, pert, gas); };
    FieldSnapshot init = initial_field(grid, coeffs, pert, gas, strip);
    sims[t] = std::make_unique<Simulation>(grid, lat, gas, std::move(bcs), init);
    Simulation& sim = *sims[t];
    sim.set_reference(pert.rho_amb, pert.p_amb);
    constexpr double t_eps = 1e-12;  // solver.hpp:647
    while (sim.time() < t_start - t_eps) {
      double dt = sim.suggest_dt();
      if (!std::isfinite(dt) || dt <= 0.0) {
        alive[t] = 0;
        return;
      }
      dt = std::min(dt, t_start - sim.time());
      sim.step(dt);
      if (!sim.state_finite()) {
        alive[t] = 0;
        return;
      }
    }
  });
  const auto t1 = std::chrono::steady_clock::now();
  std::atomic<long> total{0};
  pool_run([&](int t) {
    if (!alive[t]) return;
    Simulation& sim = *sims[t];
    long done = 0;
    for (long s = 0; s < steps; ++s) {
      const double dt = sim.suggest_dt();
      if (!std::isfinite(dt) || dt <= 0.0) break;
      sim.step(dt);
      ++done;
      if (!sim.state_finite()) break;
    }
    total += done * static_cast<long>(grid.cells());
  });
  const auto t2 = std::chrono::steady_clock::now();
  if (updates) *updates = total.load();
  if (pre_seconds) *pre_seconds = std::chrono::duration<double>(t1 - t0).count();
  return std::chrono::duration<double>(t2 - t1).count();
}

// wasserstein1 + strong_error (+ restrict_field of the fine ensemble) timed as
// compute_metrics runs them (metrics.hpp:284-300), single-threaded.
double ref_postproc_timed(int M, int nxc, int nyc, const double* coarse, const double* fine,
                          double* w1, double* es) {
  Grid gc, gf;
  gc.nx = nxc;
  gc.ny = nyc;
  gf.nx = 2 * nxc;
  gf.ny = 2 * nyc;
  std::vector<FieldSnapshot> ca, fr;
  for (int m = 0; m < M; ++m) {
    ca.push_back(field_from_planes(gc, coarse + 4 * gc.cells() * m));
  }
  std::vector<FieldSnapshot> ff;
  for (int m = 0; m < M; ++m) ff.push_back(field_from_planes(gf, fine + 4 * gf.cells() * m));
  const auto t0 = std::chrono::steady_clock::now();
  for (int m = 0; m < M; ++m) fr.push_back(restrict_field(ff[m]));
  std::vector<const FieldSnapshot*> pa, pb;
  for (const auto& s : ca) pa.push_back(&s);
  for (const auto& s : fr) pb.push_back(&s);
  *w1 = wasserstein1(pa, pb, Variable::Rho);
  *es = strong_error(ca, fr);
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
