// vlbm_b200.hpp — C++ drop-in for the reference's host code, over the C ABI
// of vlbm_b200.h (libvlbm_b200.so, sm_100a kernels; no CPU fallback).
//
// Include it after the reference's own headers (it uses their types and
// their file formats):
//
//   #include "vlbm/metrics.hpp"      // /root/reference/proj/include
//   #include "vlbm_b200.hpp"
//
// and swap the call sites:
//   run_sample(spec)            ->  vlbm::gpu::run_samples({spec, ...})  solver.hpp:625
//   run_ensemble(cfg, ...)      ->  vlbm::gpu::run_ensemble(cfg, ...)    ensemble.hpp:235
//   wasserstein1 / strong_error / restrict_field / ensemble_moments /
//   compute_metrics             ->  vlbm::gpu::<same name>              metrics.hpp:29-327
//   cmd_render (CLI render)     ->  vlbm::gpu::render                   vlbm_main.cpp:67-108
// Same arguments, results (bit-identical), exceptions and files: the
// manifest and the .vlbm snapshots are written by the reference's own
// write_manifest / write_snapshot.
#pragma once

#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vlbm_b200.h"
// the reference headers this drop-in builds on (render.hpp pulls in
// metrics.hpp, ensemble.hpp and solver.hpp)
#include "vlbm/render.hpp"

namespace vlbm::gpu {

inline void check(int rc) {
  if (rc == VLBM_OK) return;
  const std::string msg = vlbm_last_error();
  if (rc == VLBM_E_INVALID) throw std::invalid_argument(msg);
  if (rc == VLBM_E_DOMAIN) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

inline vlbm_grid to_c(const Grid& g) { return {g.nx, g.ny, g.x_max, g.y_min, g.y_max}; }

inline vlbm_params to_c(const LatticeParams& l, const GasParams& gas) {
  vlbm_params p;
  vlbm_default_params(&p);
  p.gamma = gas.gamma;
  p.alpha = l.alpha;
  p.safety = l.safety;
  p.rlmp_relaxation = l.rlmp_relaxation;
  p.positivity_floor = l.positivity_floor;
  p.limiter = static_cast<int>(l.limiter);
  p.conservative_bound = l.conservative_bound ? 1 : 0;
  return p;
}

inline vlbm_perturbation to_c(const PerturbationParams& pp) {
  return {pp.amplitude, pp.modes, pp.decay_exponent, pp.r_jet, pp.rho_jet_bar,
          pp.rho_amb, pp.p_amb, pp.v_jet};
}

// FieldSnapshot data (AoS ConservedState) <-> .vlbm plane blocks.
inline void to_planes(const FieldSnapshot& s, double* out) {
  const std::size_t n = s.data.size();
  for (int k = 0; k < 4; ++k)
    for (std::size_t c = 0; c < n; ++c) out[k * n + c] = s.data[c][k];
}
inline void from_planes(const double* in, FieldSnapshot& s) {
  const std::size_t n = s.data.size();
  for (int k = 0; k < 4; ++k)
    for (std::size_t c = 0; c < n; ++c) s.data[c][k] = in[k * n + c];
}

// RAII handle of a device batch.
class Batch {
 public:
  explicit Batch(vlbm_batch* b) : b_(b) {}
  ~Batch() { vlbm_batch_destroy(b_); }
  Batch(const Batch&) = delete;
  Batch& operator=(const Batch&) = delete;
  vlbm_batch* get() const { return b_; }

 private:
  vlbm_batch* b_;
};

// run_sample (solver.hpp:625-669) for several samples at once.  All specs must
// share grid, lattice, gas, perturbation parameters, strip width and snapshot
// times (one ensemble on one grid); each keeps its own coefficients and its
// own adaptive time step.
inline std::vector<SampleResult> run_samples(const std::vector<SampleSpec>& specs,
                                             int device = 0) {
  std::vector<SampleResult> out(specs.size());
  if (specs.empty()) return out;
  const SampleSpec& s0 = specs.front();
  s0.perturbation.validate();
  for (std::size_t i = 1; i < s0.snapshot_times.size(); ++i)
    if (s0.snapshot_times[i] <= s0.snapshot_times[i - 1])
      throw std::invalid_argument("run_sample: snapshot times must be strictly increasing");
  const int S = static_cast<int>(specs.size());
  const int K = s0.perturbation.modes;
  std::vector<double> y(static_cast<std::size_t>(K) * S), z(y.size());
  for (int s = 0; s < S; ++s) {
    const SampleSpec& sp = specs[s];
    if (!(sp.grid == s0.grid) || sp.snapshot_times != s0.snapshot_times ||
        static_cast<int>(sp.coeffs.y_coeffs.size()) != K ||
        static_cast<int>(sp.coeffs.z_coeffs.size()) != K)
      throw std::invalid_argument("run_samples: specs of one batch must share grid and times");
    std::memcpy(&y[static_cast<std::size_t>(K) * s], sp.coeffs.y_coeffs.data(), sizeof(double) * K);
    std::memcpy(&z[static_cast<std::size_t>(K) * s], sp.coeffs.z_coeffs.data(), sizeof(double) * K);
  }
  const vlbm_grid g = to_c(s0.grid);
  const vlbm_params p = to_c(s0.lattice, s0.gas);
  const vlbm_perturbation pp = to_c(s0.perturbation);
  vlbm_batch* raw = nullptr;
  check(vlbm_batch_create_coeffs(&g, &p, &pp, S, y.data(), z.data(), s0.inlet_strip_width, device,
                                 &raw));
  Batch batch(raw);
  const std::size_t n = s0.grid.cells();
  std::vector<double> fields(4 * n * S), t(S);
  std::vector<int64_t> steps(S);
  std::vector<int> status(S);
  for (double target : s0.snapshot_times) {
    check(vlbm_batch_run_to(batch.get(), target));
    check(vlbm_batch_get_fields(batch.get(), fields.data()));
    check(vlbm_batch_get_scalars(batch.get(), t.data(), steps.data(), status.data()));
    for (int s = 0; s < S; ++s) {
      const bool div = status[s] == VLBM_SAMPLE_DIVERGED;
      FieldSnapshot snap;
      snap.grid = s0.grid;
      snap.time = div ? t[s] : target;
      snap.sample_seed = specs[s].coeffs.seed;
      snap.diverged = div;
      snap.data.resize(n);
      from_planes(&fields[4 * n * s], snap);
      out[s].snapshots.push_back(std::move(snap));
    }
  }
  check(vlbm_batch_get_scalars(batch.get(), t.data(), steps.data(), status.data()));
  for (int s = 0; s < S; ++s) {
    out[s].admissible = status[s] != VLBM_SAMPLE_DIVERGED;
    out[s].steps = steps[s];
  }
  return out;
}

// The batches of one grid of run_ensemble spread over `ndev` GPUs (see
// run_ensemble).  Returns false when should_stop ended the run early.
inline bool run_grid_on_devices(const CaseConfig& cfg, EnsembleManifest& man, std::size_t gi,
                                const std::vector<int>& todo, int ndev, int batch_samples,
                                const std::filesystem::path& manifest_path, EnsembleProgress& prog,
                                const std::function<void(const EnsembleProgress&)>& progress,
                                const std::function<bool()>& should_stop) {
  const Grid grid = cfg.make_grid(gi);
  const std::string grid_dir = "grid_" + grid.label();
  const std::filesystem::path root = cfg.output_dir;
  std::vector<std::pair<std::size_t, std::size_t>> batches;
  // enough batches to keep every device busy, at most batch_samples each
  const std::size_t per = std::max<std::size_t>(
      1, std::min<std::size_t>(batch_samples, (todo.size() + ndev - 1) / ndev));
  for (std::size_t b0 = 0; b0 < todo.size(); b0 += per)
    batches.emplace_back(b0, std::min(todo.size(), b0 + per));
  std::mutex mu;
  std::size_t next = 0;
  bool stopped = false;
  std::exception_ptr err;
  auto worker = [&](int dev) {
    for (;;) {
      std::size_t k;
      {
        std::lock_guard<std::mutex> lock(mu);
        if (stopped || err || next >= batches.size()) return;
        if (should_stop && should_stop()) {
          stopped = true;
          return;
        }
        k = next++;
      }
      try {
        const auto [b0, b1] = batches[k];
        std::vector<SampleSpec> specs;
        for (std::size_t q = b0; q < b1; ++q) {
          SampleSpec spec;
          spec.grid = grid;
          spec.lattice = cfg.lattice;
          spec.gas = cfg.gas;
          spec.perturbation = cfg.perturbation;
          spec.coeffs = man.samples[todo[q]].coeffs;
          spec.inlet_strip_width = cfg.inlet_strip_width;
          spec.snapshot_times = cfg.snapshot_times;
          specs.push_back(std::move(spec));
        }
        const std::vector<SampleResult> results =
            run_samples(specs, dev % std::max(1, vlbm_device_count()));
        std::lock_guard<std::mutex> lock(mu);
        for (std::size_t q = b0; q < b1; ++q) {
          const int m = todo[q];
          const SampleResult& res = results[q - b0];
          std::vector<std::string> rel_files;
          for (std::size_t ti = 0; ti < res.snapshots.size(); ++ti) {
            const std::string rel = grid_dir + "/" + snapshot_filename(m, static_cast<int>(ti));
            write_snapshot(res.snapshots[ti], root / rel);
            rel_files.push_back(rel);
          }
          const bool ok = res.admissible &&
                          admissibility_flag(res.snapshots, cfg.gas, cfg.positivity_admissibility);
          man.samples[m].status[gi] = ok ? RunStatus::Admissible : RunStatus::Diverged;
          man.samples[m].files[gi] = rel_files;
          write_manifest(man, manifest_path);
          ++prog.completed;
          if (!ok) ++prog.diverged;
          if (progress) progress(prog);
        }
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!err) err = std::current_exception();
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int d = 0; d < ndev; ++d) pool.emplace_back(worker, d);
  for (auto& t : pool) t.join();
  if (err) std::rethrow_exception(err);
  return !stopped;
}

// run_ensemble (ensemble.hpp:235-342) with the march on the GPU.  Same
// manifest (format, atomic rewrite after every completion, byte-identical
// config check on resume), same snapshot files and statuses; the work unit is
// a batch of up to `batch_samples` NotRun samples of one grid instead of one
// (sample, grid) task per CPU thread.  should_stop is polled between batches.
// device < 0: every visible GPU, one host thread per device taking batches
// from a shared list (the reference's worker pool with GPUs as workers; the
// snapshot writes and manifest updates are serialised by a mutex, as there).
inline EnsembleManifest run_ensemble(
    const CaseConfig& cfg, const std::function<void(const EnsembleProgress&)>& progress = {},
    const std::function<bool()>& should_stop = {}, int device = 0, int batch_samples = 1024) {
  cfg.validate();
  const std::filesystem::path root = cfg.output_dir;
  std::filesystem::create_directories(root);
  const std::filesystem::path manifest_path = root / "manifest.txt";
  EnsembleManifest man;
  if (std::filesystem::exists(manifest_path)) {
    man = read_manifest(manifest_path);
    if (serialize_config(man.config) != serialize_config(cfg))
      throw std::runtime_error(
          "run_ensemble: output directory holds a manifest for a different configuration");
  } else {
    man.config = cfg;
    man.root = root;
    man.samples.resize(cfg.samples);
    for (int m = 0; m < cfg.samples; ++m) {
      SampleRecord& r = man.samples[m];
      r.index = m;
      r.coeffs = draw_coefficients(cfg.base_seed, m, cfg.perturbation.modes);
      r.seed = r.coeffs.seed;
      r.status.assign(cfg.grids.size(), RunStatus::NotRun);
      r.files.resize(cfg.grids.size());
    }
    write_manifest(man, manifest_path);
  }
  EnsembleProgress prog;
  prog.total = cfg.samples * static_cast<int>(cfg.grids.size());
  for (const SampleRecord& r : man.samples)
    for (RunStatus st : r.status)
      if (st != RunStatus::NotRun) {
        ++prog.completed;
        if (st == RunStatus::Diverged) ++prog.diverged;
      }
  for (std::size_t gi = 0; gi < cfg.grids.size(); ++gi) {
    const Grid grid = cfg.make_grid(gi);
    const std::string grid_dir = "grid_" + grid.label();
    std::filesystem::create_directories(root / grid_dir);
    std::vector<int> todo;
    for (int m = 0; m < cfg.samples; ++m)
      if (man.samples[m].status[gi] == RunStatus::NotRun) todo.push_back(m);
    // workers: every visible GPU (VLBM_DEVICES overrides the count; worker w
    // runs on device w mod the visible count -- a test hook for this path)
    int ndev = 1;
    if (device < 0) {
      ndev = std::max(1, vlbm_device_count());
      if (const char* e = std::getenv("VLBM_DEVICES")) ndev = std::max(1, std::atoi(e));
    }
    if (ndev > 1) {
      if (!run_grid_on_devices(cfg, man, gi, todo, ndev, batch_samples, manifest_path, prog,
                               progress, should_stop))
        return man;
      continue;
    }
    for (std::size_t b0 = 0; b0 < todo.size(); b0 += batch_samples) {
      if (should_stop && should_stop()) return man;
      const std::size_t b1 = std::min(todo.size(), b0 + static_cast<std::size_t>(batch_samples));
      std::vector<SampleSpec> specs;
      for (std::size_t q = b0; q < b1; ++q) {
        SampleSpec spec;
        spec.grid = grid;
        spec.lattice = cfg.lattice;
        spec.gas = cfg.gas;
        spec.perturbation = cfg.perturbation;
        spec.coeffs = man.samples[todo[q]].coeffs;
        spec.inlet_strip_width = cfg.inlet_strip_width;
        spec.snapshot_times = cfg.snapshot_times;
        specs.push_back(std::move(spec));
      }
      const std::vector<SampleResult> results = run_samples(specs, device < 0 ? 0 : device);
      for (std::size_t q = b0; q < b1; ++q) {
        const int m = todo[q];
        const SampleResult& res = results[q - b0];
        std::vector<std::string> rel_files;
        for (std::size_t ti = 0; ti < res.snapshots.size(); ++ti) {
          const std::string rel = grid_dir + "/" + snapshot_filename(m, static_cast<int>(ti));
          write_snapshot(res.snapshots[ti], root / rel);
          rel_files.push_back(rel);
        }
        const bool ok = res.admissible &&
                        admissibility_flag(res.snapshots, cfg.gas, cfg.positivity_admissibility);
        man.samples[m].status[gi] = ok ? RunStatus::Admissible : RunStatus::Diverged;
        man.samples[m].files[gi] = rel_files;
        write_manifest(man, manifest_path);
        ++prog.completed;
        if (!ok) ++prog.diverged;
        if (progress) progress(prog);
      }
    }
  }
  return man;
}

// ---- metrics (metrics.hpp:29-177) on the device ------------------------------

inline FieldSnapshot restrict_field(const FieldSnapshot& fine) {
  if (fine.grid.nx % 2 != 0 || fine.grid.ny % 2 != 0)
    throw std::invalid_argument("restrict_field: fine dimensions must be even");
  FieldSnapshot c;
  c.grid = fine.grid;
  c.grid.nx = fine.grid.nx / 2;
  c.grid.ny = fine.grid.ny / 2;
  c.time = fine.time;
  c.sample_seed = fine.sample_seed;
  c.diverged = fine.diverged;
  c.data.resize(c.grid.cells());
  std::vector<double> f(4 * fine.data.size()), o(4 * c.data.size());
  to_planes(fine, f.data());
  check(vlbm_restrict_field(fine.grid.nx, fine.grid.ny, f.data(), o.data()));
  from_planes(o.data(), c);
  return c;
}

inline double strong_error(const std::vector<FieldSnapshot>& coarse,
                           const std::vector<FieldSnapshot>& restricted_fine,
                           std::vector<double>* per_component = nullptr) {
  if (coarse.empty() || coarse.size() != restricted_fine.size())
    throw std::invalid_argument("strong_error: sample counts differ or are empty");
  const std::size_t n = coarse[0].data.size();
  std::vector<double> a(4 * n * coarse.size()), b(a.size());
  for (std::size_t m = 0; m < coarse.size(); ++m) {
    if (coarse[m].data.size() != n || restricted_fine[m].data.size() != n)
      throw std::invalid_argument("strong_error: grid mismatch between coarse and restricted");
    to_planes(coarse[m], &a[4 * n * m]);
    to_planes(restricted_fine[m], &b[4 * n * m]);
  }
  double r = 0.0, pc[4];
  check(vlbm_strong_error(static_cast<int>(coarse.size()), static_cast<int64_t>(n), a.data(),
                          b.data(), &r, pc));
  if (per_component) per_component->assign(pc, pc + 4);
  return r;
}

inline double wasserstein1(const std::vector<const FieldSnapshot*>& a,
                           const std::vector<const FieldSnapshot*>& b,
                           Variable var = Variable::Rho) {
  if (a.empty() || a.size() != b.size())
    throw std::invalid_argument("wasserstein1: sample counts differ or are empty");
  const std::size_t n = a[0]->data.size();
  std::vector<double> pa(4 * n * a.size()), pb(pa.size());
  for (std::size_t m = 0; m < a.size(); ++m) {
    if (a[m]->data.size() != n || b[m]->data.size() != n)
      throw std::invalid_argument("wasserstein1: inconsistent field sizes");
    to_planes(*a[m], &pa[4 * n * m]);
    to_planes(*b[m], &pb[4 * n * m]);
  }
  double r = 0.0;
  check(vlbm_wasserstein1(static_cast<int>(a.size()), static_cast<int64_t>(n), pa.data(),
                          pb.data(), static_cast<int>(var), &r));
  return r;
}

inline std::pair<FieldSnapshot, FieldSnapshot> ensemble_moments(
    const std::vector<const FieldSnapshot*>& samples) {
  if (samples.empty()) throw std::invalid_argument("ensemble_moments: no samples");
  const std::size_t n = samples[0]->data.size();
  std::vector<double> x(4 * n * samples.size()), mu(4 * n), sd(4 * n);
  for (std::size_t m = 0; m < samples.size(); ++m) {
    if (samples[m]->data.size() != n) throw std::invalid_argument("ensemble_moments: size mismatch");
    to_planes(*samples[m], &x[4 * n * m]);
  }
  check(vlbm_ensemble_moments(static_cast<int>(samples.size()), static_cast<int64_t>(n), x.data(),
                              mu.data(), sd.data()));
  FieldSnapshot mean = *samples[0], stddev = *samples[0];
  from_planes(mu.data(), mean);
  from_planes(sd.data(), stddev);
  return {std::move(mean), std::move(stddev)};
}

// compute_metrics (metrics.hpp:259-327): W1, E_strong and M* per grid pair and
// snapshot time, then the per-time rate fits (host scalar work, reference
// fit_rate).  Device resident: for each (pair, time) the jointly valid
// samples' coarse and fine snapshots are read (reference read_snapshot) in
// batches on a reader thread while the device takes the previous batch --
// each ensemble is uploaded once (vlbm_metrics_*: strong_error partials with
// the restriction fused as each batch lands, the metric variable's planes
// kept on the device, W1 over them at the end); no field is restricted or
// reduced on the host.
inline MetricsReport compute_metrics(const EnsembleManifest& man, int device = 0) {
  const CaseConfig& cfg = man.config;
  if (cfg.grids.size() < 2) throw std::runtime_error("metrics: need >= 2 grids for Cauchy errors");
  const Variable var = variable_from_name(cfg.metric_variable);
  MetricsReport rep;
  const std::size_t n_pairs = cfg.grids.size() - 1, n_times = cfg.snapshot_times.size();
  std::vector<std::vector<double>> w1s(n_pairs, std::vector<double>(n_times)),
      strongs(n_pairs, std::vector<double>(n_times));
  std::vector<double> coarse_dx(n_pairs);
  for (std::size_t p = 0; p < n_pairs; ++p) {
    const Grid cg = cfg.make_grid(p), fg = cfg.make_grid(p + 1);
    if (fg.nx != 2 * cg.nx || fg.ny != 2 * cg.ny)
      throw std::runtime_error("metrics: consecutive grids must refine by exactly 2x");
    coarse_dx[p] = cg.dx();
    const ValidityMask mask = joint_validity(man, p, p + 1);
    const int m_star = mask.m_star();
    if (m_star < 1) throw std::runtime_error("metrics: no jointly valid samples for pair");
    std::vector<std::size_t> valid;
    for (std::size_t m = 0; m < man.samples.size(); ++m)
      if (mask.mask[m]) valid.push_back(m);
    const std::size_t nc = static_cast<std::size_t>(cg.cells()), nf = 4 * nc;
    // reader batches of about 256 MiB of host fields
    const std::size_t B = std::max<std::size_t>(
        1, std::min<std::size_t>(valid.size(), (256u << 20) / (32 * (nc + nf))));
    for (std::size_t ti = 0; ti < n_times; ++ti) {
      struct Batch {
        std::vector<double> c, f;
      };
      auto read_batch = [&](std::size_t b0, Batch& out) {
        const std::size_t nb = std::min(B, valid.size() - b0);
        out.c.resize(4 * nc * nb);
        out.f.resize(4 * nf * nb);
        for (std::size_t k = 0; k < nb; ++k) {
          const auto& rec = man.samples[valid[b0 + k]];
          to_planes(read_snapshot(man.root / rec.files[p][ti], cg), &out.c[4 * nc * k]);
          to_planes(read_snapshot(man.root / rec.files[p + 1][ti], fg), &out.f[4 * nf * k]);
        }
      };
      vlbm_metrics* ctx = nullptr;
      check(vlbm_metrics_begin(m_star, cg.nx, cg.ny, static_cast<int>(var), device, &ctx));
      struct Guard {
        vlbm_metrics* c;
        ~Guard() { vlbm_metrics_destroy(c); }
      } guard{ctx};
      Batch cur, next;
      read_batch(0, cur);
      for (std::size_t b0 = 0; b0 < valid.size(); b0 += B) {
        std::exception_ptr err;
        std::thread reader;
        if (b0 + B < valid.size())
          reader = std::thread([&] {
            try {
              read_batch(b0 + B, next);
            } catch (...) {
              err = std::current_exception();
            }
          });
        const int nb = static_cast<int>(std::min(B, valid.size() - b0));
        const int rc = vlbm_metrics_add(ctx, static_cast<int>(b0), nb, cur.c.data(), cur.f.data());
        if (reader.joinable()) reader.join();
        check(rc);
        if (err) std::rethrow_exception(err);
        std::swap(cur, next);
      }
      MetricsRow row;
      row.time = cfg.snapshot_times[ti];
      row.pair = std::to_string(cg.nx) + "->" + std::to_string(fg.nx);
      row.m_star = m_star;
      check(vlbm_metrics_finish(ctx, &row.w1, &row.e_strong, nullptr));
      w1s[p][ti] = row.w1;
      strongs[p][ti] = row.e_strong;
      rep.rows.push_back(row);
    }
  }
  for (std::size_t ti = 0; ti < n_times; ++ti) {
    RateRow rr;
    rr.time = cfg.snapshot_times[ti];
    std::vector<double> ew, es;
    for (std::size_t p = 0; p < n_pairs; ++p) {
      ew.push_back(w1s[p][ti]);
      es.push_back(strongs[p][ti]);
    }
    auto safe_fit = [&](const std::vector<double>& e) {
      try {
        return fit_rate(e, coarse_dx);
      } catch (const std::invalid_argument&) {
        return std::numeric_limits<double>::quiet_NaN();
      }
    };
    rr.r_w1 = safe_fit(ew);
    rr.r_strong = safe_fit(es);
    rep.rates.push_back(rr);
  }
  return rep;
}

// The CLI's render command (tools/vlbm_main.cpp cmd_render) with the
// ensemble moments on the device: what = "sample:M", "mean" or "std"; the
// PPM is written by the reference's render_ppm (render.hpp:52-80).  Same
// arguments, exceptions and output file.
inline void render(const EnsembleManifest& man, int time_index, const std::string& what,
                   std::string grid_label, const std::string& variable, const std::string& out) {
  const CaseConfig& cfg = man.config;
  if (grid_label.empty()) grid_label = cfg.make_grid(cfg.grids.size() - 1).label();
  const std::size_t gi = man.grid_index(grid_label);
  if (time_index < 0 || time_index >= static_cast<int>(cfg.snapshot_times.size()))
    throw std::runtime_error("render: time index out of range");
  const Variable var = variable_from_name(variable);
  FieldSnapshot field;
  if (what.rfind("sample:", 0) == 0) {
    const int m = std::stoi(what.substr(7));
    if (m < 0 || m >= static_cast<int>(man.samples.size()))
      throw std::runtime_error("render: sample index out of range");
    if (man.samples[m].status[gi] != RunStatus::Admissible)
      throw std::runtime_error("render: sample " + std::to_string(m) + " on grid " + grid_label +
                               " is not admissible");
    field = read_snapshot(man.root / man.samples[m].files[gi][time_index], cfg.make_grid(gi));
  } else if (what == "mean" || what == "std") {
    std::vector<FieldSnapshot> fields;
    for (const SampleRecord& r : man.samples) {
      if (r.status[gi] != RunStatus::Admissible) continue;
      fields.push_back(read_snapshot(man.root / r.files[gi][time_index], cfg.make_grid(gi)));
    }
    if (fields.size() < 2) throw std::runtime_error("render: need >= 2 admissible samples");
    std::vector<const FieldSnapshot*> ptrs;
    for (const auto& f : fields) ptrs.push_back(&f);
    auto [mean, stddev] = gpu::ensemble_moments(ptrs);
    field = what == "mean" ? std::move(mean) : std::move(stddev);
  } else {
    throw std::runtime_error("render: --what must be sample:M, mean, or std");
  }
  render_ppm(field, var, cfg.render_floor, cfg.colormap, out);
}

}  // namespace vlbm::gpu
