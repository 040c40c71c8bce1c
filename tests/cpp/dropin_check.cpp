// tests/cpp/dropin_check.cpp — TEST INFRASTRUCTURE: the C++ drop-in
// (include/vlbm_b200.hpp) against the reference's own host code, compiled
// together from the unmodified reference headers (/root/reference/proj/include)
// by tests/cpp/Makefile; the binary travels to the GPU box.
//
//   dropin_check ic                 host IC identical (no GPU needed)
//   dropin_check nogpu              the march throws std::runtime_error
//   dropin_check ensemble <dir> [M] reference run_ensemble vs gpu::run_ensemble
//                                   on a smoke-style case: byte-identical
//                                   output directories (manifest + snapshots)
//   dropin_check ensemble_all <dir> [M]  the same through the multi-GPU worker
//                                   path (run_ensemble device -1; VLBM_DEVICES)
//   dropin_check metrics <dir>      compute_metrics vs gpu::compute_metrics on
//                                   that ensemble: identical rows (bitwise)
//   dropin_check outputs <dir>      metrics / rates CSVs (write_metrics_csv) and
//                                   rendered PPMs (cmd_render vs gpu::render:
//                                   mean, std, sample; rho, energy) byte-identical
//   dropin_check acceptance <dir>   the reference's acceptance criteria 6-9 with
//                                   the GPU drop-ins (reference's output format)
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>

#include "vlbm/metrics.hpp"
#include "vlbm/render.hpp"
#include "vlbm_b200.hpp"

using namespace vlbm;
namespace fs = std::filesystem;

static std::map<std::string, std::string> dir_bytes(const fs::path& root) {
  std::map<std::string, std::string> out;
  for (const auto& e : fs::recursive_directory_iterator(root)) {
    if (!e.is_regular_file()) continue;
    std::ifstream in(e.path(), std::ios::binary);
    std::ostringstream ss;
    ss << in.rdbuf();
    out[fs::relative(e.path(), root).string()] = ss.str();
  }
  return out;
}

static CaseConfig smoke_case(const std::string& out_dir, int M) {
  CaseConfig cfg;  // reference defaults: jet physics, snapshot times 0..0.003
  cfg.grids = {{125, 25}, {250, 50}};
  cfg.samples = M;
  cfg.output_dir = out_dir;
  cfg.workers = 0;
  return cfg;
}

static int check_ic() {
  int bad = 0;
  for (uint64_t m = 0; m < 64; ++m) {
    const ModeCoefficients c = draw_coefficients(42, m, 10);
    double y[10], z[10];
    const uint64_t seed = vlbm_draw_coefficients(42, m, 10, y, z);
    if (seed != c.seed || std::memcmp(y, c.y_coeffs.data(), sizeof y) ||
        std::memcmp(z, c.z_coeffs.data(), sizeof z))
      ++bad;
    const Grid g = CaseConfig{}.make_grid(0);
    std::vector<double> rows(4 * g.ny);
    const vlbm_grid cg = gpu::to_c(g);
    const vlbm_perturbation pp = gpu::to_c(PerturbationParams{});
    gpu::check(vlbm_inlet_rows(&cg, &pp, 5.0 / 3.0, y, z, rows.data()));
    for (int j = 0; j < g.ny; ++j) {
      const ConservedState u = inlet_state(g.y_center(j), c, PerturbationParams{}, GasParams{});
      for (int k = 0; k < 4; ++k) {
        const double want = u[k];
        if (std::memcmp(&rows[4 * j + k], &want, sizeof(double))) ++bad;
      }
    }
  }
  std::printf("ic: %d mismatches\n", bad);
  return bad ? 1 : 0;
}

static int check_nogpu() {
  SampleSpec spec;
  spec.grid = Grid{40, 8};
  spec.coeffs = draw_coefficients(42, 0, 10);
  spec.snapshot_times = {0.0};
  try {
    gpu::run_samples({spec});
  } catch (const std::runtime_error& e) {
    std::printf("nogpu: runtime_error: %s\n", e.what());
    return 0;
  }
  std::printf("nogpu: no exception\n");
  return 1;
}

static int check_ensemble(const fs::path& dir, int M, int device = 0) {
  const fs::path run = dir / "run", cpu = dir / "cpu";
  fs::remove_all(dir);
  const CaseConfig cfg = smoke_case(run.string(), M);
  run_ensemble(cfg);  // the reference, on all host threads
  fs::rename(run, cpu);
  int calls = 0;
  gpu::run_ensemble(cfg, [&calls](const EnsembleProgress&) { ++calls; }, {}, device);
  const auto a = dir_bytes(cpu), b = dir_bytes(run);
  int diff = 0;
  for (const auto& [k, v] : a) {
    auto it = b.find(k);
    if (it == b.end() || it->second != v) {
      if (diff < 5) std::printf("differs: %s\n", k.c_str());
      ++diff;
    }
  }
  if (a.size() != b.size()) ++diff;
  std::printf("ensemble: %zu files, %d differ, progress calls %d\n", a.size(), diff, calls);
  return diff ? 1 : 0;
}

static int check_metrics(const fs::path& dir) {
  const EnsembleManifest man = read_manifest(dir / "run" / "manifest.txt");
  const MetricsReport want = compute_metrics(man);
  const MetricsReport got = gpu::compute_metrics(man);
  int bad = want.rows.size() != got.rows.size();
  for (std::size_t i = 0; i < want.rows.size() && !bad; ++i) {
    const auto& w = want.rows[i];
    const auto& g = got.rows[i];
    if (std::memcmp(&w.w1, &g.w1, 8) || std::memcmp(&w.e_strong, &g.e_strong, 8) ||
        w.m_star != g.m_star || w.pair != g.pair)
      ++bad;
    std::printf("t=%g %s M*=%d W1 %.17g/%.17g E %.17g/%.17g\n", w.time, w.pair.c_str(), w.m_star,
                w.w1, g.w1, w.e_strong, g.e_strong);
  }
  return bad ? 1 : 0;
}

static std::string file_bytes(const fs::path& p) {
  std::ifstream f(p, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(f), {});
}

// The metrics / rates CSVs (write_metrics_csv over the two reports) and the
// rendered PPMs (cmd_render's path vs gpu::render) must be byte-identical.
static int check_outputs(const fs::path& dir) {
  const EnsembleManifest man = read_manifest(dir / "run" / "manifest.txt");
  const MetricsReport want = compute_metrics(man);
  const MetricsReport got = gpu::compute_metrics(man);
  write_metrics_csv(want, dir / "cpu_metrics.csv", dir / "cpu_rates.csv");
  write_metrics_csv(got, dir / "gpu_metrics.csv", dir / "gpu_rates.csv");
  int bad = 0;
  for (const char* k : {"metrics", "rates"}) {
    const bool same = file_bytes(dir / (std::string("cpu_") + k + ".csv")) ==
                      file_bytes(dir / (std::string("gpu_") + k + ".csv"));
    bad += !same;
    std::printf("%s csv: %s\n", k, same ? "identical" : "DIFFERS");
  }
  const CaseConfig& cfg = man.config;
  int renders = 0;
  for (std::size_t gi = 0; gi < cfg.grids.size(); ++gi) {
    const std::string label = cfg.make_grid(gi).label();
    for (int ti = 0; ti < static_cast<int>(cfg.snapshot_times.size()); ++ti) {
      for (const std::string what : {"mean", "std", "sample:3"}) {
        for (const std::string var : {"rho", "energy"}) {
          // the reference's cmd_render path: host ensemble_moments + render_ppm
          FieldSnapshot field;
          if (what == "sample:3") {
            field = read_snapshot(man.root / man.samples[3].files[gi][ti], cfg.make_grid(gi));
          } else {
            std::vector<FieldSnapshot> fields;
            for (const SampleRecord& r : man.samples)
              if (r.status[gi] == RunStatus::Admissible)
                fields.push_back(read_snapshot(man.root / r.files[gi][ti], cfg.make_grid(gi)));
            std::vector<const FieldSnapshot*> ptrs;
            for (const auto& f : fields) ptrs.push_back(&f);
            auto [mean, stddev] = ensemble_moments(ptrs);
            field = what == "mean" ? mean : stddev;
          }
          const fs::path a = dir / "cpu.ppm", b = dir / "gpu.ppm";
          render_ppm(field, variable_from_name(var), cfg.render_floor, cfg.colormap, a.string());
          gpu::render(man, ti, what, label, var, b.string());
          const bool same = file_bytes(a) == file_bytes(b);
          bad += !same;
          ++renders;
          if (!same) std::printf("render %s t%d %s %s DIFFERS\n", label.c_str(), ti, what.c_str(), var.c_str());
        }
      }
    }
  }
  std::printf("renders: %d compared, %d differ\n", renders, bad);
  return bad ? 1 : 0;
}

// The reference's acceptance criteria 6-9 (tests/acceptance.cpp:251-402)
// re-run with the GPU drop-ins in place of run_sample / run_ensemble /
// compute_metrics; the lines are printed in the reference's own format so
// they can be compared with its recorded results (tests/golden/acceptance.json).
static void accept_report(int number, const std::string& label, bool pass,
                          const std::string& detail) {
  std::printf("criterion %2d %-28s %s  (%s)\n", number, label.c_str(), pass ? "PASS" : "FAIL",
              detail.c_str());
}

static std::string afmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  std::vsnprintf(buf, sizeof(buf), f, ap);
  va_end(ap);
  return buf;
}

static int check_acceptance(const fs::path& dir) {
  {  // criterion 6: jet-head velocity of the unperturbed jet (acceptance.cpp:251-281)
    PerturbationParams pp;
    pp.amplitude = 0.0;
    SampleSpec spec;
    spec.grid = Grid{500, 100};
    spec.gas = GasParams{5.0 / 3.0};
    spec.perturbation = pp;
    spec.coeffs = draw_coefficients(42, 0, pp.modes);
    spec.snapshot_times = {0.001, 0.0015, 0.002, 0.0025, 0.003};
    const SampleResult res = gpu::run_samples({spec})[0];
    std::vector<double> ts, xs;
    for (const FieldSnapshot& sn : res.snapshots) {
      ts.push_back(sn.time);
      xs.push_back(jet_head_position(sn, pp.rho_amb, pp.r_jet, 2.0));
    }
    const double v = fit_slope(ts, xs);
    accept_report(6, "jet-head velocity", res.admissible && std::abs(v - 666.7) <= 0.10 * 666.7,
                  afmt("fitted head speed %.1f over t in [0.001,0.003], want 666.7 +/- 10%%", v));
  }
  CaseConfig cfg;  // the 64-sample, three-grid desk case (acceptance.cpp:285-293)
  cfg.output_dir = (dir / "accept").string();
  const EnsembleManifest man = gpu::run_ensemble(cfg);
  {  // criterion 7 (acceptance.cpp:295-317)
    const MetricsReport rep = gpu::compute_metrics(man);
    double r_w1_end = NAN, r_s_end = NAN, r_w1_0 = NAN, r_s_0 = NAN;
    for (const RateRow& r : rep.rates) {
      if (std::abs(r.time - man.config.t_end) < 1e-12) r_w1_end = r.r_w1, r_s_end = r.r_strong;
      if (r.time == 0.0) r_w1_0 = r.r_w1, r_s_0 = r.r_strong;
    }
    auto in = [](double v, double lo, double hi) { return v >= lo && v <= hi; };
    const bool pass = (r_w1_end - r_s_end) >= 0.2 && r_s_end <= 0.2 && in(r_w1_0, 0.8, 1.2) &&
                      in(r_s_0, 0.8, 1.2);
    accept_report(7, "statistical rate separation", pass,
                  afmt("t=end: r_W1 %.3f, r_strong %.3f (need gap >= 0.2, r_strong <= 0.2); "
                       "t=0: %.3f/%.3f (need [0.8,1.2])",
                       r_w1_end, r_s_end, r_w1_0, r_s_0));
  }
  {  // criterion 8: determinism and resume (acceptance.cpp:358-402), one sample per batch
    CaseConfig c8;
    c8.grids = {{40, 8}, {80, 16}};
    c8.samples = 4;
    c8.t_end = 0.0005;
    c8.snapshot_times = {0.0, 0.00025, 0.0005};
    const fs::path root = dir / "det";
    c8.output_dir = (root / "run").string();
    auto execute = [&](const std::function<bool()>& stop) {
      const EnsembleManifest m = gpu::run_ensemble(c8, {}, stop, 0, 1);
      bool complete = true;
      for (const SampleRecord& r : m.samples)
        for (RunStatus st : r.status)
          if (st == RunStatus::NotRun) complete = false;
      if (complete) {
        const MetricsReport rep = gpu::compute_metrics(m);
        write_metrics_csv(rep, m.root / "metrics.csv", m.root / "rates.csv");
      }
    };
    fs::remove_all(root);
    execute({});
    const auto first = dir_bytes(c8.output_dir);
    fs::remove_all(root);
    execute({});
    const bool rerun_same = dir_bytes(c8.output_dir) == first;
    fs::remove_all(root);
    int done = 0;
    execute([&done] { return ++done > 3; });
    const bool was_partial = dir_bytes(c8.output_dir) != first;
    execute({});
    const bool resume_same = dir_bytes(c8.output_dir) == first;
    accept_report(8, "determinism and resume", rerun_same && was_partial && resume_same,
                  afmt("rerun identical: %s; interrupted run partial: %s; resumed identical: %s",
                       rerun_same ? "yes" : "no", was_partial ? "yes" : "no",
                       resume_same ? "yes" : "no"));
  }
  {  // criterion 9 (acceptance.cpp:319-352)
    const double eps = 1e-7;
    const GasParams gas = man.config.gas;
    const double rho_floor = eps * man.config.perturbation.rho_amb;
    const double p_floor = eps * man.config.perturbation.p_amb;
    double min_rho = INFINITY, min_p = INFINITY;
    int admissible = 0, diverged = 0;
    for (std::size_t gi = 0; gi < man.config.grids.size(); ++gi) {
      for (std::size_t m = 0; m < man.samples.size(); ++m) {
        if (man.samples[m].status[gi] == RunStatus::Diverged) {
          ++diverged;
          continue;
        }
        ++admissible;
        for (const FieldSnapshot& sn : load_sample_snapshots(man, gi, static_cast<int>(m))) {
          for (const ConservedState& u : sn.data) {
            min_rho = std::min(min_rho, u.rho);
            min_p = std::min(min_p, pressure(u, gas));
          }
        }
      }
    }
    accept_report(9, "positivity across ensemble", min_rho >= rho_floor && min_p >= p_floor,
                  afmt("min rho %.3e (floor %.3e), min p %.3e (floor %.3e); %d admissible, "
                       "%d diverged runs all recorded",
                       min_rho, rho_floor, min_p, p_floor, admissible, diverged));
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "ic") return check_ic();
    if (mode == "nogpu") return check_nogpu();
    if (mode == "ensemble" && argc >= 3) return check_ensemble(argv[2], argc > 3 ? std::atoi(argv[3]) : 8);
    if (mode == "ensemble_all" && argc >= 3)  // device -1: the multi-GPU worker path
      return check_ensemble(argv[2], argc > 3 ? std::atoi(argv[3]) : 8, -1);
    if (mode == "metrics" && argc >= 3) return check_metrics(argv[2]);
    if (mode == "outputs" && argc >= 3) return check_outputs(argv[2]);
    if (mode == "acceptance" && argc >= 3) return check_acceptance(argv[2]);
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 3;
  }
  return 2;
}
