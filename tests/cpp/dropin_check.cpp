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
//   dropin_check metrics <dir>      compute_metrics vs gpu::compute_metrics on
//                                   that ensemble: identical rows (bitwise)
//   dropin_check outputs <dir>      metrics / rates CSVs (write_metrics_csv) and
//                                   rendered PPMs (cmd_render vs gpu::render:
//                                   mean, std, sample; rho, energy) byte-identical
#include <cstdio>
#include <cstring>
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

static int check_ensemble(const fs::path& dir, int M) {
  const fs::path run = dir / "run", cpu = dir / "cpu";
  fs::remove_all(dir);
  const CaseConfig cfg = smoke_case(run.string(), M);
  run_ensemble(cfg);  // the reference, on all host threads
  fs::rename(run, cpu);
  int calls = 0;
  gpu::run_ensemble(cfg, [&calls](const EnsembleProgress&) { ++calls; });
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

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "ic") return check_ic();
    if (mode == "nogpu") return check_nogpu();
    if (mode == "ensemble" && argc >= 3) return check_ensemble(argv[2], argc > 3 ? std::atoi(argv[3]) : 8);
    if (mode == "metrics" && argc >= 3) return check_metrics(argv[2]);
    if (mode == "outputs" && argc >= 3) return check_outputs(argv[2]);
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 3;
  }
  return 2;
}
