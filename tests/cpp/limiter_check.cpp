// tests/cpp/limiter_check.cpp — TEST INFRASTRUCTURE: the device limiter
// (paper_2605_25282_b200/csrc/rlmp.cuh, rlmp_replay.cuh) compiled for the host
// and run on limiter inputs dumped by the C oracle (vo_sim_limiter_cells):
// every path the kernels take must reproduce the reference's theta bit for bit
//   plain     rlmp_theta_hard_plain (30 full feasible() steps)
//   queued    rlmp_hard_stage + bisect_certified / bisect_uncertified (replay off)
//   replay    rlmp_hard_stage + bisect_replay with at most kReplayInline exact
//             steps, the rest resumed by bisect_uncertified (k_bisect_tail)
// and the theta = 1 quadratic-form decision of the vertex floors
// (vertex_floors_quadform) must never contradict the exact checks.
// The audit counters (a re-run of the full feasible() at every step) must
// stay zero.  Output: one JSON line of counts.
// usage: limiter_check records.bin   (27 doubles per cell, see vlbm_oracle.h)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
using std::isfinite;
using std::isinf;
using std::isnan;
#define __device__
#define __host__
#define __forceinline__ inline
static inline int __popc(unsigned x) { return __builtin_popcount(x); }
static inline int __ffs(int x) { return __builtin_ffs(x); }
static inline double __longlong_as_double(long long x) {
  double d;
  std::memcpy(&d, &x, 8);
  return d;
}
static inline unsigned long long atomicAdd(unsigned long long* p, unsigned long long v) {
  const unsigned long long o = *p;
  *p += v;
  return o;
}
#include "rlmp_replay.cuh"

using namespace vlbm_dev;

static bool same(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: limiter_check records.bin gamma\n");
    return 2;
  }
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  const double gm1 = std::atof(argv[2]) - 1.0;
  double r[27];
  long cells = 0, at_one = 0, hard = 0, bisect = 0, stopped = 0;
  long bad_plain = 0, bad_queued = 0, bad_replay = 0, margin_bad = 0;
  long quad_pass = 0, quad_fail = 0, quad_open = 0, quad_bad = 0;
  unsigned long long audit[16] = {0};
  while (std::fread(r, sizeof r, 1, f) == 1) {
    ++cells;
    const cs fo = {r[0], r[1], r[2], r[3]};
    cs cf[4];
    for (int q = 0; q < 4; ++q) cf[q] = {r[4 + 4 * q], r[5 + 4 * q], r[6 + 4 * q], r[7 + 4 * q]};
    RlmpBounds b = {r[20], r[21], r[22], r[23], r[24], r[25]};
    const double want = r[26];
    const cs delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
    if (diag_ok(1.0, fo, delta, b, gm1)) {
      const bool ok = vertex_floors_ok(1.0, fo, cf, b, gm1);
      // the quadratic-form decision of the same 15 checks: never contradicts them
      const int q = vertex_floors_quadform(fo, cf, b.rho_floor, b.p_floor, gm1, 1.0 / gm1);
      quad_pass += q == 1;
      quad_fail += q == 0;
      quad_open += q < 0;
      quad_bad += (q == 1 && !ok) || (q == 0 && ok);
      if (ok) {
        ++at_one;
        bad_plain += !same(want, 1.0);
        continue;
      }
    }
    ++hard;
    bad_plain += !same(rlmp_theta_hard_plain(fo, cf, b, gm1), want);
    if (!(finite4(fo) && finite4(cf[0]) && finite4(cf[1]) && finite4(cf[2]) && finite4(cf[3]) &&
          finite4(delta)))
      continue;  // the kernels take the plain path for these
    const HardStage h = rlmp_hard_stage(fo, cf, delta, b, gm1);
    if (h.done) {
      bad_queued += !same(h.result, want);
      bad_replay += !same(h.result, want);
      continue;
    }
    ++bisect;
    {  // every vertex the stage marks as clearing the margins at thc really does
      const cs t[4] = {scale(h.thc, cf[0]), scale(h.thc, cf[1]), scale(h.thc, cf[2]),
                       scale(h.thc, cf[3])};
      for (int S = 1; S < 16; ++S) {
        if (!(h.mhi >> S & 1)) continue;
        const cs v = vertex_at(fo, t, S);
        const double p = pressure(v, gm1);
        margin_bad += !vertex_margin(p, p, v.r, v.r, b, h.err, h.er);
      }
    }
    const double q = h.unc ? bisect_uncertified(fo, cf, delta, b, h, gm1, audit)
                           : bisect_certified(fo, delta, b, h.thc, gm1);
    bad_queued += !same(q, want);
    Bracket br;
    double t;
    if (bisect_replay(fo, cf, delta, b, h, gm1, 1, br, audit)) {
      t = br.lo;
    } else {
      ++stopped;
      t = bisect_uncertified(fo, cf, delta, b, h, gm1, audit, br.lo, br.hi, br.it);
    }
    bad_replay += !same(t, want);
  }
  std::fclose(f);
  // hypot_ref (signal speed with the conservative bound) against this host's
  // libm hypot over the whole double range, deterministic pseudo-random pairs
  long hyp_n = 0, hyp_bad = 0;
  unsigned long long st = 0x9e3779b97f4a7c15ull;
  auto next = [&st] {
    unsigned long long z = (st += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  for (int q = 0; q < 400000; ++q) {
    const double a = (double)(next() >> 11) * 0x1p-53, bb = (double)(next() >> 11) * 0x1p-53;
    const int e1 = (int)(next() % 2000) - 1000, e2 = e1 + (int)(next() % 200) - 100;
    double x = std::ldexp(a, e1), y = std::ldexp(bb, e2 < -1074 ? -1074 : (e2 > 1000 ? 1000 : e2));
    if (next() & 1) x = -x;
    if (q % 3 == 0) x = a * 4000.0, y = bb * 4000.0;  // the jet's momentum range
    const double want = std::hypot(x, y), got = hypot_ref(x, y);
    ++hyp_n;
    hyp_bad += !same(want, got);
  }
  // vertex_floors_quadform against the exact vertex checks on synthetic cells
  // built to sit ON the pressure floor: a jet-core state (kinetic energy up to
  // 1e8 x pressure), corrections of relative size 1e-1 .. 1e-12, the energy
  // tuned so that one vertex pressure lands within ~1e-17 .. 1e-9 (relative to
  // its kinetic energy) of the floor, either side (for every second cell it
  // is the smallest of the 15); plus zero / negative
  // densities and non-finite components.  Both decided answers must be right.
  long fz_n = 0, fz_pass = 0, fz_fail = 0, fz_open = 0, fz_bad = 0;
  {
    auto uni = [&] { return (double)(next() >> 11) * 0x1p-53; };
    for (int q = 0; q < 600000; ++q) {
      const double rho = std::ldexp(0.5 + uni(), (int)(next() % 5) - 2);
      const double vel = std::ldexp(1.0 + uni(), (int)(next() % 12));  // up to ~4000
      const double ang = 6.283185307179586 * uni();
      const double pr = std::ldexp(0.3 + uni(), (int)(next() % 6) - 3);
      cs fo = {rho, rho * vel * std::cos(ang), rho * vel * std::sin(ang),
               pr / gm1 + 0.5 * rho * vel * vel};
      cs cf[4];
      const double rel = std::ldexp(1.0, -(int)(next() % 40) - 3);
      for (int f = 0; f < 4; ++f)
        cf[f] = {fo.r * rel * (2 * uni() - 1), fo.mx * rel * (2 * uni() - 1) + rel * (uni() - 0.5),
                 fo.my * rel * (2 * uni() - 1) + rel * (uni() - 0.5), fo.e * rel * (2 * uni() - 1)};
      RlmpBounds b = {0, 0, 0, 0, 1e-12 * (0.5 + uni()), 1e-12 * (0.5 + uni())};
      if (q % 7 == 0) b.p_floor = 0.0;
      // move the energy so that vertex S's pressure is the floor + eps * K
      const int S = 1 + (int)(next() % 15);
      cs v = vertex_at(fo, cf, S);
      const double K = 0.5 * (v.mx * v.mx + v.my * v.my) / v.r;
      const double eps = std::ldexp(uni() - 0.5, -(int)(next() % 28) - 28);
      fo.e += (b.p_floor / gm1 + K + eps * K) - v.e;
      if (q & 1) {  // ... or the SMALLEST vertex pressure (exercises the all-pass decision)
        double pmin = kInf, kmin = 0.0;
        for (int m = 1; m < 16; ++m) {
          const cs w = vertex_at(fo, cf, m);
          const double pw = pressure(w, gm1);
          if (pw < pmin) pmin = pw, kmin = 0.5 * (w.mx * w.mx + w.my * w.my) / w.r;
        }
        fo.e += ((b.p_floor + eps * kmin) - pmin) / gm1;
      }
      if (q % 1000 == 1) fo.r = -fo.r;
      if (q % 1000 == 2) cf[q % 4].e = __longlong_as_double(0x7ff8000000000000ll);
      if (q % 1000 == 3) cf[q % 4].mx = kInf;
      if (q % 1000 == 4) fo.r = 0.0;
      const bool ok = vertex_floors_ok(1.0, fo, cf, b, gm1);
      const int d = vertex_floors_quadform(fo, cf, b.rho_floor, b.p_floor, gm1, 1.0 / gm1);
      ++fz_n;
      fz_pass += d == 1;
      fz_fail += d == 0;
      fz_open += d < 0;
      fz_bad += (d == 1 && !ok) || (d == 0 && ok);
    }
  }
  std::printf(
      "{\"cells\": %ld, \"theta_one\": %ld, "
      "\"hard\": %ld, \"bisections\": %ld, \"replay_stopped\": %ld, \"mismatch_plain\": %ld, "
      "\"mismatch_queued\": %ld, \"mismatch_replay\": %ld, \"audit_errors\": %llu, "
      "\"margin_errors\": %ld, \"hypot_checks\": %ld, \"hypot_errors\": %ld, "
      "\"quadform_pass\": %ld, \"quadform_fail\": %ld, \"quadform_open\": %ld, "
      "\"quadform_errors\": %ld, \"fuzz_cells\": %ld, \"fuzz_pass\": %ld, \"fuzz_fail\": %ld, "
      "\"fuzz_open\": %ld, \"fuzz_errors\": %ld}\n",
      cells, at_one, hard, bisect, stopped, bad_plain, bad_queued, bad_replay,
      audit[0], margin_bad, hyp_n, hyp_bad, quad_pass, quad_fail, quad_open, quad_bad, fz_n, fz_pass,
      fz_fail, fz_open, fz_bad);
  return 0;
}
