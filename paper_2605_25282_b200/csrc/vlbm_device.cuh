// vlbm_device.cuh — fp64 device primitives of the VLBM march, bit-identical to
// the reference's host arithmetic.
//
// Bit-parity rules (SURVEY.md §7.3, §8a bit-parity notes):
//  * compiled with --fmad=false: every a*b+c below is a separate DMUL + DADD,
//    as in the reference's x86-64 build (no FMA contraction);
//  * '/' and sqrt are IEEE round-to-nearest (div.rn.f64 / sqrt.rn.f64);
//  * association order is the reference's, term by term;
//  * std::min/std::max semantics: ties (and +-0) keep the FIRST argument.
#pragma once
#include <cstdint>

namespace vlbm_dev {

// 64-bit audit counters (test hook; production-scale runs exceed 2^32 events)
using AuditCtr = unsigned long long;

struct cs {  // ConservedState, euler.hpp:16-46 (rho, mom_x, mom_y, energy)
  double r, mx, my, e;
};

__device__ __forceinline__ cs add(const cs& a, const cs& b) {
  return {a.r + b.r, a.mx + b.mx, a.my + b.my, a.e + b.e};
}
__device__ __forceinline__ cs sub(const cs& a, const cs& b) {
  return {a.r - b.r, a.mx - b.mx, a.my - b.my, a.e - b.e};
}
// operator*(double s, ConservedState a) == a *= s, euler.hpp:39-50
__device__ __forceinline__ cs scale(double s, const cs& a) {
  return {a.r * s, a.mx * s, a.my * s, a.e * s};
}
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// pressure, euler.hpp:62-65 — no clamp.
__device__ __forceinline__ double pressure(const cs& u, double gm1) {
  const double kinetic = 0.5 * (u.mx * u.mx + u.my * u.my) / u.r;
  return gm1 * (u.e - kinetic);
}

// flux_x / flux_y, euler.hpp:86-97.
__device__ __forceinline__ cs flux_x(const cs& u, double gm1) {
  const double v1 = u.mx / u.r;
  const double p = pressure(u, gm1);
  return {u.mx, u.mx * v1 + p, u.my * v1, (u.e + p) * v1};
}
__device__ __forceinline__ cs flux_y(const cs& u, double gm1) {
  const double v2 = u.my / u.r;
  const double p = pressure(u, gm1);
  return {u.my, u.mx * v2, u.my * v2 + p, (u.e + p) * v2};
}

// maxwellians, lattice.hpp:43-55, split by direction: M1/M2 need only f,
// M3/M4 only g (each M_k is computed exactly as the reference computes it).
// w = 0.25*(1-alpha) and inv2a = 0.5/a are passed in (identical values).
__device__ __forceinline__ void maxw_x(const cs& u, double w, double inv2a, double gm1, cs& m0,
                                       cs& m1) {
  const cs f = flux_x(u, gm1);
  const cs wu = scale(w, u);
  const cs fa = scale(inv2a, f);
  m0 = add(wu, fa);
  m1 = sub(wu, fa);
}
__device__ __forceinline__ void maxw_y(const cs& u, double w, double inv2a, double gm1, cs& m2,
                                       cs& m3) {
  const cs g = flux_y(u, gm1);
  const cs wu = scale(w, u);
  const cs ga = scale(inv2a, g);
  m2 = add(wu, ga);
  m3 = sub(wu, ga);
}
__device__ __forceinline__ cs maxw_k(const cs& u, int k, double w, double inv2a, double gm1) {
  cs a, b;
  if (k < 2) {
    maxw_x(u, w, inv2a, gm1, a, b);
  } else {
    maxw_y(u, w, inv2a, gm1, a, b);
  }
  return (k & 1) ? b : a;
}

// std::hypot exactly as the reference's libm (glibc 2.39, x86-64) computes
// it: sqrt(ax^2 + ay^2) corrected by the unfused step of C. F. Borges, "An
// Improved Algorithm for hypot(a,b)" (2019), with the argument scaling by
// 2^-600 / 2^600 beyond 2^511 / below 2^-511 and the ay <= ax 2^-54 shortcut.
// The device hypot() is not correctly rounded either and differs in the last
// bit for about one argument pair in six; this restatement matched the host
// libm on 600 k random pairs over the whole double range (tests/
// test_limiter_host.py checks it against libm on every build host).
__device__ __forceinline__ double hypot_corr(double ax, double ay) {
  const double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    const double d = h - ay;
    t1 = ax * (2.0 * d - ax);
    t2 = (d - 2.0 * (ax - ay)) * d;
  } else {
    const double d = h - ax;
    t1 = 2.0 * d * (ax - 2.0 * ay);
    t2 = (4.0 * d - ay) * ay + d * d;
  }
  return h - (t1 + t2) / (2.0 * h);
}
__device__ __forceinline__ double hypot_ref(double x, double y) {
  const double eps = 0x1p-54, scale = 0x1p-600;
  if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000ll);
  if (isnan(x) || isnan(y)) return x + y;
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > 0x1p511) return ay <= ax * eps ? ax + ay : hypot_corr(ax * scale, ay * scale) / scale;
  if (ay < 0x1p-511) return ax >= ay / eps ? ax + ay : hypot_corr(ax / scale, ay / scale) * scale;
  if (ay <= ax * eps) return ax + ay;
  return hypot_corr(ax, ay);
}

// signal_speed, solver.hpp:203-209.  Returns NaN for rho<=0 or p<=0.
__device__ __forceinline__ double signal_speed(const cs& u, double gamma, double gm1,
                                               int conservative) {
  const double p = pressure(u, gm1);
  if (!(u.r > 0.0) || !(p > 0.0)) return __longlong_as_double(0x7ff8000000000000ll);
  const double c = sqrt(gamma * p / u.r);
  if (conservative) return hypot_ref(u.mx, u.my) / u.r + c;
  return smax(fabs(u.mx), fabs(u.my)) / u.r + c;
}

__device__ __forceinline__ bool finite4(const cs& u) {
  return isfinite(u.r) && isfinite(u.mx) && isfinite(u.my) && isfinite(u.e);
}

}  // namespace vlbm_dev
