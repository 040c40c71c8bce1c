// rlmp_replay.cuh — the limiter's 30-step bisection (solver.hpp:477-486)
// replayed from certified classifications of its constraints instead of
// evaluating feasible() at every midpoint; bit-identical result.
//
// feasible(th) is the AND of (diag density in [rho_lo, rho_hi]), (diag
// pressure >= p_lo), (diag pressure <= p_hi) and the 15 vertex floors.  Along
// the diagonal ray u(th) = u_FO + th * delta and along each vertex ray the
// EXACT pressure p = (gamma-1)(E - |m|^2 / 2 rho) is concave in th (rho > 0),
// and the pressure the reference computes at th differs from it by at most
// `err` (HardStage::err, the rigorous rounding bound of rlmp.cuh, valid on
// [0, thc] for the diagonal and every vertex).  Hence, for a constraint
// p >= c whose computed value at 0 clears c by 3 err:
//   * if the computed pressure at x clears c by 3 err, the exact pressure is
//     >= c + 2 err at 0 and x, so >= c + 2 err on [0, x] (concavity): every
//     computed check on [0, x] passes;
//   * if the computed pressure at x is below c - 3 err, the exact pressure
//     decreases through x (it is higher at 0), so by concavity it stays below
//     c - 2 err on [x, inf): every computed check there fails.
// For p <= p_hi the exact superlevel set {p >= c'} is an interval: two points
// above c + 3 err bracket a certified-false interval, and a point below
// c - 3 err on the far side of one of them certifies everything beyond it;
// near 0 a tangent bound (p lies below its tangent at 0) certifies [0, t].
// The crossing points are estimated from the quadratic that p(th) = c reduces
// to; the estimates only place the test points, the certificates are the
// exact pressure evaluations at those points.  During the replay each
// midpoint is classified by comparisons; feasible() is evaluated (exactly as
// the reference does) only for midpoints inside an uncertified band, usually
// the last few steps once the bracket is narrower than the rounding band.
#pragma once
#include "rlmp.cuh"

namespace vlbm_dev {

constexpr double kInf = __builtin_huge_val();

// Certified classification of a constraint on the bisection interval:
// passes on [0, t1] and [t2, inf), fails on [f1, f2]; unknown elsewhere.
struct RayCls {
  double t1, t2, f1, f2;
};
__device__ __forceinline__ RayCls cls_unknown() { return {-1.0, kInf, kInf, -kInf}; }

// Pressure the reference computes on the diagonal at th (feasible(), :445-447).
#ifdef VLBM_REPLAY_STATS
extern long g_replay_probes;  // host experiment hooks: pressure evaluations of the setup,
extern int g_replay_phase2;   // steps left for phase 2
#define VLBM_PROBE() (++g_replay_probes)
#else
#define VLBM_PROBE() ((void)0)
#endif
__device__ __forceinline__ double diag_p(const cs& fo, const cs& delta, double th, double gm1) {
  VLBM_PROBE();
  return pressure(add(fo, scale(th, delta)), gm1);
}
// ... and at vertex S (feasible(), :449-456).
__device__ __forceinline__ double vertex_p(const cs& fo, const cs* cf, int S, double th,
                                           double gm1) {
  VLBM_PROBE();
  const cs t[4] = {scale(th, cf[0]), scale(th, cf[1]), scale(th, cf[2]), scale(th, cf[3])};
  return pressure(vertex_at(fo, t, S), gm1);
}

// Estimated crossings th > 0 of p(u_FO + th d) = c (ascending; returns the
// count).  Uses p / (gamma-1) = A_w(u) - |m - w rho|^2 / 2 rho with w the
// velocity of u_FO, which keeps the cancellation of the jet core out of the
// coefficients:  (D + th A1)(rho0 + th d.r) - th^2 Q = 0.
__device__ __forceinline__ int crossings(const cs& fo, double p0, const cs& d, double c,
                                         double gm1, double* r, double* slope) {
  const double rinv = arcp(fo.r);
  const double wx = fo.mx * rinv, wy = fo.my * rinv;
  const double A1 = (d.e - (wx * d.mx + wy * d.my)) + 0.5 * (wx * wx + wy * wy) * d.r;
  const double qx = d.mx - wx * d.r, qy = d.my - wy * d.r;
  const double Q = 0.5 * (qx * qx + qy * qy);
  const double D = (p0 - c) * arcp(gm1);
  const double a2 = A1 * d.r - Q, a1 = D * d.r + A1 * fo.r, a0 = D * fo.r;
  double x0, x1;
  if (a2 == 0.0) {
    if (a1 == 0.0) return 0;
    x0 = x1 = -a0 * arcp(a1);
  } else {
    const double disc = a1 * a1 - 4.0 * a2 * a0;
    if (!(disc >= 0.0)) return 0;
    const double s = sqrt(disc);
    const double q = -0.5 * (a1 + (a1 < 0.0 ? -s : s));
    if (q == 0.0) return 0;
    x0 = q * arcp(a2);
    x1 = a0 * arcp(q);
    if (x1 < x0) {
      const double t = x0;
      x0 = x1;
      x1 = t;
    }
  }
  int n = 0;
  if (x0 > 0.0 && isfinite(x0)) r[n++] = x0;
  if (x1 > 0.0 && isfinite(x1) && x1 != x0) r[n++] = x1;
  // |dp/dth| at the crossings: (gamma-1) |h'(x)| / rho(x)
  for (int k = 0; k < n; ++k)
    slope[k] = gm1 * fabs(2.0 * a2 * r[k] + a1) * arcp(fabs(fo.r + r[k] * d.r));
  return n;
}

// Half-width of the test band around an estimated crossing x: the rounding
// band 5 err / |p'(x)| plus a relative floor for the estimate's own error;
// widened 16x per failed certification.
#ifndef VLBM_BAND0
#define VLBM_BAND0 1e-13
#endif
__device__ __forceinline__ double band0(double x, double thc) {
  return VLBM_BAND0 * thc + 1e-12 * x;
}

// p >= c along a ray (the diagonal p_lo check or a vertex floor).  P0: the
// computed pressure at 0 (u_FO).  PF(th): the computed pressure at th.
template <class PF>
__device__ __forceinline__ RayCls classify_ge(const cs& fo, const cs& d, double P0, double c,
                                              double err, double thc, double gm1, PF&& P) {
  RayCls k = cls_unknown();
  if (!(P0 >= c + 3.0 * err) || !isfinite(err)) return k;
  double r[2], sl[2];
  const int n = crossings(fo, P0, d, c, gm1, r, sl);
  if (n == 0 || !(r[0] < thc)) {  // no crossing before thc (estimated)
    if (P(thc) >= c + 3.0 * err) k.t1 = thc;
    return k;
  }
  const double x = r[0];
  double w = band0(x, thc) + 5.0 * err * arcp(sl[0]);
  if (!(w < thc)) return k;
  bool tdone = false, fdone = !(x + w < thc);
  for (int tr = 0; tr < 3 && !(tdone && fdone); ++tr, w *= 16.0) {
    if (!tdone) {
      const double xt = x - w;
      if (!(xt > 0.0)) {
        tdone = true;
      } else if (P(xt) >= c + 3.0 * err) {
        k.t1 = xt;
        tdone = true;
      }
    }
    if (!fdone) {
      const double xf = x + w;
      if (!(xf < thc)) {
        fdone = true;
      } else if (P(xf) < c - 3.0 * err) {
        k.f1 = xf;
        k.f2 = kInf;
        fdone = true;
      }
    }
  }
  return k;
}

// p <= c on the diagonal (the p_hi check).
__device__ __forceinline__ RayCls classify_le_diag(const cs& fo, const cs& delta, double P0,
                                                   double c, double err, double thc, double gm1) {
  RayCls k = cls_unknown();
  if (!(P0 <= c - 3.0 * err) || !isfinite(err) || !(fo.r > 0.0)) return k;
  const double u = 1.1102230246251565e-16;
  // Tangent bound: for any w, p/(gamma-1) = A_w(u) - |m - w rho|^2 / 2 rho
  // <= A_w(u), affine in th: A_w(u_FO) + th A_w(delta), and A_w(u_FO) =
  // p(u_FO)/(gamma-1) + |m_FO - w rho_FO|^2 / 2 rho_FO.
  const double rinv = arcp(fo.r);  // any w works in the identity below
  const double wx = fo.mx * rinv, wy = fo.my * rinv;
  const double ax = fabs(wx), ay = fabs(wy), kk = 0.5 * (wx * wx + wy * wy);
  const double A1 = (delta.e - (wx * delta.mx + wy * delta.my)) + kk * delta.r;
  const double eA = 8.0 * u * (((fabs(delta.e) + ax * fabs(delta.mx)) + ay * fabs(delta.my)) +
                               kk * fabs(delta.r));
  const double w0x = fabs(fo.mx - wx * fo.r) + 3.0 * u * (fabs(fo.mx) + ax * fo.r);
  const double w0y = fabs(fo.my - wy * fo.r) + 3.0 * u * (fabs(fo.my) + ay * fo.r);
  const double lift = 1.01 * gm1 * (w0x * w0x + w0y * w0y) * arcp(2.0 * fo.r);
  const double base = (P0 + 2.01 * err) + lift;
  const double m = (c - base) - 4.0 * u * (fabs(c) + fabs(base));
  if (m > 0.0) {
    const double s = 1.01 * gm1 * (A1 + eA);
    k.t1 = s <= 0.0 ? thc : 0.999999 * (m * arcp(s));
    if (!(k.t1 >= 0.0)) k.t1 = -1.0;
    if (k.t1 >= thc) return k;
  }
  double r[2], sl[2];
  const int n = crossings(fo, P0, delta, c, gm1, r, sl);
  if (n == 0 || !(r[0] < thc)) return k;
  const double x1 = r[0], x2 = n > 1 ? r[1] : kInf;
  const double w = band0(x1, thc) + 5.0 * err * arcp(n > 1 ? smin(sl[0], sl[1]) : sl[0]);
  if (!(w < thc)) return k;
  const double y1 = x1 + w, y2 = smin(x2 - w, thc);
  if (!(y1 <= y2)) return k;
  auto P = [&](double th) { return diag_p(fo, delta, th, gm1); };
  if (!(P(y1) > c + 3.0 * err) || !(y2 == y1 || P(y2) > c + 3.0 * err)) return k;
  k.f1 = y1;
  k.f2 = y2;
  const double xa = x1 - w;
  if (xa > 0.0 && xa > k.t1 && P(xa) < c - 3.0 * err) k.t1 = xa;
  const double xb = x2 + w;
  if (xb < thc && P(xb) < c - 3.0 * err) k.t2 = xb;
  return k;
}

// feasible(th) given that the vertices outside `unc` pass on [0, thc].
__device__ __forceinline__ bool feasible_unc(double th, const cs& fo, const cs& delta,
                                             const cs* cf, const RlmpBounds& b, unsigned unc,
                                             double gm1) {
  if (!diag_ok(th, fo, delta, b, gm1)) return false;
  if (!unc) return true;
  const cs t[4] = {scale(th, cf[0]), scale(th, cf[1]), scale(th, cf[2]), scale(th, cf[3])};
  for (unsigned m = unc; m; m &= m - 1u) {
    const cs v = vertex_at(fo, t, __ffs(m) - 1);
    if (!(v.r >= b.rho_floor) || !(pressure(v, gm1) >= b.p_floor)) return false;
  }
  return true;
}

// The bisection of rlmp_theta (solver.hpp:477-486) for a cell whose stage
// (rlmp_hard_stage) left it undecided, replayed from classifications.
// `unc`: the vertices without a floor certificate on [0, thc].
// Bracket of a bisection in progress: [lo, hi] after `it` steps.
struct Bracket {
  double lo, hi;
  int it;
};

// Runs the bisection; returns false (bracket in `br`) when more than
// `max_exact` steps would need exact evaluations (the caller hands the cell to
// bisect_finish), else true with the result in br.lo.
__device__ __forceinline__ bool bisect_replay(const cs& fo, const cs* cf, const cs& delta,
                                              const RlmpBounds& b, const HardStage& h, double gm1,
                                              int max_exact, Bracket& br, AuditCtr* audit = nullptr,
                                              int* evals = nullptr) {
  const double thc = h.thc, err = h.err, P0 = h.p0;
  // the concavity arguments need rho > 0 along the diagonal on [0, thc]
  const bool rho_pos = fo.r > 4.0 * h.er && fo.r + thc * delta.r > 4.0 * h.er;
  RayCls klo = cls_unknown(), khi = cls_unknown();
  double vt = h.unc ? -1.0 : kInf, vf = kInf;  // vertices: all pass on [0, vt], one fails on [vf, inf)
  unsigned rho_unc = 0u;  // uncertified vertices whose density floor is not certified on [0, thc]
  if (h.certifiable && rho_pos) {
    klo = classify_ge(fo, delta, P0, b.p_lo, err, thc, gm1,
                      [&](double th) { return diag_p(fo, delta, th, gm1); });
    khi = classify_le_diag(fo, delta, P0, b.p_hi, err, thc, gm1);
    if (h.unc && h.lo_all) {
      const cs t[4] = {scale(thc, cf[0]), scale(thc, cf[1]), scale(thc, cf[2]), scale(thc, cf[3])};
      vt = kInf;
      for (unsigned m = h.unc; m; m &= m - 1u) {
        const int S = __ffs(m) - 1;
        if (!(smin(fo.r, vertex_r_at(fo.r, t, S)) - 4.0 * h.er >= b.rho_floor)) rho_unc |= 1u << S;
        cs d = {0.0, 0.0, 0.0, 0.0};
        for (int f = 0; f < 4; ++f)
          if (S >> f & 1) d = add(d, cf[f]);
        const RayCls kv = classify_ge(fo, d, P0, b.p_floor, err, thc, gm1,
                                      [&](double th) { return vertex_p(fo, cf, S, th, gm1); });
        vt = smin(vt, kv.t1);
        vf = smin(vf, kv.f1);
      }
      if (rho_unc) vt = -1.0;
    }
  }
  // Status of a midpoint from the classifications: 0 fails, 1 passes, else a
  // mask of the parts still to evaluate (2: diagonal pressure, 4: vertices).
  auto status = [&](double mid) {
    const double ur = fo.r + mid * delta.r;  // the diagonal density, computed exactly
    if (!(ur >= b.rho_lo) || !(ur <= b.rho_hi)) return 0;
    if (mid >= klo.f1 || (mid >= khi.f1 && mid <= khi.f2) || mid >= vf) return 0;
    const bool dk = mid <= klo.t1 && (mid <= khi.t1 || mid >= khi.t2);
    const bool vk = mid <= vt;
    return (dk && vk) ? 1 : (dk ? 0 : 2) | (vk ? 0 : 4);
  };
  double lo = 0.0, hi = thc;
  int it = 0;
  // Phase 1: classified midpoints only (comparisons; every lane runs the same
  // code) up to the first midpoint inside an uncertified band.
  for (; it < 30; ++it) {
    const double mid = 0.5 * (lo + hi);
    const int st = status(mid);
    if (st > 1) break;
    if (audit && (st == 1) != feasible(mid, fo, delta, cf, b, gm1)) atomicAdd(audit, 1ull);
    if (st)
      lo = mid;
    else
      hi = mid;
  }
  // Phase 2: the remaining steps (usually none to two), the uncertified parts
  // of feasible() evaluated exactly as the reference does.
#ifdef VLBM_REPLAY_STATS
  g_replay_phase2 = 30 - it;
#endif
  if (30 - it > max_exact) {
    br = {lo, hi, it};
    return false;
  }
  for (; it < 30; ++it) {
    const double mid = 0.5 * (lo + hi);
    const int st = status(mid);
    bool ok = st == 1;
    if (st > 1) {
      if (evals) ++*evals;
      ok = true;
      if (st & 2) {
        const double p = diag_p(fo, delta, mid, gm1);
        ok = (p >= b.p_lo) && (p <= b.p_hi);
      }
      if (ok && (st & 4)) {
        const cs t[4] = {scale(mid, cf[0]), scale(mid, cf[1]), scale(mid, cf[2]),
                         scale(mid, cf[3])};
        for (unsigned m = h.unc; m; m &= m - 1u) {
          const cs v = vertex_at(fo, t, __ffs(m) - 1);
          if (!(v.r >= b.rho_floor) || !(pressure(v, gm1) >= b.p_floor)) {
            ok = false;
            break;
          }
        }
      }
    }
    if (audit && ok != feasible(mid, fo, delta, cf, b, gm1)) atomicAdd(audit, 1ull);
    if (ok)
      lo = mid;
    else
      hi = mid;
  }
  br = {lo, hi, 30};
  return true;
}

// The remaining steps of a bisection stopped by bisect_replay, evaluated
// exactly (the vertices outside `unc` pass on [0, thc]).
__device__ __forceinline__ double bisect_finish(const cs& fo, const cs* cf, const cs& delta,
                                                const RlmpBounds& b, unsigned unc, Bracket br,
                                                double gm1, AuditCtr* audit = nullptr) {
  for (int it = br.it; it < 30; ++it) {
    const double mid = 0.5 * (br.lo + br.hi);
    const bool ok = feasible_unc(mid, fo, delta, cf, b, unc, gm1);
    if (audit && ok != feasible(mid, fo, delta, cf, b, gm1)) atomicAdd(audit, 1ull);
    if (ok)
      br.lo = mid;
    else
      br.hi = mid;
  }
  return br.lo;
}

// The whole of rlmp_theta after a failed feasible(1.0), in one thread, with
// the replayed bisection.
__device__ __forceinline__ double rlmp_theta_hard_replay(const cs& fo, const cs* cf,
                                                         const RlmpBounds& b, double gm1,
                                                         AuditCtr* audit = nullptr) {
  const cs delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
  if (!(finite4(fo) && finite4(cf[0]) && finite4(cf[1]) && finite4(cf[2]) && finite4(cf[3]) &&
        finite4(delta)))
    return rlmp_theta_hard_plain(fo, cf, b, gm1);  // never seen on a running sample
  const HardStage h = rlmp_hard_stage(fo, cf, delta, b, gm1);
  if (h.done) return h.result;
  if (audit) {  // statistics: [1] bisections, [2] certified at thc, [3] uncertified
    atomicAdd(audit + 1, 1ull);
    atomicAdd(audit + (h.unc ? 3 : 2), 1ull);
  }
  Bracket br;
  bisect_replay(fo, cf, delta, b, h, gm1, 30, br, audit);
  return br.lo;
}

}  // namespace vlbm_dev
