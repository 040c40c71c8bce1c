// march_tiled.cu — the production march kernels for sm_100a.
//
// A CTA owns a TX x TY tile of interior cells of one sample (blockIdx.y), one
// thread per cell.  Every global value the tile needs is fetched ONCE into
// shared memory with cp.async (LDGSTS, all loads of the tile in flight at
// once): the macroscopic state on the tile + halo (2 for the limiter, 1 for
// the advance) and the four streamed populations on the tile + the one-cell
// ring each of them is pulled from.  Boundary tiles synthesise the ghost ring
// while staging (fill_ghosts semantics, march_common.cuh).  From the staged u
// each halo cell's inv2a*f(u), inv2a*g(u) and p(u) are formed once, so every
// flux / pressure division is evaluated once per cell; M_k(u) is rebuilt from
// them exactly as maxwellians() forms it (w*u +/- inv2a*f, lattice.hpp:43-55),
// hence bit-identical to the reference.
//
//   k_theta_tiled   u_FO, rlmp_bounds, feasible(1) per cell; cells that fail
//                   it (the limiter's hard cells) are appended to a global
//                   queue (warp-aggregated slots, one atomic per CTA)
//   k_theta_hard    the rest of rlmp_theta for the queued cells at full
//                   occupancy (solver.hpp:462-486)
//   k_advance_tiled blended pull stream-collide (solver.hpp:536-575) + the
//                   per-sample kinetic-speed / finiteness epilogue
#include <cuda_runtime.h>

#include "internal.h"
#include "march.cuh"
#include "march_common.cuh"
#include "rlmp.cuh"

namespace vlbm_dev {
namespace tiled {
constexpr int TX = 32, TY = 8, NT = TX * TY;
// population staging: P0 on x in [-1,TX), P1 on x in [0,TX], P2 on y in
// [-1,TY), P3 on y in [0,TY]  (the pull sources of the tile, plus the tile)
constexpr int NPX = (TX + 1) * TY;      // 264
constexpr int NPY = TX * (TY + 1);      // 288
constexpr int NPC = 2 * NPX + 2 * NPY;  // per component
constexpr int NPOP = 4 * NPC;           // 4416 doubles
constexpr int RX2 = TX + 4, RY2 = TY + 4, NR2 = RX2 * RY2;  // limiter region (halo 2)
constexpr int FX = TX + 2, FY = TY + 2, NF = FX * FY;       // u_FO region (ring 1)
constexpr int RX1 = TX + 2, RY1 = TY + 2, NR1 = RX1 * RY1;  // advance region (halo 1)
constexpr int kStagedTheta = 13;  // u(4), inv2a*f(4), inv2a*g(4), p
constexpr int kStagedAdv = 12;    // u(4), inv2a*f(4), inv2a*g(4)
constexpr size_t kThetaSmem = sizeof(double) * (kStagedTheta * NR2 + 2 * NF + NPOP);
constexpr size_t kAdvanceSmem = sizeof(double) * (kStagedAdv * NR1 + NPOP);
}  // namespace tiled

__device__ __forceinline__ void cp_async8(double* dst_smem, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}
__device__ __forceinline__ double comp(const cs& v, int c) {
  return c == 0 ? v.r : (c == 1 ? v.mx : (c == 2 ? v.my : v.e));
}

// Stage component c of u at padded (gi, gj) into *dst.
__device__ __forceinline__ void stage_u_elem(const MarchParams& P, const double* src,
                                             const double* rows, int gi, int gj, int c,
                                             double* dst, bool interior) {
  if (interior) {
    cp_async8(dst, src + c * P.plane + (long long)gj * P.pitch + gi);
    return;
  }
  const Src r = resolve(P, clampi(gi, -2, P.nx + 1), clampi(gj, -2, P.ny + 1));
  const bool neg = r.mirror && c == 2;
  if (r.inlet) {
    const double v = rows[4 * r.j + c];
    *dst = neg ? -v : v;
    return;
  }
  const double* g = src + c * P.plane + (long long)r.j * P.pitch + r.i;
  if (neg)
    *dst = -*g;
  else
    cp_async8(dst, g);
}

// Stage u on the tile + halo H: R[c * NR + q], q = (y + H) * RX + (x + H).
template <int H>
__device__ __forceinline__ void issue_u(const MarchParams& P, const double* src,
                                        const double* rows, int x0, int y0, double* R) {
  using namespace tiled;
  constexpr int RX = TX + 2 * H, NR = RX * (TY + 2 * H);
  const bool interior = x0 >= H && x0 + TX + H <= P.nx && y0 >= H && y0 + TY + H <= P.ny;
  for (int e = threadIdx.x; e < 4 * NR; e += NT) {
    const int c = e / NR, q = e - c * NR;
    stage_u_elem(P, src, rows, x0 + q % RX - H, y0 + q / RX - H, c, R + e, interior);
  }
}

// Stage the populations (layout of tiled::NPOP; element e decodes to k, c, x, y).
__device__ __forceinline__ void issue_pops(const MarchParams& P, const double* src,
                                           const double* rows, int x0, int y0, double inv2a,
                                           double* SP) {
  using namespace tiled;
  const bool interior = x0 >= 1 && x0 + TX + 1 <= P.nx && y0 >= 1 && y0 + TY + 1 <= P.ny;
  for (int e = threadIdx.x; e < NPOP; e += NT) {
    const int c = e / NPC;
    int r = e - c * NPC, k, x, y;
    if (r < NPX) {
      k = 0, y = r / (TX + 1), x = r - y * (TX + 1) - 1;
    } else if (r < 2 * NPX) {
      r -= NPX;
      k = 1, y = r / (TX + 1), x = r - y * (TX + 1);
    } else if (r < 2 * NPX + NPY) {
      r -= 2 * NPX;
      k = 2, y = r / TX - 1, x = r % TX;
    } else {
      r -= 2 * NPX + NPY;
      k = 3, y = r / TX, x = r % TX;
    }
    const int gi = x0 + x, gj = y0 + y;
    if (interior) {
      cp_async8(SP + e, src + (4 + 4 * k + c) * P.plane + (long long)gj * P.pitch + gi);
      continue;
    }
    const Src s = resolve(P, clampi(gi, -2, P.nx + 1), clampi(gj, -2, P.ny + 1));
    const int ks = s.mirror ? (k ^ ((k >> 1) & 1)) : k;  // {0,1,3,2} under the wall mirror
    const bool neg = s.mirror && c == 2;
    if (s.inlet) {  // inlet ghost populations: M_k(u_in, a) (solver.hpp:236-243)
      const double v = comp(maxw_k(inlet_row(rows, s.j), ks, P.w, inv2a, P.gm1), c);
      SP[e] = neg ? -v : v;
      continue;
    }
    const double* g = src + (4 + 4 * ks + c) * P.plane + (long long)s.j * P.pitch + s.i;
    if (neg)
      SP[e] = -*g;
    else
      cp_async8(SP + e, g);
  }
}

// Population k at tile-relative (x, y) from the staged layout.
__device__ __forceinline__ cs spop(const double* SP, int k, int x, int y) {
  using namespace tiled;
  int o;
  if (k == 0)
    o = y * (TX + 1) + (x + 1);
  else if (k == 1)
    o = NPX + y * (TX + 1) + x;
  else if (k == 2)
    o = 2 * NPX + (y + 1) * TX + x;
  else
    o = 2 * NPX + NPY + y * TX + x;
  return {SP[o], SP[NPC + o], SP[2 * NPC + o], SP[3 * NPC + o]};
}

// inv2a*f(u), inv2a*g(u) and (optionally) p(u) of a staged cell, in place.
// flux_x/flux_y (euler.hpp:86-97) each evaluate pressure(u): computed once.
__device__ __forceinline__ void flux_cell(double* R, int NR, int q, double inv2a, double gm1,
                                          bool with_p) {
  const cs u = {R[q], R[NR + q], R[2 * NR + q], R[3 * NR + q]};
  const double p = pressure(u, gm1);
  const double v1 = u.mx / u.r;
  const double v2 = u.my / u.r;
  R[4 * NR + q] = u.mx * inv2a;
  R[5 * NR + q] = (u.mx * v1 + p) * inv2a;
  R[6 * NR + q] = (u.my * v1) * inv2a;
  R[7 * NR + q] = ((u.e + p) * v1) * inv2a;
  R[8 * NR + q] = u.my * inv2a;
  R[9 * NR + q] = (u.mx * v2) * inv2a;
  R[10 * NR + q] = (u.my * v2 + p) * inv2a;
  R[11 * NR + q] = ((u.e + p) * v2) * inv2a;
  if (with_p) R[12 * NR + q] = p;
}

__device__ __forceinline__ cs staged_u(const double* R, int NR, int q) {
  return {R[q], R[NR + q], R[2 * NR + q], R[3 * NR + q]};
}

// M_k of a staged cell: w*u + inv2a*f (k=0), w*u - inv2a*f (1), +/- inv2a*g (2, 3).
__device__ __forceinline__ cs staged_m(const double* R, int NR, int q, int k, double w) {
  const cs wu = scale(w, staged_u(R, NR, q));
  const int b = (k < 2 ? 4 : 8) * NR;
  const cs a = {R[b + q], R[b + NR + q], R[b + 2 * NR + q], R[b + 3 * NR + q]};
  return (k & 1) ? sub(wu, a) : add(wu, a);
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(tiled::NT, 2) k_theta_tiled(MarchParams P, int tiles_x) {
  using namespace tiled;
  extern __shared__ double sm[];
  __shared__ int qn, qbase;
  const int s = blockIdx.y;
  const SampleCtl* c = P.ctl + s;
  if (!c->active) return;
  double* R = sm;                         // kStagedTheta x NR2
  double* RF = R + kStagedTheta * NR2;    // rfo[NF], pfo[NF]
  double* SP = RF + 2 * NF;               // populations
  const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * TY;
  const double* src = state_src(P, s, c->parity);
  const double* rows = P.inlet + (long long)s * P.ny * 4;
  const double inv2a = 0.5 / c->a;
  const double gm1 = P.gm1, w = P.w, al = P.alpha;
  if (threadIdx.x == 0) qn = 0;

  issue_u<2>(P, src, rows, x0, y0, R);
  cp_async_commit();
  issue_pops(P, src, rows, x0, y0, inv2a, SP);
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();
  for (int q = threadIdx.x; q < NR2; q += NT) flux_cell(R, NR2, q, inv2a, gm1, true);
  __syncthreads();

  // First-order candidates (compute_candidates, solver.hpp:301-316) on the
  // tile and its 1-ring (the ring corners are never used).
  auto rq = [](int x, int y) { return (y + 2) * RX2 + (x + 2); };
  auto fq = [](int x, int y) { return (y + 1) * FX + (x + 1); };
  auto ufo_at = [&](int x, int y) {
    const cs a = add(staged_m(R, NR2, rq(x - 1, y), 0, w), staged_m(R, NR2, rq(x + 1, y), 1, w));
    const cs b = add(staged_m(R, NR2, rq(x, y - 1), 2, w), staged_m(R, NR2, rq(x, y + 1), 3, w));
    return add(add(a, b), scale(al, staged_u(R, NR2, rq(x, y))));
  };
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const cs foC = ufo_at(tx, ty);
  RF[fq(tx, ty)] = foC.r;
  RF[NF + fq(tx, ty)] = pressure(foC, gm1);
  if (threadIdx.x < 2 * TX + 2 * TY) {
    const int t = threadIdx.x;
    int x, y;
    if (t < TX) {
      x = t, y = -1;
    } else if (t < 2 * TX) {
      x = t - TX, y = TY;
    } else if (t < 2 * TX + TY) {
      x = -1, y = t - 2 * TX;
    } else {
      x = TX, y = t - 2 * TX - TY;
    }
    const cs fo = ufo_at(x, y);
    RF[fq(x, y)] = fo.r;
    RF[NF + fq(x, y)] = pressure(fo, gm1);
  }
  cp_async_wait<0>();
  __syncthreads();

  // Limiter inputs of this thread's cell (face_corrections :321-329,
  // rlmp_bounds :364-435) and the theta = 1 test.
  const int i = x0 + tx, j = y0 + ty;
  const bool valid = i < P.nx && j < P.ny;
  cs cf[4];
  RlmpBounds b;
  bool hard = false;
  if (valid) {
    const int qc = rq(tx, ty);
    cf[0] = sub(sub(staged_m(R, NR2, rq(tx - 1, ty), 0, w), spop(SP, 0, tx - 1, ty)),
                sub(staged_m(R, NR2, qc, 1, w), spop(SP, 1, tx, ty)));
    cf[1] = sub(sub(staged_m(R, NR2, rq(tx + 1, ty), 1, w), spop(SP, 1, tx + 1, ty)),
                sub(staged_m(R, NR2, qc, 0, w), spop(SP, 0, tx, ty)));
    cf[2] = sub(sub(staged_m(R, NR2, rq(tx, ty - 1), 2, w), spop(SP, 2, tx, ty - 1)),
                sub(staged_m(R, NR2, qc, 3, w), spop(SP, 3, tx, ty)));
    cf[3] = sub(sub(staged_m(R, NR2, rq(tx, ty + 1), 3, w), spop(SP, 3, tx, ty + 1)),
                sub(staged_m(R, NR2, qc, 2, w), spop(SP, 2, tx, ty)));
    RlmpStencil st;
    st.fo = foC;
    const int fpts[5] = {fq(tx, ty), fq(tx - 1, ty), fq(tx + 1, ty), fq(tx, ty - 1), fq(tx, ty + 1)};
#pragma unroll
    for (int n = 0; n < 5; ++n) {
      st.rfo[n] = RF[fpts[n]];
      st.pfo[n] = RF[NF + fpts[n]];
    }
    const int rpts[9] = {rq(tx, ty),     rq(tx - 1, ty), rq(tx + 1, ty), rq(tx, ty - 1), rq(tx, ty + 1),
                         rq(tx - 2, ty), rq(tx + 2, ty), rq(tx, ty - 2), rq(tx, ty + 2)};
#pragma unroll
    for (int n = 0; n < 9; ++n) {
      st.rprev[n] = R[rpts[n]];
      st.pprev[n] = R[12 * NR2 + rpts[n]];
    }
    b = rlmp_bounds(st, P.kappa, P.rho_floor_coef, P.p_floor_coef);
    const cs delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
    if (feasible(1.0, foC, delta, cf, b, gm1))
      P.theta[(long long)s * P.plane + (long long)j * P.pitch + i] = 1.0;
    else
      hard = true;
  }
  // Hard cells: warp-aggregated slots in this CTA, one global atomic per CTA.
  const unsigned lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, hard);
  int slot = 0;
  if (m) {
    const int leader = __ffs(m) - 1;
    int wb = 0;
    if ((int)lane == leader) wb = atomicAdd(&qn, __popc(m));
    wb = __shfl_sync(0xffffffffu, wb, leader);
    slot = wb + __popc(m & ((1u << lane) - 1u));
  }
  __syncthreads();
  if (threadIdx.x == 0) qbase = (qn && P.hq) ? atomicAdd(P.hq_n, qn) : 0;
  __syncthreads();
  if (!hard) return;
  const long long cell = (long long)s * P.plane + (long long)j * P.pitch + i;
  if (P.hq && qbase + qn <= P.hq_cap) {
    const long long cap = P.hq_cap;
    double* q = P.hq + qbase + slot;
    q[0] = foC.r;
    q[cap] = foC.mx;
    q[2 * cap] = foC.my;
    q[3 * cap] = foC.e;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      q[(4 + 4 * f) * cap] = cf[f].r;
      q[(5 + 4 * f) * cap] = cf[f].mx;
      q[(6 + 4 * f) * cap] = cf[f].my;
      q[(7 + 4 * f) * cap] = cf[f].e;
    }
    q[20 * cap] = b.rho_lo;
    q[21 * cap] = b.rho_hi;
    q[22 * cap] = b.p_lo;
    q[23 * cap] = b.p_hi;
    P.hq_idx[qbase + slot] = cell;
  } else {  // queue full (or absent): finish in place
    if (P.hq && qbase + slot < P.hq_cap) P.hq_idx[qbase + slot] = -1;
    P.theta[cell] = rlmp_theta_hard(foC, cf, b, gm1, P.audit);
  }
}

// The limiter's hard cells, in three convergent passes (the rest of
// rlmp_theta after a failed feasible(1.0), solver.hpp:462-486; the certified
// bisection is documented in rlmp.cuh):
//   k_theta_hard    feasible(0), the closed-form cap, feasible(thc) and the
//                   vertex certificates; cells that must bisect go to bq (all
//                   vertices certified) or cq (some not)
//   k_bisect_cert   30 diagonal-only steps: every lane runs the same code
//   k_bisect_unc    30 steps re-checking the uncertified vertices
// Queues use block-aggregated slots (one global atomic per CTA pass); a CTA
// that would overflow a queue finishes those cells in place.
__device__ __forceinline__ void load_hard_entry(const MarchParams& P, int slot, cs& fo, cs* cf,
                                                RlmpBounds& b) {
  const long long cap = P.hq_cap;
  const double* q = P.hq + slot;
  fo = {q[0], q[cap], q[2 * cap], q[3 * cap]};
#pragma unroll
  for (int f = 0; f < 4; ++f)
    cf[f] = {q[(4 + 4 * f) * cap], q[(5 + 4 * f) * cap], q[(6 + 4 * f) * cap],
             q[(7 + 4 * f) * cap]};
  b.rho_lo = q[20 * cap];
  b.rho_hi = q[21 * cap];
  b.p_lo = q[22 * cap];
  b.p_hi = q[23 * cap];
  b.rho_floor = P.rho_floor_coef;
  b.p_floor = P.p_floor_coef;
}

constexpr long long kIdxMask = (1ll << 40) - 1;

__global__ void __launch_bounds__(256, 2) k_theta_hard(MarchParams P) {
  __shared__ int nb, nc, baseb, basec;
  const int n = min(P.hq_n[0], P.hq_cap);
  const long long cap = P.hq_cap;
  const double gm1 = P.gm1;
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const int slot = base + threadIdx.x;
    int cls = 0;  // 0: finished here, 1: -> bq, 2: -> cq
    long long idx = -1;
    cs fo, cf[4], delta;
    RlmpBounds b;
    HardStage h;
    if (slot < n) idx = P.hq_idx[slot];
    if (idx >= 0) {
      load_hard_entry(P, slot, fo, cf, b);
      delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
      if (!(finite4(fo) && finite4(cf[0]) && finite4(cf[1]) && finite4(cf[2]) && finite4(cf[3]) &&
            finite4(delta))) {
        P.theta[idx] = rlmp_theta_hard_plain(fo, cf, b, gm1);  // never seen on a running sample
      } else {
        h = rlmp_hard_stage(fo, cf, delta, b, gm1);
        if (h.done) {
          P.theta[idx] = h.result;
        } else {
          cls = (h.unc || P.audit) ? 2 : 1;
          if (P.audit) {
            atomicAdd(P.audit + 1, 1);
            atomicAdd(P.audit + (h.unc ? 3 : 2), 1);
          }
        }
      }
    }
    if (threadIdx.x == 0) nb = nc = 0;
    __syncthreads();
    int my = 0;
    if (cls == 1) my = atomicAdd(&nb, 1);
    if (cls == 2) my = atomicAdd(&nc, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      baseb = nb ? atomicAdd(P.hq_n + 2, nb) : 0;
      basec = nc ? atomicAdd(P.hq_n + 3, nc) : 0;
    }
    __syncthreads();
    if (cls == 1) {
      const int s = baseb + my;
      if (baseb + nb <= P.hq_cap) {
        double* q = P.bq + s;
        q[0] = fo.r, q[cap] = fo.mx, q[2 * cap] = fo.my, q[3 * cap] = fo.e;
        q[4 * cap] = delta.r, q[5 * cap] = delta.mx, q[6 * cap] = delta.my, q[7 * cap] = delta.e;
        q[8 * cap] = b.rho_lo, q[9 * cap] = b.rho_hi, q[10 * cap] = b.p_lo, q[11 * cap] = b.p_hi;
        q[12 * cap] = h.thc;
        P.bq_idx[s] = idx;
      } else {
        if (s < P.hq_cap) P.bq_idx[s] = -1;
        P.theta[idx] = bisect_certified(fo, delta, b, h.thc, gm1);
      }
    } else if (cls == 2) {
      const int s = basec + my;
      if (basec + nc <= P.hq_cap) {
        double* q = P.cq + s;
        q[0] = fo.r, q[cap] = fo.mx, q[2 * cap] = fo.my, q[3 * cap] = fo.e;
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          q[(4 + 4 * f) * cap] = cf[f].r;
          q[(5 + 4 * f) * cap] = cf[f].mx;
          q[(6 + 4 * f) * cap] = cf[f].my;
          q[(7 + 4 * f) * cap] = cf[f].e;
        }
        q[20 * cap] = b.rho_lo, q[21 * cap] = b.rho_hi, q[22 * cap] = b.p_lo, q[23 * cap] = b.p_hi;
        q[24 * cap] = h.thc, q[25 * cap] = h.p0;
        q[26 * cap] = h.certifiable ? h.err : -1.0;
        q[27 * cap] = h.er;
        P.cq_idx[s] = idx | ((long long)h.unc << 40);
      } else {
        if (s < P.hq_cap) P.cq_idx[s] = -1;
        P.theta[idx] = bisect_uncertified(fo, cf, delta, b, h, gm1, P.audit);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_bisect_cert(MarchParams P) {
  const int n = min(P.hq_n[2], P.hq_cap);
  const long long cap = P.hq_cap;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const long long idx = P.bq_idx[s];
    if (idx < 0) continue;
    const double* q = P.bq + s;
    const cs fo = {q[0], q[cap], q[2 * cap], q[3 * cap]};
    const cs delta = {q[4 * cap], q[5 * cap], q[6 * cap], q[7 * cap]};
    RlmpBounds b;
    b.rho_lo = q[8 * cap], b.rho_hi = q[9 * cap], b.p_lo = q[10 * cap], b.p_hi = q[11 * cap];
    b.rho_floor = P.rho_floor_coef;
    b.p_floor = P.p_floor_coef;
    P.theta[idx] = bisect_certified(fo, delta, b, q[12 * cap], P.gm1);
  }
}

__global__ void __launch_bounds__(256, 2) k_bisect_unc(MarchParams P) {
  const int n = min(P.hq_n[3], P.hq_cap);
  const long long cap = P.hq_cap;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const long long packed = P.cq_idx[s];
    if (packed < 0) continue;
    const double* q = P.cq + s;
    const cs fo = {q[0], q[cap], q[2 * cap], q[3 * cap]};
    cs cf[4];
#pragma unroll
    for (int f = 0; f < 4; ++f)
      cf[f] = {q[(4 + 4 * f) * cap], q[(5 + 4 * f) * cap], q[(6 + 4 * f) * cap],
               q[(7 + 4 * f) * cap]};
    RlmpBounds b;
    b.rho_lo = q[20 * cap], b.rho_hi = q[21 * cap], b.p_lo = q[22 * cap], b.p_hi = q[23 * cap];
    b.rho_floor = P.rho_floor_coef;
    b.p_floor = P.p_floor_coef;
    HardStage h;
    h.done = false;
    h.thc = q[24 * cap];
    h.p0 = q[25 * cap];
    h.err = q[26 * cap];
    h.certifiable = h.err >= 0.0;
    h.er = q[27 * cap];
    h.unc = (unsigned)(packed >> 40);
    const cs delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
    P.theta[packed & kIdxMask] = bisect_uncertified(fo, cf, delta, b, h, P.gm1, P.audit);
  }
}

// ---------------------------------------------------------------------------
template <int kMode>
__global__ void __launch_bounds__(tiled::NT, 3) k_advance_tiled(MarchParams P, double const_theta,
                                                                int tiles_x) {
  using namespace tiled;
  extern __shared__ double sm[];
  const int s = blockIdx.y;
  SampleCtl* c = P.ctl + s;
  if (!c->active) return;
  double* R = sm;                     // kStagedAdv x NR1
  double* SP = R + kStagedAdv * NR1;  // populations
  const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * TY;
  const double* src = state_src(P, s, c->parity);
  double* dst = state_dst(P, s, c->parity);
  const double* rows = P.inlet + (long long)s * P.ny * 4;
  const double inv2a = 0.5 / c->a;
  const double gm1 = P.gm1, w = P.w;
  issue_u<1>(P, src, rows, x0, y0, R);
  cp_async_commit();
  issue_pops(P, src, rows, x0, y0, inv2a, SP);
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();
  for (int q = threadIdx.x; q < NR1; q += NT) flux_cell(R, NR1, q, inv2a, gm1, false);
  cp_async_wait<0>();
  __syncthreads();

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int i = x0 + tx, j = y0 + ty;
  unsigned long long bits = 0;
  int bad = 0, nonfin = 0;
  if (i < P.nx && j < P.ny) {
    auto rq = [](int x, int y) { return (y + 1) * RX1 + (x + 1); };
    double tw, te, ts, tn;
    face_thetas<kMode>(P, s, i, j, const_theta, tw, te, ts, tn);
    const long long off = (long long)j * P.pitch + i;
    const int qc = rq(tx, ty);
    const cs M0W = staged_m(R, NR1, rq(tx - 1, ty), 0, w);
    const cs M1E = staged_m(R, NR1, rq(tx + 1, ty), 1, w);
    const cs M2S = staged_m(R, NR1, rq(tx, ty - 1), 2, w);
    const cs M3N = staged_m(R, NR1, rq(tx, ty + 1), 3, w);
    const cs n1 = add(M0W, scale(tw, sub(M0W, spop(SP, 0, tx - 1, ty))));
    const cs n2 = add(M1E, scale(te, sub(M1E, spop(SP, 1, tx + 1, ty))));
    const cs n3 = add(M2S, scale(ts, sub(M2S, spop(SP, 2, tx, ty - 1))));
    const cs n4 = add(M3N, scale(tn, sub(M3N, spop(SP, 3, tx, ty + 1))));
    store_plane4(dst + 4 * P.plane, P.plane, off, n1);
    store_plane4(dst + 8 * P.plane, P.plane, off, n2);
    store_plane4(dst + 12 * P.plane, P.plane, off, n3);
    store_plane4(dst + 16 * P.plane, P.plane, off, n4);
    cs un = add(add(add(n1, n2), add(n3, n4)), scale(P.alpha, staged_u(R, NR1, qc)));
    const cs out = add(add(scale(tw, sub(staged_m(R, NR1, qc, 1, w), spop(SP, 1, tx, ty))),
                           scale(te, sub(staged_m(R, NR1, qc, 0, w), spop(SP, 0, tx, ty)))),
                       add(scale(ts, sub(staged_m(R, NR1, qc, 3, w), spop(SP, 3, tx, ty))),
                           scale(tn, sub(staged_m(R, NR1, qc, 2, w), spop(SP, 2, tx, ty)))));
    un = sub(un, out);
    store_plane4(dst, P.plane, off, un);
    const double sp = signal_speed(un, P.gamma, gm1, P.conservative);
    if (!isfinite(sp))
      bad = 1;
    else
      bits = (unsigned long long)__double_as_longlong(sp);
    nonfin = !finite4(un);
  }
  reduce_signal(c, bits, bad, nonfin);
}

}  // namespace vlbm_dev

namespace vlbm_impl {
using namespace vlbm_dev;

static cudaError_t smem_attrs() {
  static const cudaError_t done = [] {
    cudaError_t e = cudaFuncSetAttribute(k_theta_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tiled::kThetaSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_advance_tiled<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)tiled::kAdvanceSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_advance_tiled<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)tiled::kAdvanceSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_advance_tiled<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)tiled::kAdvanceSmem);
    return e;
  }();
  return done;
}

static dim3 tiled_grid(const MarchParams& P, int& tiles_x) {
  tiles_x = (P.nx + tiled::TX - 1) / tiled::TX;
  const int ty = (P.ny + tiled::TY - 1) / tiled::TY;
  return dim3(tiles_x * ty, P.S);
}

cudaError_t launch_theta_tiled(const MarchParams& P, cudaStream_t st) {
  if (cudaError_t e = smem_attrs()) return e;
  int tx;
  const dim3 g = tiled_grid(P, tx);
  k_theta_tiled<<<g, tiled::NT, tiled::kThetaSmem, st>>>(P, tx);
  if (P.hq) {
    k_theta_hard<<<148 * 8, 256, 0, st>>>(P);
    k_bisect_cert<<<148 * 8, 256, 0, st>>>(P);
    k_bisect_unc<<<148 * 8, 256, 0, st>>>(P);
  }
  return cudaGetLastError();
}

cudaError_t launch_advance_tiled(const MarchParams& P, int mode, double const_theta,
                                 cudaStream_t st) {
  if (cudaError_t e = smem_attrs()) return e;
  int tx;
  const dim3 g = tiled_grid(P, tx);
  const size_t sm = tiled::kAdvanceSmem;
  if (mode == 0)
    k_advance_tiled<0><<<g, tiled::NT, sm, st>>>(P, const_theta, tx);
  else if (mode == 1)
    k_advance_tiled<1><<<g, tiled::NT, sm, st>>>(P, const_theta, tx);
  else
    k_advance_tiled<2><<<g, tiled::NT, sm, st>>>(P, const_theta, tx);
  return cudaGetLastError();
}

}  // namespace vlbm_impl
