// march_tiled.cu — the production march kernels for sm_100a.
//
// A CTA owns a TX x TY tile of interior cells of one sample (blockIdx.z), one
// thread per cell.  The tile's inputs arrive in shared memory by TMA
// (cp.async.bulk.tensor, 4-D tensor maps over [sample][plane][y][x] of each
// state buffer, completion on an mbarrier): ONE bulk copy of the 20 state
// planes on the tile + 1-ring for the advance; for the limiter, u on the tile
// + 2-ring and the 16 population planes on the tile + 1-ring.  Boundary
// tiles then overwrite the out-of-domain cells of the staged box with the
// ghost values of the reference's fill_ghosts (march_common.cuh::resolve).
// From the staged u each cell's inv2a*f(u), inv2a*g(u) and p(u) are formed
// once, so every flux / pressure division is evaluated once per cell; M_k(u)
// is rebuilt from them exactly as maxwellians() forms it (w*u +/- inv2a*f,
// lattice.hpp:43-55), hence bit-identical to the reference.
//
//   k_theta_tiled   u_FO, rlmp_bounds, feasible(1) per cell; cells that fail
//                   it (the limiter's hard cells) are appended to a global
//                   queue (warp-aggregated slots, one atomic per CTA)
//   k_theta_hard / k_bisect_cert / k_bisect_unc
//                   the rest of rlmp_theta for the queued cells
//   k_advance_tiled blended pull stream-collide (solver.hpp:536-575) + the
//                   per-sample kinetic-speed / finiteness epilogue
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "internal.h"
#include "march.cuh"
#include "march_common.cuh"
#include "rlmp.cuh"
#include "rlmp_replay.cuh"

#ifndef VLBM_THETA_GPOP
#define VLBM_THETA_GPOP 0  // 1: limiter reads populations from global (no SP stage)
#endif
#ifndef VLBM_THETA_MINB
#define VLBM_THETA_MINB 2
#endif
#ifndef VLBM_ADV_MINB
#define VLBM_ADV_MINB 4  // resident advance CTAs per SM (register budget)
#endif
namespace vlbm_dev {
namespace tiled {
constexpr int TX = 32, TY = 8, NT = TX * TY;  // advance tile
// limiter tile pass: TX x TYT cells, one warp per row
constexpr int TYT = VLBM_THETA_TY, NTT = TX * TYT;
constexpr int RX2 = TX + 4, RY2 = TYT + 4, NR2 = RX2 * RY2;  // limiter u box (halo 2): 36 x 12
constexpr int RX1 = TX + 2, RY1 = TYT + 2, NR1 = RX1 * RY1;  // halo-1 box: 34 x 10
constexpr int FX = RX1, NF = NR1;                           // u_FO ring region
constexpr int AYT = TYT + 2, NAT = (TX + 4) * AYT;          // limiter population box: 36 x 10
// TMA boxes start at an even x (16-byte aligned for 8-byte elements; an odd
// origin faults): the halo-1 boxes are loaded from x0-2, 36 wide.
constexpr int AX = TX + 4, AY = TY + 2, NA = AX * AY;        // 36 x 10
constexpr int kStagedTheta = 13;  // u(4) [TMA], inv2a*f(4), inv2a*g(4), p
// limiter smem: R [13][NR2] | RF [2][NF] | pad | SP [16][NA] (TMA, 128-B aligned)
constexpr int kThetaSP = ((kStagedTheta * NR2 + 2 * NF) + 15) / 16 * 16;
constexpr int kThetaSPn = VLBM_THETA_GPOP ? 0 : 16 * NAT;
constexpr size_t kThetaSmem = sizeof(double) * (kThetaSP + kThetaSPn);
constexpr unsigned kThetaTx = sizeof(double) * (4 * NR2 + kThetaSPn);
// advance smem: R [4][NA] (TMA: u) | F [8][NA] (inv2a f, inv2a g); the
// populations are read from global memory by their pulling thread.
constexpr int kAdvF = 4 * NA;
constexpr size_t kAdvanceSmem = sizeof(double) * (kAdvF + 8 * NA);
constexpr unsigned kAdvanceTx = sizeof(double) * 4 * NA;
}  // namespace tiled

// ---- TMA + mbarrier (PTX) -----------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count = 1) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: a waiting warp is parked by the
// hardware until the phase completes (or the hint expires) instead of
// spinning, so warps that reach the next tile early do not take issue slots
// from the warps still finishing this one.
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(0x989680)
      : "memory");
}
// 4-D tile [x, y, plane, sample] -> shared memory, OOB elements zero-filled.
__device__ __forceinline__ void tma_load_4d(double* dst, const CUtensorMap* map,
                                            unsigned long long* bar, int x, int y, int p, int s) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(p), "r"(s)
      : "memory");
}

// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}
__device__ __forceinline__ bool in_domain(const MarchParams& P, int i, int j) {
  return i >= 0 && i < P.nx && j >= 0 && j < P.ny;
}

// Overwrite the out-of-domain cells of a staged box [planes][RY][RX] whose
// cell (0, 0) is padded (bx, by) with the ghost values of fill_ghosts
// (solver.hpp:230-286): the ghost source is resolved once per cell, then
// kPops = false fills the 4 u planes, kPops = true the 16 population planes
// (population k of a wall ghost comes from k' = {0,1,3,2}[k], mom_y negated;
// an inlet ghost holds u_in(row) and M_k(u_in, a)).
template <bool kPops>
__device__ __forceinline__ void patch_box(const MarchParams& P, const double* src,
                                          const double* rows, double* box, int RX, int RY, int bx,
                                          int by, double inv2a) {
  const int n = RX * RY;
  auto put = [&](int k, int q, cs v, bool mirror) {
    if (mirror) v.my = -v.my;
    box[(4 * k) * n + q] = v.r;
    box[(4 * k + 1) * n + q] = v.mx;
    box[(4 * k + 2) * n + q] = v.my;
    box[(4 * k + 3) * n + q] = v.e;
  };
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const int gi = bx + q % RX, gj = by + q / RX;
    if (in_domain(P, gi, gj)) continue;
    const Src r = resolve(P, clampi(gi, -2, P.nx + 1), clampi(gj, -2, P.ny + 1));
    const long long off = (long long)r.j * P.pitch + r.i;
    if (!kPops) {
      put(0, q, r.inlet ? inlet_row(rows, r.j) : load_plane4(src, P.plane, off), r.mirror);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int ks = r.mirror ? (k ^ ((k >> 1) & 1)) : k;
        put(k, q,
            r.inlet ? maxw_k(inlet_row(rows, r.j), ks, P.w, inv2a, P.gm1)
                    : load_plane4(src + (4 + 4 * ks) * P.plane, P.plane, off),
            r.mirror);
      }
    }
  }
}

// inv2a*f(u), inv2a*g(u) (and p(u)) of one staged cell: u at U[c*NU + q],
// outputs at F[k*NF + q], k = 0..7 (and p at F[8*NF + q]).  flux_x/flux_y
// (euler.hpp:86-97) each evaluate pressure(u): computed once.
__device__ __forceinline__ void flux_cell(const double* U, int NU, double* F, int NFs, int q,
                                          double inv2a, double gm1, bool with_p) {
  const cs u = {U[q], U[NU + q], U[2 * NU + q], U[3 * NU + q]};
  const double p = pressure(u, gm1);
  const double v1 = u.mx / u.r;
  const double v2 = u.my / u.r;
  F[q] = u.mx * inv2a;
  F[NFs + q] = (u.mx * v1 + p) * inv2a;
  F[2 * NFs + q] = (u.my * v1) * inv2a;
  F[3 * NFs + q] = ((u.e + p) * v1) * inv2a;
  F[4 * NFs + q] = u.my * inv2a;
  F[5 * NFs + q] = (u.mx * v2) * inv2a;
  F[6 * NFs + q] = (u.my * v2 + p) * inv2a;
  F[7 * NFs + q] = ((u.e + p) * v2) * inv2a;
  if (with_p) F[8 * NFs + q] = p;
}

// The same for two staged cells at once: both cells' loads, then both cells'
// arithmetic in one block (six independent divisions in flight), then the
// stores -- the values are flux_cell's, operation by operation.
__device__ __forceinline__ void flux_cell_pair(const double* U, int NU, double* F, int NFs, int qa,
                                               int qb, double inv2a, double gm1) {
  const cs ua = {U[qa], U[NU + qa], U[2 * NU + qa], U[3 * NU + qa]};
  const cs ub = {U[qb], U[NU + qb], U[2 * NU + qb], U[3 * NU + qb]};
  const double pa = pressure(ua, gm1), pb = pressure(ub, gm1);
  const double a1 = ua.mx / ua.r, b1 = ub.mx / ub.r;
  const double a2 = ua.my / ua.r, b2 = ub.my / ub.r;
  const double fa[8] = {ua.mx * inv2a,          (ua.mx * a1 + pa) * inv2a,
                        (ua.my * a1) * inv2a,   ((ua.e + pa) * a1) * inv2a,
                        ua.my * inv2a,          (ua.mx * a2) * inv2a,
                        (ua.my * a2 + pa) * inv2a, ((ua.e + pa) * a2) * inv2a};
  const double fb[8] = {ub.mx * inv2a,          (ub.mx * b1 + pb) * inv2a,
                        (ub.my * b1) * inv2a,   ((ub.e + pb) * b1) * inv2a,
                        ub.my * inv2a,          (ub.mx * b2) * inv2a,
                        (ub.my * b2 + pb) * inv2a, ((ub.e + pb) * b2) * inv2a};
#pragma unroll
  for (int k = 0; k < 8; ++k) F[k * NFs + qa] = fa[k];
  F[8 * NFs + qa] = pa;
#pragma unroll
  for (int k = 0; k < 8; ++k) F[k * NFs + qb] = fb[k];
  F[8 * NFs + qb] = pb;
}

__device__ __forceinline__ cs plane4(const double* A, int N, int q) {
  return {A[q], A[N + q], A[2 * N + q], A[3 * N + q]};
}

// M_k of a staged cell: w*u + inv2a*f (k=0), w*u - inv2a*f (1), +/- inv2a*g (2, 3).
__device__ __forceinline__ cs staged_m(const double* U, int NU, const double* F, int NFs, int q,
                                       int k, double w) {
  const cs wu = scale(w, plane4(U, NU, q));
  const cs a = plane4(F + (k < 2 ? 0 : 4 * NFs), NFs, q);
  return (k & 1) ? sub(wu, a) : add(wu, a);
}

// Slot of this lane among the flagged lanes of its warp in a global queue:
// one atomic on `counter` per warp (by its first flagged lane); returns the
// warp's base in *wbase and its count in *wcount.  All lanes call it.
__device__ __forceinline__ int warp_slot(bool flag, int* counter, int* wbase, int* wcount) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, flag);
  int base = 0;
  if (m) {
    const int leader = __ffs(m) - 1;
    if ((int)lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
  }
  *wbase = base;
  *wcount = __popc(m);
  return base + __popc(m & ((1u << lane) - 1u));
}

// Append the warp's hard cells (flag) to the global limiter queue: warp-
// aggregated slots, one global atomic per warp with hard cells, no CTA
// barrier (warps that finish their cells early move on to the next tile).
// When the queue cannot hold the warp's cells (or is absent) they finish in
// place.  All lanes of the warp call it.
__device__ __forceinline__ void enqueue_hard(const MarchParams& P, bool hard, long long cell,
                                             const cs& fo, const cs* cf, const RlmpBounds& b,
                                             double gm1) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, hard);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if ((int)lane == leader && P.hq) base = atomicAdd(P.hq_n, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!hard) return;
  const int slot = base + __popc(m & ((1u << lane) - 1u));
  if (P.hq && base + __popc(m) <= P.hq_cap) {
    const long long cap = P.hq_cap;
    double* q = P.hq + slot;
    q[0] = fo.r;
    q[cap] = fo.mx;
    q[2 * cap] = fo.my;
    q[3 * cap] = fo.e;
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
    P.hq_idx[slot] = cell;
  } else {  // queue full (or absent): finish in place
    if (P.hq && slot < P.hq_cap) P.hq_idx[slot] = -1;
    if (P.qstats && lane == (unsigned)leader) atomicAdd(P.qstats, (unsigned long long)__popc(m));
    P.theta[cell] = rlmp_theta_hard(fo, cf, b, gm1, P.audit);  // rare: plain bisection
  }
}

// ---------------------------------------------------------------------------
// Persistent: each CTA starts at tile blockIdx.x and then claims tiles from a
// per-step counter, skipping inactive samples (t = (sample * tiles_y +
// tile_y) * tiles_x + tile_x).  A
// tile's staged data is read only until its cells hold u_FO, c_f and the
// bounds in registers; then the CTA issues the NEXT tile's TMA into the same
// buffers, so the load overlaps this tile's feasibility work.
__global__ void __launch_bounds__(tiled::NTT, VLBM_THETA_MINB)
    k_theta_tiled(MarchParams P, const __grid_constant__ CUtensorMap tmu0,
                  const __grid_constant__ CUtensorMap tmu1, const __grid_constant__ CUtensorMap tmp0,
                  const __grid_constant__ CUtensorMap tmp1) {
  using namespace tiled;
  extern __shared__ __align__(128) double sm[];
  // bar: the tile's TMA loads have landed; bar_free: every warp has taken its
  // last value from the staged tile (one arrival per warp), so thread 0 may
  // overwrite the buffers with the next tile's loads
  __shared__ __align__(8) unsigned long long bar, bar_free;
  // the CTA's current tile, written by thread 0 before it issues the tile's
  // loads (ordered before every other thread's read by the mbarrier)
  __shared__ int s_next, s_ns, s_nx0, s_ny0, s_par;
  __shared__ double s_inv2a;
  double* R = sm;                    // u [4][NR2] by TMA, then inv2a f/g, p: [9][NR2]
  double* RF = R + kStagedTheta * NR2;  // rfo[NF], pfo[NF]
  double* SP = sm + kThetaSP;        // populations [16][NAT] by TMA
  const int tiles_x = (P.nx + TX - 1) / TX, tiles_y = (P.ny + TYT - 1) / TYT;
  const int per_sample = tiles_x * tiles_y;
  const int total = P.S * per_sample;  // < 2^31 tiles (host-checked)
  const double gm1 = P.gm1, w = P.w, al = P.alpha;
  const double igm1 = 1.0 / gm1;
  auto next_active = [&](int t) {
    while (t < total && !P.ctl[t / per_sample].active) t += gridDim.x;
    return t;
  };
  // thread 0: the next tile of this CTA -- claimed from the step's tile
  // counter (hq_n[6], reset by k_sched) so CTAs stay balanced whatever the
  // per-tile cost (boundary tiles, hard cells); static striding without queues
  // The claim's atomic is issued at the top of the tile (claim_start) and its
  // result used only when the tile's staged data has been consumed
  // (claim_finish), so its round trip overlaps the tile's work.
  auto claim_start = [&](int t) {
    return P.hq_n ? (int)gridDim.x + atomicAdd(P.hq_n + 6, 1) : next_active(t + (int)gridDim.x);
  };
  auto claim_finish = [&](int tn) {
    if (P.hq_n)
      while (tn < total && !P.ctl[tn / per_sample].active)
        tn = (int)gridDim.x + atomicAdd(P.hq_n + 6, 1);
    return tn;
  };
  // thread 0: publish tile t (sample, origin, buffer parity, 0.5/a) and issue
  // its TMA loads; past the last tile a plain arrival completes the phase so
  // that the waiting threads wake up and leave
  auto publish = [&](int t) {
    s_next = t;
    if (t >= total) {
      mbar_arrive(&bar);
      return;
    }
    const int s = t / per_sample, r = t - s * per_sample;
    const int x0 = (r % tiles_x) * TX, y0 = (r / tiles_x) * TYT;
    const int parity = P.ctl[s].parity;
    s_ns = s, s_nx0 = x0, s_ny0 = y0, s_par = parity;
    s_inv2a = P.ctl[s].inv2a;
    mbar_expect_tx(&bar, kThetaTx);
    tma_load_4d(R, parity ? &tmu1 : &tmu0, &bar, x0 - 2, y0 - 2, 0, s);
    if (!VLBM_THETA_GPOP) tma_load_4d(SP, parity ? &tmp1 : &tmp0, &bar, x0 - 2, y0 - 1, 4, s);
  };
  {
    const int t0 = next_active(blockIdx.x);
    if (t0 >= total) return;
    if (threadIdx.x == 0) {
      mbar_init(&bar);
      mbar_init(&bar_free, NTT / 32);
      publish(t0);
    }
    __syncthreads();
  }
  for (unsigned it = 0;; ++it) {
    mbar_wait(&bar, it & 1u);
    const int t = s_next;
    if (t >= total) break;
    const int s = s_ns, x0 = s_nx0, y0 = s_ny0, parity = s_par;
    const double inv2a = s_inv2a;
    const double* src = state_src(P, s, parity);
    const double* rows = P.inlet + (long long)s * P.ny * 4;
    int tn_claim = 0;
    if (threadIdx.x == 0) tn_claim = claim_start(t);
    if (!(x0 >= 2 && x0 + TX + 2 <= P.nx && y0 >= 2 && y0 + TYT + 2 <= P.ny)) {
      patch_box<false>(P, src, rows, R, RX2, RY2, x0 - 2, y0 - 2, inv2a);
      if (!VLBM_THETA_GPOP) patch_box<true>(P, src, rows, SP, AX, AYT, x0 - 2, y0 - 1, inv2a);
      __syncthreads();
    }
    double* F = R + 4 * NR2;
    {
      // NR2 staged cells on NTT threads: the warps with a second cell take
      // both in one straight-line block, so the two cells' division chains
      // overlap (a warp whose second round is part-filled repeats the last
      // cell: same values to the same addresses)
      static_assert(NR2 > NTT && NR2 <= 2 * NTT, "one or two staged cells per thread");
      const int q0 = threadIdx.x;
      if ((q0 & ~31) + NTT < NR2) {
        flux_cell_pair(R, NR2, F, NR2, q0, min(q0 + NTT, NR2 - 1), inv2a, gm1);
      } else {
        flux_cell(R, NR2, F, NR2, q0, inv2a, gm1, true);
      }
    }
    __syncthreads();

    // First-order candidates (compute_candidates, solver.hpp:301-316) on the
    // tile and its 1-ring (the ring corners are never used).
    auto rq = [](int x, int y) { return (y + 2) * RX2 + (x + 2); };
    auto fq = [](int x, int y) { return (y + 1) * FX + (x + 1); };
    auto M = [&](int q, int k) { return staged_m(R, NR2, F, NR2, q, k, w); };
    auto ufo_at = [&](int x, int y) {
      const cs a = add(M(rq(x - 1, y), 0), M(rq(x + 1, y), 1));
      const cs b = add(M(rq(x, y - 1), 2), M(rq(x, y + 1), 3));
      return add(add(a, b), scale(al, plane4(R, NR2, rq(x, y))));
    };
    const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
    // This cell's four incoming Maxwellians, formed ONCE: they give both its
    // u_FO (compute_candidates) and its face corrections (face_corrections
    // :321-329), so the corrections are taken here, before the barrier.
    const int i = x0 + tx, j = y0 + ty;
    const bool valid = i < P.nx && j < P.ny;
    cs cf[4];
    cs foC;
    {
      auto pop = [&](int k, int x, int y) {
        if (VLBM_THETA_GPOP) {
          const int ii = x0 + x, jj = y0 + y;
          if (ii >= 0 && ii < P.nx && jj >= 0 && jj < P.ny)
            return load_plane4(src + (4 + 4 * k) * P.plane, P.plane, (long long)jj * P.pitch + ii);
          return load_pop(P, src, rows, k, ii, jj, inv2a);
        }
        return plane4(SP + 4 * k * NAT, NAT, (y + 1) * AX + (x + 2));
      };
      const int qc = rq(tx, ty);
      const cs mw = M(rq(tx - 1, ty), 0), me = M(rq(tx + 1, ty), 1);
      const cs ms = M(rq(tx, ty - 1), 2), mn = M(rq(tx, ty + 1), 3);
      foC = add(add(add(mw, me), add(ms, mn)), scale(al, plane4(R, NR2, qc)));
      if (valid) {
        cf[0] = sub(sub(mw, pop(0, tx - 1, ty)), sub(M(qc, 1), pop(1, tx, ty)));
        cf[1] = sub(sub(me, pop(1, tx + 1, ty)), sub(M(qc, 0), pop(0, tx, ty)));
        cf[2] = sub(sub(ms, pop(2, tx, ty - 1)), sub(M(qc, 3), pop(3, tx, ty)));
        cf[3] = sub(sub(mn, pop(3, tx, ty + 1)), sub(M(qc, 2), pop(2, tx, ty)));
      }
    }
    RF[fq(tx, ty)] = foC.r;
    RF[NF + fq(tx, ty)] = pressure(foC, gm1);
    if (threadIdx.x < 2 * TX + 2 * TYT) {
      const int q = threadIdx.x;
      int x, y;
      if (q < TX) {
        x = q, y = -1;
      } else if (q < 2 * TX) {
        x = q - TX, y = TYT;
      } else if (q < 2 * TX + TYT) {
        x = -1, y = q - 2 * TX;
      } else {
        x = TX, y = q - 2 * TX - TYT;
      }
      const cs fo = ufo_at(x, y);
      RF[fq(x, y)] = fo.r;
      RF[NF + fq(x, y)] = pressure(fo, gm1);
    }
    __syncthreads();

    // Limiter inputs of this thread's cell (rlmp_bounds :364-435): the last
    // reads of the staged tile.
    cs delta;
    RlmpBounds b;
    bool hard = false;
    if (valid) {
      RlmpStencil st;
      st.fo = foC;
      const int fpts[5] = {fq(tx, ty), fq(tx - 1, ty), fq(tx + 1, ty), fq(tx, ty - 1),
                           fq(tx, ty + 1)};
#pragma unroll
      for (int n = 0; n < 5; ++n) {
        st.rfo[n] = RF[fpts[n]];
        st.pfo[n] = RF[NF + fpts[n]];
      }
      const int rpts[9] = {rq(tx, ty),     rq(tx - 1, ty), rq(tx + 1, ty),
                           rq(tx, ty - 1), rq(tx, ty + 1), rq(tx - 2, ty),
                           rq(tx + 2, ty), rq(tx, ty - 2), rq(tx, ty + 2)};
#pragma unroll
      for (int n = 0; n < 9; ++n) {
        st.rprev[n] = R[rpts[n]];
        st.pprev[n] = F[8 * NR2 + rpts[n]];
      }
      b = rlmp_bounds(st, P.kappa, P.rho_floor_coef, P.p_floor_coef);
      delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
    }
    // This warp has taken its last value from the staged tile.  Thread 0 waits
    // for every warp's arrival (no CTA barrier: the other warps go straight on
    // to their feasibility work) and then issues the next tile's loads into
    // the same buffers, so the loads overlap this tile's feasibility work.
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&bar_free);
    if (threadIdx.x == 0) {
      const int tn = claim_finish(tn_claim);
      mbar_wait(&bar_free, it & 1u);
      publish(tn);
    }

    // feasible(1): the diagonal first; then the 15 vertex floors decided by
    // the quadratic form (rlmp.cuh::vertex_floors_quadform: no pressure
    // divisions), evaluated exactly only for the few cells it leaves open.
    unsigned aflags = 0;  // audit statistics of this cell (bits = counter indices)
    if (valid) {
      if (diag_ok(1.0, foC, delta, b, gm1)) {
        const int q = P.cert1 ? vertex_floors_quadform(foC, cf, b.rho_floor, b.p_floor, gm1, igm1)
                              : -1;
#ifdef VLBM_EXP_NOVERTEX  // timing experiment only (WRONG results): the vertex checks' share
        const bool ok = true;
#else
        const bool ok = q > 0 || (q < 0 && vertex_floors_ok(1.0, foC, cf, b, gm1));
#endif
        if (P.audit) {  // [8] diagonal passed, [9] decided by the form, [10] feasible; [0] its errors
          aflags |= 1u << 8;
          if (q >= 0) aflags |= 1u << 9;
          if (ok) aflags |= 1u << 10;
          if (q >= 0 && (q > 0) != vertex_floors_ok(1.0, foC, cf, b, gm1)) aflags |= 1u;
          if (q < 0) aflags |= 1u << 12;  // [12] left open: exact vertex checks
        }
        if (ok)
          P.theta[(long long)s * P.plane + (long long)j * P.pitch + i] = 1.0;
        else
          hard = true;
      } else {
        hard = true;
      }
    }
    if (P.audit) {  // warp-aggregated: one atomic per counter and warp
      for (int k = 0; k < 15; ++k) {
        const unsigned mk = __ballot_sync(0xffffffffu, (aflags >> k) & 1u);
        if ((threadIdx.x & 31) == 0 && mk) atomicAdd(P.audit + k, (AuditCtr)__popc(mk));
      }
    }
    const long long cell = (long long)s * P.plane + (long long)j * P.pitch + i;
    enqueue_hard(P, hard, cell, foC, cf, b, gm1);
  }
}

// The limiter's hard cells, in three convergent passes (the rest of
// rlmp_theta after a failed feasible(1.0), solver.hpp:462-486; the certified
// bisection is documented in rlmp.cuh):
//   k_theta_hard    feasible(0), the closed-form cap, feasible(thc) and the
//                   vertex certificates; cells that must bisect go to bq (all
//                   vertices certified) or cq (some not)
//   k_bisect_cert   30 diagonal-only steps: every lane runs the same code
//   k_bisect_unc    30 steps re-checking the uncertified vertices (replay on:
//                   the bisection replayed, rlmp_replay.cuh)
//   k_bisect_tail   the replayed bisections that need more exact steps
// Queues use warp-aggregated slots (one global atomic per warp and queue); a
// warp that would overflow a queue finishes those cells in place.
// Hard-queue entries staged in shared memory: kHB consecutive slots, one
// bulk copy per SoA word plane (kHardWords + the cell index).
#ifndef VLBM_HARD_THREADS
// k_theta_hard: threads per CTA = slots per staged chunk, and resident CTAs
// per SM (register budget).  128 x 3 (168 registers, no spills to speak of,
// 12 warps/SM) measured 0.905 ms for the hard path against 0.930 for 256 x 2
// (128 registers, 220 B of spills, 16 warps/SM); 128 x 4: 0.943, 512 x 1: 0.935
#define VLBM_HARD_THREADS 128
#define VLBM_HARD_MINB 3
#endif
constexpr int kHB = VLBM_HARD_THREADS;
constexpr size_t kHardSmem = sizeof(double) * kHardWords * kHB + sizeof(long long) * kHB;
__device__ __forceinline__ void load_hard_staged(const MarchParams& P, const double* H, int t,
                                                 cs& fo, cs* cf, RlmpBounds& b) {
  fo = {H[t], H[kHB + t], H[2 * kHB + t], H[3 * kHB + t]};
#pragma unroll
  for (int f = 0; f < 4; ++f)
    cf[f] = {H[(4 + 4 * f) * kHB + t], H[(5 + 4 * f) * kHB + t], H[(6 + 4 * f) * kHB + t],
             H[(7 + 4 * f) * kHB + t]};
  b.rho_lo = H[20 * kHB + t];
  b.rho_hi = H[21 * kHB + t];
  b.p_lo = H[22 * kHB + t];
  b.p_hi = H[23 * kHB + t];
  b.rho_floor = P.rho_floor_coef;
  b.p_floor = P.p_floor_coef;
}

constexpr long long kIdxMask = (1ll << 40) - 1;

// Uncertified bisections are binned by their number of uncertified vertices
// (1, 2, >= 3) into thirds of cq, so lanes of a warp run similar vertex loops.
__device__ __forceinline__ int unc_class(unsigned unc) {
  const int n = __popc(unc);
  return n <= 1 ? 0 : (n == 2 ? 1 : 2);
}

// Persistent over chunks of kHB queue slots: a chunk's entries arrive in
// shared memory by bulk copies; once every thread holds its entry in
// registers the next chunk's copies are issued into the same buffer, so
// they overlap this chunk's work.
__global__ void __launch_bounds__(kHB, VLBM_HARD_MINB) k_theta_hard(MarchParams P) {
  extern __shared__ __align__(128) double H[];  // [kHardWords][kHB] | idx[kHB]
  // bar: the chunk's bulk copies have landed; bar_free: every warp holds its
  // entries in registers (one arrival per warp), the buffer may be refilled
  __shared__ __align__(8) unsigned long long bar, bar_free;
  long long* HI = reinterpret_cast<long long*>(H + kHardWords * kHB);
  const int n = min(P.hq_n[0], P.hq_cap);
  const long long cap = P.hq_cap;
  const double gm1 = P.gm1;
  const int nchunks = (n + kHB - 1) / kHB;
  if ((int)blockIdx.x >= nchunks) return;
  auto issue = [&](int chunk) {  // thread 0
    const int s0 = chunk * kHB;
    const unsigned bytes = 8u * (unsigned)((min(kHB, n - s0) + 1) & ~1);  // even count: 16-B
    mbar_expect_tx(&bar, bytes * (kHardWords + 1));
    for (int w = 0; w < kHardWords; ++w) bulk_load(H + w * kHB, P.hq + w * cap + s0, bytes, &bar);
    bulk_load(HI, P.hq_idx + s0, bytes, &bar);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar);
    mbar_init(&bar_free, kHB / 32);
    issue(blockIdx.x);
  }
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  for (int chunk = blockIdx.x, it = 0; chunk < nchunks; chunk += gridDim.x, ++it) {
    const int slot = chunk * kHB + threadIdx.x;
    int cls = 0;  // 0: finished here, 1: -> bq, 2: -> cq
    int ccls = 0;  // cq bin
    long long idx = -1;
    cs fo, cf[4], delta;
    RlmpBounds b;
    HardStage h;
    mbar_wait(&bar, it & 1);
    if (slot < n) {
      idx = HI[threadIdx.x];
      load_hard_staged(P, H, threadIdx.x, fo, cf, b);
    }
    // the buffer is free once every warp has arrived: thread 0 alone waits for
    // that and issues the next chunk's copies; no CTA barrier in this loop, so
    // no warp waits for another warp's slower branch of the stage
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar_free);
    if (threadIdx.x == 0 && chunk + (int)gridDim.x < nchunks) {
      mbar_wait(&bar_free, it & 1);
      issue(chunk + gridDim.x);
    }
    if (idx >= 0) {
      delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
      if (!(finite4(fo) && finite4(cf[0]) && finite4(cf[1]) && finite4(cf[2]) && finite4(cf[3]) &&
            finite4(delta))) {
        P.theta[idx] = rlmp_theta_hard_plain(fo, cf, b, gm1);  // never seen on a running sample
      } else {
        h = rlmp_hard_stage(fo, cf, delta, b, gm1);
        if (P.audit && h.form >= 0) {
          // audit of the stage's quadratic-form decisions at thc: the vertex
          // floors and every margin bit against their exact evaluations
          bool bad = (h.form > 0) != vertex_floors_ok(h.thc, fo, cf, b, gm1);
          const cs t[4] = {scale(h.thc, cf[0]), scale(h.thc, cf[1]), scale(h.thc, cf[2]),
                           scale(h.thc, cf[3])};
          for (unsigned m = h.mhi; m; m &= m - 1u) {
            const cs v = vertex_at(fo, t, __ffs(m) - 1);
            const double p = pressure(v, gm1);
            bad = bad || !vertex_margin(p, p, v.r, v.r, b, h.err, h.er);
          }
          if (bad) atomicAdd(P.audit, 1ull);
          atomicAdd(P.audit + 13, 1ull);  // [13] stages decided by the form
        }
        if (h.done) {
          P.theta[idx] = h.result;
        } else {
          if (P.audit) {
            atomicAdd(P.audit + 1, 1ull);
            atomicAdd(P.audit + (h.unc ? 3 : 2), 1ull);
          }
          cls = (h.unc || P.audit) ? 2 : 1;
          ccls = unc_class(h.unc);
        }
      }
    }
    // Queue slots, warp-aggregated: queue 0 = bq, 1..3 = the cq bins; lane k
    // reserves queue k's slots for the warp (the four atomics are in flight
    // together), every lane takes its rank among the warp's entries of its queue.
    const int myq = cls == 1 ? 0 : (cls == 2 ? 1 + ccls : -1);
    unsigned qm[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) qm[k] = __ballot_sync(0xffffffffu, myq == k);
    int qbase = 0;
    if (lane < 4) {
      const unsigned m = lane == 0 ? qm[0] : (lane == 1 ? qm[1] : (lane == 2 ? qm[2] : qm[3]));
      if (m) qbase = atomicAdd(P.hq_n + 2 + lane, __popc(m));
    }
    int my = 0, nb = 0, baseb = 0;  // this lane's queue: rank, the warp's count and base
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int bk = __shfl_sync(0xffffffffu, qbase, k);
      if (myq == k) my = __popc(qm[k] & ((1u << lane) - 1u)), nb = __popc(qm[k]), baseb = bk;
    }
    const int third = P.hq_cap / 3;
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
        if (P.qstats) atomicAdd(P.qstats, 1ull);
        P.theta[idx] = bisect_certified(fo, delta, b, h.thc, gm1);
      }
    } else if (cls == 2) {
      const int s = ccls * third + baseb + my;
      if (baseb + nb <= third) {
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
        P.cq_idx[s] = idx | ((long long)h.mhi << 40) | ((long long)h.lo_all << 56);
      } else {
        if (baseb + my < third) P.cq_idx[s] = -1;
        if (P.qstats) atomicAdd(P.qstats, 1ull);
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

// One cq entry (k_theta_hard's layout) back into registers.
__device__ __forceinline__ void load_unc_entry(const MarchParams& P, int s, long long packed, cs& fo,
                                               cs* cf, RlmpBounds& b, HardStage& h) {
  const long long cap = P.hq_cap;
  const double* q = P.cq + s;
  fo = {q[0], q[cap], q[2 * cap], q[3 * cap]};
#pragma unroll
  for (int f = 0; f < 4; ++f)
    cf[f] = {q[(4 + 4 * f) * cap], q[(5 + 4 * f) * cap], q[(6 + 4 * f) * cap],
             q[(7 + 4 * f) * cap]};
  b.rho_lo = q[20 * cap], b.rho_hi = q[21 * cap], b.p_lo = q[22 * cap], b.p_hi = q[23 * cap];
  b.rho_floor = P.rho_floor_coef;
  b.p_floor = P.p_floor_coef;
  h.done = false;
  h.thc = q[24 * cap];
  h.p0 = q[25 * cap];
  h.err = q[26 * cap];
  h.certifiable = h.err >= 0.0;
  h.er = q[27 * cap];
  h.mhi = (unsigned)(packed >> 40) & kAllVertices;
  h.lo_all = ((packed >> 56) & 1) != 0;
  h.unc = kAllVertices & ~((h.lo_all ? kAllVertices : 0u) & h.mhi);
}

// Steps a replayed bisection may evaluate exactly in k_bisect_unc (1 measured
// best of 0, 1, 2, 4, 6); a cell
// that needs more (its classifications leave a wide band) continues in
// k_bisect_tail, so no warp waits on one lane's long exact tail.
#ifndef VLBM_REPLAY_INLINE
#define VLBM_REPLAY_INLINE 1
#endif
constexpr int kReplayInline = VLBM_REPLAY_INLINE;

// blockIdx.y = cq bin; bins run concurrently.
#ifndef VLBM_UNC_GRID
#define VLBM_UNC_GRID 2  // k_bisect_unc CTAs per bin = 148 x this (measured: 1, 3, 6 slower)
#endif
#ifndef VLBM_UNC_MINB
#define VLBM_UNC_MINB 2
#endif
#ifndef VLBM_UNC_THREADS
#define VLBM_UNC_THREADS 256  // threads per CTA (the grid keeps its thread count)
#endif
__global__ void __launch_bounds__(VLBM_UNC_THREADS, VLBM_UNC_MINB) k_bisect_unc(MarchParams P) {
  const int third = P.hq_cap / 3;
  const int n = min(P.hq_n[3 + blockIdx.y], third);
  const long long cap = P.hq_cap;
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const int s0 = base + threadIdx.x;
    const int s = (int)blockIdx.y * third + s0;
    const long long packed = s0 < n ? P.cq_idx[s] : -1;
    bool stopped = false;
    Bracket br;
    if (packed >= 0) {
      cs fo, cf[4];
      RlmpBounds b;
      HardStage h;
      load_unc_entry(P, s, packed, fo, cf, b, h);
      const cs delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
      if (P.replay) {
        stopped = !bisect_replay(fo, cf, delta, b, h, P.gm1, kReplayInline, br, P.audit);
        if (!stopped) P.theta[packed & kIdxMask] = br.lo;
      } else {
        P.theta[packed & kIdxMask] = bisect_uncertified(fo, cf, delta, b, h, P.gm1, P.audit);
      }
    }
    if (!P.replay) continue;
    // stopped bisections -> the tail queue.  The tail has its own tq storage:
    // k_bisect_cert may still be running on P.side, so bq must not be reused.
    int tbase, nt;
    const int t = warp_slot(stopped, P.hq_n + 7, &tbase, &nt);
    if (stopped) {
      if (tbase + nt <= P.hq_cap) {
        P.tq[t] = br.lo;
        P.tq[cap + t] = br.hi;
        P.tq_idx[t] = (long long)s | ((long long)br.it << 40);
      } else {  // tail full: finish here
        cs fo, cf[4];
        RlmpBounds b;
        HardStage h;
        load_unc_entry(P, s, packed, fo, cf, b, h);
        const cs delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
        if (t < P.hq_cap) P.tq_idx[t] = -1;
        if (P.qstats) atomicAdd(P.qstats, 1ull);
        P.theta[packed & kIdxMask] = bisect_finish(fo, cf, delta, b, h.unc, br, P.gm1, P.audit);
      }
    }
  }
}

// The bisections k_bisect_unc stopped, finished with exact evaluations.
#ifndef VLBM_TAIL_MINB
#define VLBM_TAIL_MINB 4
#endif
__global__ void __launch_bounds__(128, VLBM_TAIL_MINB) k_bisect_tail(MarchParams P) {
  const int n = min(P.hq_n[7], P.hq_cap);
  const long long cap = P.hq_cap;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const long long tp = P.tq_idx[t];
    if (tp < 0) continue;
    const int s = (int)(tp & kIdxMask);
    const long long packed = P.cq_idx[s];
    cs fo, cf[4];
    RlmpBounds b;
    HardStage h;
    load_unc_entry(P, s, packed, fo, cf, b, h);
    const cs delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
    P.theta[packed & kIdxMask] = bisect_uncertified(fo, cf, delta, b, h, P.gm1, P.audit, P.tq[t],
                                                    P.tq[cap + t], (int)(tp >> 40));
  }
}

// ---------------------------------------------------------------------------
template <int kMode>
__global__ void __launch_bounds__(tiled::NT, VLBM_ADV_MINB)
    k_advance_tiled(MarchParams P, double const_theta,
                    const __grid_constant__ CUtensorMap tma0,
                    const __grid_constant__ CUtensorMap tma1) {
  using namespace tiled;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long bar;
  const int s = blockIdx.z;
  SampleCtl* c = P.ctl + s;
  if (!c->active) return;
  double* R = sm;          // [4][NA]: u (TMA)
  double* F = sm + kAdvF;  // [8][NA]: inv2a f, inv2a g
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int parity = c->parity;
  const double* src = state_src(P, s, parity);
  double* dst = state_dst(P, s, parity);
  const double* rows = P.inlet + (long long)s * P.ny * 4;
  const double inv2a = c->inv2a;
  const double gm1 = P.gm1, w = P.w;
  if (threadIdx.x == 0) mbar_init(&bar);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, kAdvanceTx);
    tma_load_4d(R, parity ? &tma1 : &tma0, &bar, x0 - 2, y0 - 1, 0, s);
  }
  mbar_wait(&bar, 0);
  // every cell of the tile has its four neighbours inside the domain
  const bool interior = x0 >= 1 && x0 + TX + 1 <= P.nx && y0 >= 1 && y0 + TY + 1 <= P.ny;
  if (!(x0 >= 2 && x0 + TX + 2 <= P.nx && y0 >= 1 && y0 + TY + 1 <= P.ny)) {
    patch_box<false>(P, src, rows, R, AX, AY, x0 - 2, y0 - 1, inv2a);
    __syncthreads();
  }
  for (int q = threadIdx.x; q < NA; q += NT) flux_cell(R, NA, F, NA, q, inv2a, gm1, false);
  __syncthreads();

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int i = x0 + tx, j = y0 + ty;
  unsigned long long bits = 0;
  int bad = 0, nonfin = 0;
  if (i < P.nx && j < P.ny) {
    auto rq = [](int x, int y) { return (y + 1) * AX + (x + 2); };
    auto M = [&](int q, int k) { return staged_m(R, NA, F, NA, q, k, w); };
    auto gpop = [&](int k, int ii, int jj) {  // interior: direct; ring: fill_ghosts values
      if (ii >= 0 && ii < P.nx && jj >= 0 && jj < P.ny)
        return load_plane4(src + (4 + 4 * k) * P.plane, P.plane, (long long)jj * P.pitch + ii);
      return load_pop(P, src, rows, k, ii, jj, inv2a);
    };
    double tw, te, ts, tn;
    if (kMode == 0 && interior) {  // face_thetas without the boundary branches
      const double* th = P.theta + (long long)s * P.plane + (long long)j * P.pitch + i;
      const double tc = th[0];
      tw = smin(th[-1], tc);
      te = smin(tc, th[1]);
      ts = smin(th[-P.pitch], tc);
      tn = smin(tc, th[P.pitch]);
    } else {
      face_thetas<kMode>(P, s, i, j, const_theta, tw, te, ts, tn);
    }
    const long long off = (long long)j * P.pitch + i;
    const int qc = rq(tx, ty), qw = rq(tx - 1, ty), qe = rq(tx + 1, ty), qs = rq(tx, ty - 1),
              qn = rq(tx, ty + 1);
    // Pulled populations: on interior tiles (CTA-uniform test) the 16 loads
    // sit in one branch-free block so they issue back to back.
    cs pw, pe, ps, pn;
    if (interior) {
      pw = load_plane4(src + 4 * P.plane, P.plane, off - 1);
      pe = load_plane4(src + 8 * P.plane, P.plane, off + 1);
      ps = load_plane4(src + 12 * P.plane, P.plane, off - P.pitch);
      pn = load_plane4(src + 16 * P.plane, P.plane, off + P.pitch);
    } else {
      pw = gpop(0, i - 1, j);
      pe = gpop(1, i + 1, j);
      ps = gpop(2, i, j - 1);
      pn = gpop(3, i, j + 1);
    }
    const cs M0W = M(qw, 0), M1E = M(qe, 1), M2S = M(qs, 2), M3N = M(qn, 3);
    const cs n1 = add(M0W, scale(tw, sub(M0W, pw)));
    const cs n2 = add(M1E, scale(te, sub(M1E, pe)));
    const cs n3 = add(M2S, scale(ts, sub(M2S, ps)));
    const cs n4 = add(M3N, scale(tn, sub(M3N, pn)));
    store_plane4(dst + 4 * P.plane, P.plane, off, n1);
    store_plane4(dst + 8 * P.plane, P.plane, off, n2);
    store_plane4(dst + 12 * P.plane, P.plane, off, n3);
    store_plane4(dst + 16 * P.plane, P.plane, off, n4);
    cs un = add(add(add(n1, n2), add(n3, n4)), scale(P.alpha, plane4(R, NA, qc)));
    const cs P0C = load_plane4(src + 4 * P.plane, P.plane, off);
    const cs P1C = load_plane4(src + 8 * P.plane, P.plane, off);
    const cs P2C = load_plane4(src + 12 * P.plane, P.plane, off);
    const cs P3C = load_plane4(src + 16 * P.plane, P.plane, off);
    const cs out = add(add(scale(tw, sub(M(qc, 1), P1C)), scale(te, sub(M(qc, 0), P0C))),
                       add(scale(ts, sub(M(qc, 3), P3C)), scale(tn, sub(M(qc, 2), P2C))));
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

// The dynamic shared-memory opt-ins are per device (each device's context
// holds its own copy of the kernels): set once per device.
static cudaError_t smem_attrs() {
  static std::mutex mu;
  static int done_mask[4] = {0, 0, 0, 0};  // bit per device id < 128
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (dev < 0 || dev >= 128) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lock(mu);
  if (done_mask[dev >> 5] >> (dev & 31) & 1) return cudaSuccess;
  const cudaError_t r = [] {
    cudaError_t e = cudaFuncSetAttribute(k_theta_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tiled::kThetaSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_theta_hard, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kHardSmem);
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
  if (r == cudaSuccess) done_mask[dev >> 5] |= 1 << (dev & 31);
  return r;
}

static_assert(tiled::TX == 32 && tiled::TYT == VLBM_THETA_TY, "theta_tiles() layout");
// grid: (tile x, tile y, sample)
static dim3 tiled_grid(const MarchParams& P) {
  return dim3((P.nx + tiled::TX - 1) / tiled::TX, (P.ny + tiled::TY - 1) / tiled::TY, P.S);
}

// 4-D tensor maps [x = nx, y = ny, plane = 20, sample = S] over both state
// buffers with the three tile boxes the kernels load.
int encode_tensor_maps(MarchParams& P) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !fn)
      return set_error(VLBM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<Encode>(fn);
  }
  const cuuint64_t dims[4] = {(cuuint64_t)P.nx, (cuuint64_t)P.ny, (cuuint64_t)kPlanes,
                              (cuuint64_t)P.S};
  const cuuint64_t strides[3] = {(cuuint64_t)P.pitch * 8, (cuuint64_t)P.plane * 8,
                                 (cuuint64_t)P.sample_stride * 8};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const cuuint32_t box_adv[4] = {tiled::AX, tiled::AY, 4, 1};
  const cuuint32_t box_thu[4] = {tiled::RX2, tiled::RY2, 4, 1};
  const cuuint32_t box_thp[4] = {tiled::AX, tiled::AYT, 16, 1};
  for (int b = 0; b < 2; ++b) {
    void* base = b ? P.buf1 : P.buf0;
    CUresult r = encode(&P.tm_adv[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides,
                        box_adv, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
      r = encode(&P.tm_thu[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box_thu,
                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
      r = encode(&P.tm_thp[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box_thp,
                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return set_error(VLBM_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  }
  return VLBM_OK;
}

cudaError_t launch_theta_tiled(const MarchParams& P, cudaStream_t st) {
  if (cudaError_t e = smem_attrs()) return e;
  // persistent: the resident CTAs of this sample group's share of the GPU
  const long long tiles = (long long)P.S * theta_tiles(P.nx, P.ny);
  const int g = (int)(tiles < P.persist_ctas ? tiles : P.persist_ctas);
  k_theta_tiled<<<g, tiled::NTT, tiled::kThetaSmem, st>>>(P, P.tm_thu[0], P.tm_thu[1],
                                                          P.tm_thp[0], P.tm_thp[1]);
  return cudaGetLastError();
}

int theta_ctas_per_sm() {
  if (smem_attrs() != cudaSuccess) return 1;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_theta_tiled, tiled::NTT,
                                                    tiled::kThetaSmem) != cudaSuccess)
    return 1;
  return n > 0 ? n : 1;
}

#ifndef VLBM_CERT_GRID
#define VLBM_CERT_GRID 8  // k_bisect_cert CTAs = 148 x this
#endif
#ifndef VLBM_TAIL_GRID
#define VLBM_TAIL_GRID 4  // k_bisect_tail CTAs = 148 x this
#endif
cudaError_t launch_theta_hard(const MarchParams& P, cudaStream_t st) {
  if (cudaError_t e = smem_attrs()) return e;
  if (P.hq) {
    k_theta_hard<<<148 * VLBM_HARD_MINB, kHB, kHardSmem, st>>>(P);
    // the certified (diagonal-only) bisections run beside the uncertified
    // ones: disjoint cells and queues; joined before the advance
    cudaStream_t cs_ = st;
    if (P.side) {
      if (cudaError_t e = cudaEventRecord(P.ev_fork, st)) return e;
      if (cudaError_t e = cudaStreamWaitEvent(P.side, P.ev_fork, 0)) return e;
      cs_ = P.side;
    }
    k_bisect_cert<<<148 * VLBM_CERT_GRID, 256, 0, cs_>>>(P);
    k_bisect_unc<<<dim3(148 * VLBM_UNC_GRID * (256 / VLBM_UNC_THREADS), 3), VLBM_UNC_THREADS, 0, st>>>(P);
    if (P.replay) k_bisect_tail<<<148 * VLBM_TAIL_GRID, 128, 0, st>>>(P);
    cudaError_t err = cudaGetLastError();
    if (P.side) {
      // once forked, always join (also on an error path): a stream left
      // forked inside a graph capture would surface as an opaque
      // "unjoined" capture failure instead of the real error
      const cudaError_t ej = cudaEventRecord(P.ev_join, P.side);
      const cudaError_t ew = cudaStreamWaitEvent(st, P.ev_join, 0);
      if (err == cudaSuccess) err = ej != cudaSuccess ? ej : ew;
    }
    return err;
  }
  return cudaGetLastError();
}

cudaError_t launch_advance_tiled(const MarchParams& P, int mode, double const_theta,
                                 cudaStream_t st) {
  if (cudaError_t e = smem_attrs()) return e;
  const dim3 g = tiled_grid(P);
  const size_t sm = tiled::kAdvanceSmem;
  if (mode == 0)
    k_advance_tiled<0><<<g, tiled::NT, sm, st>>>(P, const_theta, P.tm_adv[0], P.tm_adv[1]);
  else if (mode == 1)
    k_advance_tiled<1><<<g, tiled::NT, sm, st>>>(P, const_theta, P.tm_adv[0], P.tm_adv[1]);
  else
    k_advance_tiled<2><<<g, tiled::NT, sm, st>>>(P, const_theta, P.tm_adv[0], P.tm_adv[1]);
  return cudaGetLastError();
}

}  // namespace vlbm_impl
