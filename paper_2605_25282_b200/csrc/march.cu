// march.cu — sm_100a kernels of the batched VLBM march (Simulation::step,
// solver.hpp:160-170, for S samples per launch; sample index = blockIdx.y).
//
//   k_signal     kinetic_speed partials of a field (init and epilogue form)
//   k_init_pops  pops = M_k(u, a0) on the interior (ctor, solver.hpp:93-99)
//   k_sched      per-sample run_sample loop control: finalise the previous
//                step (time/steps/parity/state_finite), suggest_dt, clamp to
//                the target, divergence (solver.hpp:645-658)
//   k_theta      RLMP cell theta (solver.hpp:364-505) with the boundary ring
//                synthesised on load (fill_ghosts, solver.hpp:230-286)
//   k_advance    blended pull stream-collide (solver.hpp:536-575) + fused
//                epilogue: per-sample max signal speed and finiteness
//
// All arithmetic is fp64 in the reference's exact operation order
// (vlbm_device.cuh); build with --fmad=false.
#include <cuda_runtime.h>

#include <cstdlib>

#include "march.cuh"
#include "march_common.cuh"
#include "rlmp.cuh"

namespace vlbm_dev {

// kinetic_speed partials over the interior of the current state
// (solver.hpp:137-145).  Used at construction.
__global__ void k_signal(MarchParams P) {
  const int s = blockIdx.y;
  SampleCtl* c = P.ctl + s;
  const double* src = state_src(P, s, c->parity);
  const long long n = (long long)P.nx * P.ny;
  unsigned long long bits = 0;
  int bad = 0, nonfin = 0;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / P.nx), i = (int)(idx - (long long)j * P.nx);
    const cs u = load_plane4(src, P.plane, (long long)j * P.pitch + i);
    const double sp = signal_speed(u, P.gamma, P.gm1, P.conservative);
    if (!isfinite(sp)) {
      bad = 1;
    } else {
      const unsigned long long b = (unsigned long long)__double_as_longlong(sp);
      bits = b > bits ? b : bits;
    }
    if (!finite4(u)) nonfin = 1;
  }
  reduce_signal(c, bits, bad, nonfin);
}

// Inlet-row part of kinetic_speed (solver.hpp:146-152), constant per sample,
// and a0 = dx / suggest_dt() of the constructor (solver.hpp:93).
__global__ void k_init_sched(MarchParams P, double* a0_out) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < P.S; s += gridDim.x * blockDim.x) {
    SampleCtl* c = P.ctl + s;
    double sm = 0.0;
    int bad_inlet = 0;
    if (P.bc[0] == BC_INLET) {
      for (int j = 0; j < P.ny; ++j) {
        const double sp =
            signal_speed(inlet_row(P.inlet + (long long)s * P.ny * 4, j), P.gamma, P.gm1,
                         P.conservative);
        if (!isfinite(sp)) bad_inlet = 1;
        sm = smax(sm, sp);
      }
    }
    // A non-finite inlet signal makes every kinetic_speed NaN: kept as NaN.
    c->smax_inlet = bad_inlet ? __longlong_as_double(0x7ff8000000000000ll) : sm;
    const int bad = c->bad_signal || bad_inlet;
    const double smax_all = smax(__longlong_as_double((long long)c->smax_bits), sm);
    const double ks = bad ? __longlong_as_double(0x7ff8000000000000ll) : P.safety * smax_all;
    const double dt = P.dx / ks;
    a0_out[s] = P.dx / dt;
  }
}

// initial_field (perturbation.hpp:106-122) laid out on the device: the
// ambient state everywhere except the wedge cells i < counts[j] of row j,
// which hold the inlet state u_in(y_j) -- the same row fill_ghosts uses for
// the inlet ghosts, evaluated on the host with the reference's libm.  The
// counts come from the host with the reference's comparison (wedge_counts).
struct Amb4 {
  double v[4];
};
__global__ void k_init_field(MarchParams P, const int* counts, Amb4 amb) {
  const int s = blockIdx.y;
  double* dst = P.buf0 + (long long)s * P.sample_stride;
  const double* rows = P.inlet + (long long)s * P.ny * 4;
  const long long n = (long long)P.nx * P.ny;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / P.nx), i = (int)(idx - (long long)j * P.nx);
    const bool wedge = i < counts[j];
    const long long off = (long long)j * P.pitch + i;
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[k * P.plane + off] = wedge ? rows[4 * j + k] : amb.v[k];
  }
}

// pops = M_k(u, a0) on the interior (solver.hpp:94-99).
__global__ void k_init_pops(MarchParams P, const double* a0) {
  const int s = blockIdx.y;
  SampleCtl* c = P.ctl + s;
  double* st = const_cast<double*>(state_src(P, s, c->parity));
  const double inv2a = 0.5 / a0[s];
  const long long n = (long long)P.nx * P.ny;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / P.nx), i = (int)(idx - (long long)j * P.nx);
    const long long off = (long long)j * P.pitch + i;
    const cs u = load_plane4(st, P.plane, off);
    cs m[4];
    maxw_x(u, P.w, inv2a, P.gm1, m[0], m[1]);
    maxw_y(u, P.w, inv2a, P.gm1, m[2], m[3]);
    for (int k = 0; k < 4; ++k) {
      double* q = st + (4 + 4 * k) * P.plane + off;
      q[0] = m[k].r;
      q[P.plane] = m[k].mx;
      q[2 * P.plane] = m[k].my;
      q[3 * P.plane] = m[k].e;
    }
  }
}

// run_sample's loop control for every sample (solver.hpp:645-658), one
// thread per sample, single block.  mode 0: dt = min(suggest_dt, target-t)
// while t < target - 1e-12; mode 1: dt = fixed_dt.  Writes the number of
// samples scheduled for the next step to *P.n_active.
__global__ void k_sched(MarchParams P, double target, double fixed_dt) {
  int count = 0;
  for (int s = threadIdx.x; s < P.S; s += blockDim.x) {
    SampleCtl* c = P.ctl + s;
    if (c->active) {  // finalise the step taken since the last call
      c->t += c->dt;
      c->steps += 1;
      c->parity ^= 1;
      c->active = 0;
      if (c->nonfinite) c->status = ST_DIVERGED;  // !state_finite()
    }
    if (c->status != ST_RUNNING || c->budget <= 0) continue;
    if (!(c->t < target - 1e-12)) continue;
    double dt;
    if (fixed_dt > 0.0) {
      dt = fixed_dt;
    } else {
      const double smax_all = smax(__longlong_as_double((long long)c->smax_bits), c->smax_inlet);
      const bool bad = c->bad_signal || isnan(c->smax_inlet);
      const double ks = bad ? __longlong_as_double(0x7ff8000000000000ll) : P.safety * smax_all;
      const double dt_stable = P.dx / ks;
      if (!isfinite(dt_stable) || dt_stable <= 0.0) {
        c->status = ST_DIVERGED;
        continue;
      }
      dt = smin(dt_stable, target - c->t);
    }
    c->dt = dt;
    c->a = P.dx / dt;
    c->inv2a = 0.5 / c->a;
    c->active = 1;
    c->budget -= 1;
    c->smax_bits = 0ull;
    c->bad_signal = 0;
    c->nonfinite = 0;
    ++count;
  }
  __shared__ int s_count;
  if (threadIdx.x == 0) s_count = 0;
  __syncthreads();
  if (count) atomicAdd(&s_count, count);
  __syncthreads();
  if (threadIdx.x == 0) {
    *P.n_active = s_count;
    if (P.hq_n) {  // record the last pass's hard cells, then empty the queues
      const unsigned long long h = (unsigned long long)P.hq_n[0];
      if (P.qstats && P.hq_n[6] > 0) {  // a tile pass ran since the last reset
        if (h > P.qstats[1]) P.qstats[1] = h;
        P.qstats[2] += h;
        P.qstats[3] += 1;
      }
      for (int k = 0; k < 8; ++k) P.hq_n[k] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// RLMP cell theta, one thread per interior cell (v0: all stencil terms
// recomputed per thread from global memory, L1/L2 absorb the re-reads).
__global__ void __launch_bounds__(256) k_theta(MarchParams P) {
  const int s = blockIdx.y;
  const SampleCtl* c = P.ctl + s;
  if (!c->active) return;
  const int i = blockIdx.x % ((P.nx + 31) / 32) * 32 + (threadIdx.x & 31);
  const int j = blockIdx.x / ((P.nx + 31) / 32) * 8 + (threadIdx.x >> 5);
  if (i >= P.nx || j >= P.ny) return;
  const double* src = state_src(P, s, c->parity);
  const double* rows = P.inlet + (long long)s * P.ny * 4;
  const double inv2a = 0.5 / c->a;
  const double gm1 = P.gm1, w = P.w;

  // Macroscopic states on the radius-2 diamond plus the four diagonals.
  const cs uC = load_u(P, src, rows, i, j);
  const cs uW = load_u(P, src, rows, i - 1, j), uE = load_u(P, src, rows, i + 1, j);
  const cs uS = load_u(P, src, rows, i, j - 1), uN = load_u(P, src, rows, i, j + 1);
  const cs uWW = load_u(P, src, rows, i - 2, j), uEE = load_u(P, src, rows, i + 2, j);
  const cs uSS = load_u(P, src, rows, i, j - 2), uNN = load_u(P, src, rows, i, j + 2);
  const cs uSW = load_u(P, src, rows, i - 1, j - 1), uSE = load_u(P, src, rows, i + 1, j - 1);
  const cs uNW = load_u(P, src, rows, i - 1, j + 1), uNE = load_u(P, src, rows, i + 1, j + 1);

  cs d0, d1;  // scratch for the unused half of a maxw pair
  cs M0C, M1C, M2C, M3C;
  maxw_x(uC, w, inv2a, gm1, M0C, M1C);
  maxw_y(uC, w, inv2a, gm1, M2C, M3C);
  cs M0W, M1E, M2S, M3N;
  maxw_x(uW, w, inv2a, gm1, M0W, d1);
  maxw_x(uE, w, inv2a, gm1, d0, M1E);
  maxw_y(uS, w, inv2a, gm1, M2S, d1);
  maxw_y(uN, w, inv2a, gm1, d0, M3N);
  cs M0WW, M1EE, M2SS, M3NN;
  maxw_x(uWW, w, inv2a, gm1, M0WW, d1);
  maxw_x(uEE, w, inv2a, gm1, d0, M1EE);
  maxw_y(uSS, w, inv2a, gm1, M2SS, d1);
  maxw_y(uNN, w, inv2a, gm1, d0, M3NN);
  cs M0SW, M2SW, M1SE, M2SE, M0NW, M3NW, M1NE, M3NE;
  maxw_x(uSW, w, inv2a, gm1, M0SW, d1);
  maxw_y(uSW, w, inv2a, gm1, M2SW, d1);
  maxw_x(uSE, w, inv2a, gm1, d0, M1SE);
  maxw_y(uSE, w, inv2a, gm1, M2SE, d1);
  maxw_x(uNW, w, inv2a, gm1, M0NW, d1);
  maxw_y(uNW, w, inv2a, gm1, d0, M3NW);
  maxw_x(uNE, w, inv2a, gm1, d0, M1NE);
  maxw_y(uNE, w, inv2a, gm1, d0, M3NE);

  // First-order candidates (compute_candidates, solver.hpp:308-313).
  const double al = P.alpha;
  const cs foC = add(add(add(M0W, M1E), add(M2S, M3N)), scale(al, uC));
  const cs foW = add(add(add(M0WW, M1C), add(M2SW, M3NW)), scale(al, uW));
  const cs foE = add(add(add(M0C, M1EE), add(M2SE, M3NE)), scale(al, uE));
  const cs foS = add(add(add(M0SW, M1SE), add(M2SS, M3C)), scale(al, uS));
  const cs foN = add(add(add(M0NW, M1NE), add(M2C, M3NN)), scale(al, uN));

  // Face corrections (solver.hpp:321-329).
  const cs P0W = load_pop(P, src, rows, 0, i - 1, j, inv2a);
  const cs P1E = load_pop(P, src, rows, 1, i + 1, j, inv2a);
  const cs P2S = load_pop(P, src, rows, 2, i, j - 1, inv2a);
  const cs P3N = load_pop(P, src, rows, 3, i, j + 1, inv2a);
  const long long off = (long long)j * P.pitch + i;
  const cs P0C = load_plane4(src + 4 * P.plane, P.plane, off);
  const cs P1C = load_plane4(src + 8 * P.plane, P.plane, off);
  const cs P2C = load_plane4(src + 12 * P.plane, P.plane, off);
  const cs P3C = load_plane4(src + 16 * P.plane, P.plane, off);
  cs cf[4];
  cf[0] = sub(sub(M0W, P0W), sub(M1C, P1C));
  cf[1] = sub(sub(M1E, P1E), sub(M0C, P0C));
  cf[2] = sub(sub(M2S, P2S), sub(M3C, P3C));
  cf[3] = sub(sub(M3N, P3N), sub(M2C, P2C));

  RlmpStencil st;
  st.fo = foC;
  st.pfo[0] = pressure(foC, gm1);
  st.pfo[1] = pressure(foW, gm1);
  st.pfo[2] = pressure(foE, gm1);
  st.pfo[3] = pressure(foS, gm1);
  st.pfo[4] = pressure(foN, gm1);
  st.rfo[0] = foC.r;
  st.rfo[1] = foW.r;
  st.rfo[2] = foE.r;
  st.rfo[3] = foS.r;
  st.rfo[4] = foN.r;
  // previous-step density/pressure: C, W, E, S, N, then WW, EE, SS, NN
  st.rprev[0] = uC.r;
  st.rprev[1] = uW.r;
  st.rprev[2] = uE.r;
  st.rprev[3] = uS.r;
  st.rprev[4] = uN.r;
  st.rprev[5] = uWW.r;
  st.rprev[6] = uEE.r;
  st.rprev[7] = uSS.r;
  st.rprev[8] = uNN.r;
  st.pprev[0] = pressure(uC, gm1);
  st.pprev[1] = pressure(uW, gm1);
  st.pprev[2] = pressure(uE, gm1);
  st.pprev[3] = pressure(uS, gm1);
  st.pprev[4] = pressure(uN, gm1);
  st.pprev[5] = pressure(uWW, gm1);
  st.pprev[6] = pressure(uEE, gm1);
  st.pprev[7] = pressure(uSS, gm1);
  st.pprev[8] = pressure(uNN, gm1);

  const double th = rlmp_theta(st, cf, P.kappa, P.rho_floor_coef, P.p_floor_coef, gm1);
  P.theta[(long long)s * P.plane + off] = th;
}

// Blended stream-collide (advance, solver.hpp:536-575) + kinetic-speed and
// state_finite epilogue for the next k_sched.
template <int kMode>
__global__ void __launch_bounds__(256) k_advance(MarchParams P, double const_theta) {
  const int s = blockIdx.y;
  SampleCtl* c = P.ctl + s;
  if (!c->active) return;
  const int i = blockIdx.x % ((P.nx + 31) / 32) * 32 + (threadIdx.x & 31);
  const int j = blockIdx.x / ((P.nx + 31) / 32) * 8 + (threadIdx.x >> 5);
  unsigned long long bits = 0;
  int bad = 0, nonfin = 0;
  if (i < P.nx && j < P.ny) {
    const double* src = state_src(P, s, c->parity);
    double* dst = state_dst(P, s, c->parity);
    const double* rows = P.inlet + (long long)s * P.ny * 4;
    const double inv2a = 0.5 / c->a;
    const double gm1 = P.gm1, w = P.w;
    double tw, te, ts, tn;
    face_thetas<kMode>(P, s, i, j, const_theta, tw, te, ts, tn);

    const long long off = (long long)j * P.pitch + i;
    const cs uC = load_plane4(src, P.plane, off);
    const cs uW = load_u(P, src, rows, i - 1, j), uE = load_u(P, src, rows, i + 1, j);
    const cs uS = load_u(P, src, rows, i, j - 1), uN = load_u(P, src, rows, i, j + 1);
    cs d, M0C, M1C, M2C, M3C, M0W, M1E, M2S, M3N;
    maxw_x(uC, w, inv2a, gm1, M0C, M1C);
    maxw_y(uC, w, inv2a, gm1, M2C, M3C);
    maxw_x(uW, w, inv2a, gm1, M0W, d);
    maxw_x(uE, w, inv2a, gm1, d, M1E);
    maxw_y(uS, w, inv2a, gm1, M2S, d);
    maxw_y(uN, w, inv2a, gm1, d, M3N);
    const cs P0W = load_pop(P, src, rows, 0, i - 1, j, inv2a);
    const cs P1E = load_pop(P, src, rows, 1, i + 1, j, inv2a);
    const cs P2S = load_pop(P, src, rows, 2, i, j - 1, inv2a);
    const cs P3N = load_pop(P, src, rows, 3, i, j + 1, inv2a);
    const cs P0C = load_plane4(src + 4 * P.plane, P.plane, off);
    const cs P1C = load_plane4(src + 8 * P.plane, P.plane, off);
    const cs P2C = load_plane4(src + 12 * P.plane, P.plane, off);
    const cs P3C = load_plane4(src + 16 * P.plane, P.plane, off);

    const cs n1 = add(M0W, scale(tw, sub(M0W, P0W)));
    const cs n2 = add(M1E, scale(te, sub(M1E, P1E)));
    const cs n3 = add(M2S, scale(ts, sub(M2S, P2S)));
    const cs n4 = add(M3N, scale(tn, sub(M3N, P3N)));
    store_plane4(dst + 4 * P.plane, P.plane, off, n1);
    store_plane4(dst + 8 * P.plane, P.plane, off, n2);
    store_plane4(dst + 12 * P.plane, P.plane, off, n3);
    store_plane4(dst + 16 * P.plane, P.plane, off, n4);
    cs un = add(add(add(n1, n2), add(n3, n4)), scale(P.alpha, uC));
    const cs out = add(add(scale(tw, sub(M1C, P1C)), scale(te, sub(M0C, P0C))),
                       add(scale(ts, sub(M3C, P3C)), scale(tn, sub(M2C, P2C))));
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

template __global__ void k_advance<0>(MarchParams, double);
template __global__ void k_advance<1>(MarchParams, double);
template __global__ void k_advance<2>(MarchParams, double);


}  // namespace vlbm_dev

// ---------------------------------------------------------------------------
// Host launchers.
#include "internal.h"

namespace vlbm_dev {
__global__ void k_set_budget(MarchParams P, long long budget) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < P.S; s += gridDim.x * blockDim.x)
    P.ctl[s].budget = budget;
}
}  // namespace vlbm_dev

namespace vlbm_impl {
using namespace vlbm_dev;

static dim3 tile_grid(const MarchParams& P) {
  const int tx = (P.nx + 31) / 32, ty = (P.ny + 7) / 8;
  return dim3(tx * ty, P.S);
}

cudaError_t launch_signal(const MarchParams& P, cudaStream_t st) {
  const long long n = (long long)P.nx * P.ny;
  int bx = (int)((n + 255) / 256);
  if (bx > 1024) bx = 1024;
  k_signal<<<dim3(bx, P.S), 256, 0, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_init(const MarchParams& P, double* d_a0, cudaStream_t st) {
  k_init_sched<<<(P.S + 127) / 128, 128, 0, st>>>(P, d_a0);
  const long long n = (long long)P.nx * P.ny;
  int bx = (int)((n + 255) / 256);
  if (bx > 1024) bx = 1024;
  k_init_pops<<<dim3(bx, P.S), 256, 0, st>>>(P, d_a0);
  return cudaGetLastError();
}

cudaError_t launch_init_field(const MarchParams& P, const int* counts, const double* amb4,
                              cudaStream_t st) {
  Amb4 amb;
  for (int k = 0; k < 4; ++k) amb.v[k] = amb4[k];
  const long long n = (long long)P.nx * P.ny;
  int bx = (int)((n + 255) / 256);
  if (bx > 1024) bx = 1024;
  k_init_field<<<dim3(bx, P.S), 256, 0, st>>>(P, counts, amb);
  return cudaGetLastError();
}

cudaError_t launch_sched(const MarchParams& P, double target, double fixed_dt, cudaStream_t st) {
  k_sched<<<1, 256, 0, st>>>(P, target, fixed_dt);
  return cudaGetLastError();
}

// VLBM_KERNELS=v0 selects the untiled one-thread-per-cell kernels (the simple
// form kept for A/B checks of the tiled ones; both are sm_100a device code).
static bool use_v0() {
  static const int v = [] {
    const char* e = getenv("VLBM_KERNELS");
    return (e && e[0] == 'v' && e[1] == '0') ? 1 : 0;
  }();
  return v != 0;
}

cudaError_t launch_theta(const MarchParams& P, cudaStream_t st, int part) {
  if (use_v0()) {
    if (part == 0) k_theta<<<tile_grid(P), 256, 0, st>>>(P);
    return cudaGetLastError();
  }
  return part == 0 ? launch_theta_tiled(P, st) : launch_theta_hard(P, st);
}

cudaError_t launch_advance(const MarchParams& P, int mode, double const_theta, cudaStream_t st) {
  if (use_v0()) {
    const dim3 g = tile_grid(P);
    if (mode == 0)
      k_advance<0><<<g, 256, 0, st>>>(P, const_theta);
    else if (mode == 1)
      k_advance<1><<<g, 256, 0, st>>>(P, const_theta);
    else
      k_advance<2><<<g, 256, 0, st>>>(P, const_theta);
    return cudaGetLastError();
  }
  return launch_advance_tiled(P, mode, const_theta, st);
}

cudaError_t launch_set_budget(const MarchParams& P, long long budget, cudaStream_t st) {
  k_set_budget<<<(P.S + 127) / 128, 128, 0, st>>>(P, budget);
  return cudaGetLastError();
}

}  // namespace vlbm_impl
