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

#include "march.cuh"
#include "rlmp.cuh"

namespace vlbm_dev {

// ---------------------------------------------------------------------------
// Boundary-ring synthesis.  A padded coordinate (i, j), -2 <= i < nx+2,
// -2 <= j < ny+2, resolves to the interior cell whose value the reference's
// fill_ghosts copies into it: y sides first map the row (wall mirror or
// periodic wrap, solver.hpp:270-285), then x sides map the column at that row
// (inlet / outflow copy / periodic wrap, solver.hpp:234-269).  Corners
// therefore see the x-side value of the mirrored row, exactly as the
// reference fills them (x sides first, then y across the full width).
struct Src {
  int i, j;
  bool mirror;  // wall: mom_y negated, pops 2 <-> 3 (set_wall_ghost :218-228)
  bool inlet;   // inlet ghost: u = u_in(row j), pops = M_k(u_in, a) (:236-243)
};

__device__ __forceinline__ Src resolve(const MarchParams& P, int i, int j) {
  Src r{i, j, false, false};
  if (j < 0) {
    if (P.bc[2] == BC_WALL) {
      r.j = -1 - j;
      r.mirror = true;
    } else {
      r.j = j + P.ny;
    }
  } else if (j >= P.ny) {
    if (P.bc[3] == BC_WALL) {
      r.j = 2 * P.ny - 1 - j;
      r.mirror = true;
    } else {
      r.j = j - P.ny;
    }
  }
  if (i < 0) {
    if (P.bc[0] == BC_INLET)
      r.inlet = true;
    else if (P.bc[0] == BC_OUTFLOW)
      r.i = 0;
    else
      r.i = i + P.nx;
  } else if (i >= P.nx) {
    if (P.bc[1] == BC_OUTFLOW)
      r.i = P.nx - 1;
    else
      r.i = i - P.nx;
  }
  return r;
}

__device__ __forceinline__ cs load_plane4(const double* base, long long plane, long long off) {
  return {base[off], base[plane + off], base[2 * plane + off], base[3 * plane + off]};
}

__device__ __forceinline__ cs inlet_row(const double* rows, int j) {
  const double* q = rows + 4 * j;
  return {q[0], q[1], q[2], q[3]};
}

// Macroscopic state of padded cell (i, j).
__device__ __forceinline__ cs load_u(const MarchParams& P, const double* src, const double* rows,
                                     int i, int j) {
  const Src r = resolve(P, i, j);
  cs u = r.inlet ? inlet_row(rows, r.j)
                 : load_plane4(src, P.plane, (long long)r.j * P.pitch + r.i);
  if (r.mirror) u.my = -u.my;
  return u;
}

// Population k of padded cell (i, j) at kinetic speed parameter inv2a.
__device__ __forceinline__ cs load_pop(const MarchParams& P, const double* src, const double* rows,
                                       int k, int i, int j, double inv2a) {
  const Src r = resolve(P, i, j);
  const int ks = r.mirror ? (k ^ ((k >> 1) & 1)) : k;  // {0,1,3,2} under the mirror
  cs f;
  if (r.inlet)
    f = maxw_k(inlet_row(rows, r.j), ks, P.w, inv2a, P.gm1);
  else
    f = load_plane4(src + (4 + 4 * ks) * P.plane, P.plane, (long long)r.j * P.pitch + r.i);
  if (r.mirror) f.my = -f.my;
  return f;
}

__device__ __forceinline__ const double* state_src(const MarchParams& P, int s, int parity) {
  return (parity ? P.buf1 : P.buf0) + (long long)s * P.sample_stride;
}
__device__ __forceinline__ double* state_dst(const MarchParams& P, int s, int parity) {
  return (parity ? P.buf0 : P.buf1) + (long long)s * P.sample_stride;
}

// ---------------------------------------------------------------------------
// Block reduction of (max signal bits, bad, nonfinite) into the sample's ctl.
__device__ __forceinline__ void reduce_signal(SampleCtl* c, unsigned long long bits, int bad,
                                              int nonfin) {
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = ob > bits ? ob : bits;
  }
  bad = __any_sync(0xffffffffu, bad);
  nonfin = __any_sync(0xffffffffu, nonfin);
  __shared__ unsigned long long s_bits[32];
  __shared__ int s_flags[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
  if (lane == 0) {
    s_bits[warp] = bits;
    s_flags[warp] = (bad ? 1 : 0) | (nonfin ? 2 : 0);
  }
  __syncthreads();
  if (warp == 0) {
    bits = lane < nw ? s_bits[lane] : 0ull;
    int fl = lane < nw ? s_flags[lane] : 0;
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ob = __shfl_xor_sync(0xffffffffu, bits, o);
      bits = ob > bits ? ob : bits;
      fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    }
    if (lane == 0) {
      if (bits) atomicMax(&c->smax_bits, bits);
      if (fl & 1) atomicOr(&c->bad_signal, 1);
      if (fl & 2) atomicOr(&c->nonfinite, 1);
    }
  }
}

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
    if (P.hq_n) *P.hq_n = 0;  // empty hard-cell queue for the coming limiter pass
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

// ---------------------------------------------------------------------------
// Face theta from cell theta (interface_theta, solver.hpp:510-534).
__device__ __forceinline__ double cell_theta(const MarchParams& P, const double* th, int i,
                                             int j) {
  return th[(long long)j * P.pitch + i];
}

template <int kMode>  // 0: cell theta plane, 1: constant, 2: prescribed faces
__device__ __forceinline__ void face_thetas(const MarchParams& P, int s, int i, int j,
                                            double const_theta, double& tw, double& te,
                                            double& ts, double& tn) {
  if (kMode == 1) {
    tw = te = ts = tn = const_theta;
    return;
  }
  if (kMode == 2) {
    const double* tx = P.face_tx + (long long)s * P.ny * (P.nx + 1);
    const double* ty = P.face_ty + (long long)s * (P.ny + 1) * P.nx;
    tw = tx[(long long)j * (P.nx + 1) + i];
    te = tx[(long long)j * (P.nx + 1) + i + 1];
    ts = ty[(long long)j * P.nx + i];
    tn = ty[(long long)(j + 1) * P.nx + i];
    return;
  }
  const double* th = P.theta + (long long)s * P.plane;
  const int nx = P.nx, ny = P.ny;
  const double tc = cell_theta(P, th, i, j);
  const bool per_x = P.bc[0] == BC_PERIODIC, per_y = P.bc[2] == BC_PERIODIC;
  if (i > 0) {
    tw = smin(cell_theta(P, th, i - 1, j), tc);
  } else {
    tw = per_x ? smin(cell_theta(P, th, 0, j), cell_theta(P, th, nx - 1, j)) : tc;
  }
  if (i + 1 < nx) {
    te = smin(tc, cell_theta(P, th, i + 1, j));
  } else {
    te = per_x ? smin(cell_theta(P, th, 0, j), cell_theta(P, th, nx - 1, j)) : tc;
  }
  if (j > 0) {
    ts = smin(cell_theta(P, th, i, j - 1), tc);
  } else {
    ts = per_y ? smin(cell_theta(P, th, i, 0), cell_theta(P, th, i, ny - 1)) : tc;
  }
  if (j + 1 < ny) {
    tn = smin(tc, cell_theta(P, th, i, j + 1));
  } else {
    tn = per_y ? smin(cell_theta(P, th, i, 0), cell_theta(P, th, i, ny - 1)) : tc;
  }
}

__device__ __forceinline__ void store_plane4(double* base, long long plane, long long off,
                                             const cs& v) {
  base[off] = v.r;
  base[plane + off] = v.mx;
  base[2 * plane + off] = v.my;
  base[3 * plane + off] = v.e;
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

// ===========================================================================
// Tiled kernels (the production path).  A CTA owns a TX x TY tile of interior
// cells of one sample, one thread per cell.  The macroscopic state of the tile
// plus its halo is staged once in shared memory together with the per-cell
// quantities every stencil neighbour needs -- u, inv2a*f(u), inv2a*g(u) and
// p(u) -- so each flux / pressure division is evaluated once per cell instead
// of once per use.  M_k(u) is rebuilt from the staged terms exactly as
// maxwellians() forms it (w*u +/- inv2a*f), so every value is bit-identical to
// the reference's.
namespace tiled {
constexpr int TX = 32, TY = 8, NT = TX * TY;
// limiter: halo 2 (u at distance 2 for the allowance, M at distance 2 for u_FO)
constexpr int RX2 = TX + 4, RY2 = TY + 4, NR2 = RX2 * RY2;
constexpr int FX = TX + 2, FY = TY + 2, NF = FX * FY;  // u_FO ring region
constexpr int QW = 24;                                 // doubles per hard-cell entry
// advance: halo 1
constexpr int RX1 = TX + 2, RY1 = TY + 2, NR1 = RX1 * RY1;
constexpr int kStaged = 13;  // u(4), inv2a*f(4), inv2a*g(4), p
constexpr size_t kThetaSmem = sizeof(double) * (kStaged * NR2 + 2 * NF + QW * NT) + sizeof(int) * NT;
constexpr size_t kAdvanceSmem = sizeof(double) * (kStaged * NR1);
}  // namespace tiled

// Stage one padded cell: u, inv2a*flux_x(u), inv2a*flux_y(u), pressure(u).
// flux_x/flux_y (euler.hpp:86-97) each evaluate pressure(u); it is computed
// once here -- the same value.
__device__ __forceinline__ void stage_cell(double* R, int NR, int q, const cs& u, double inv2a,
                                           double gm1) {
  const double p = pressure(u, gm1);
  const double v1 = u.mx / u.r;
  const double v2 = u.my / u.r;
  R[q] = u.r;
  R[NR + q] = u.mx;
  R[2 * NR + q] = u.my;
  R[3 * NR + q] = u.e;
  R[4 * NR + q] = u.mx * inv2a;
  R[5 * NR + q] = (u.mx * v1 + p) * inv2a;
  R[6 * NR + q] = (u.my * v1) * inv2a;
  R[7 * NR + q] = ((u.e + p) * v1) * inv2a;
  R[8 * NR + q] = u.my * inv2a;
  R[9 * NR + q] = (u.mx * v2) * inv2a;
  R[10 * NR + q] = (u.my * v2 + p) * inv2a;
  R[11 * NR + q] = ((u.e + p) * v2) * inv2a;
  R[12 * NR + q] = p;
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

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Population k at padded (i, j); interior cells take the direct path.
__device__ __forceinline__ cs pop_at(const MarchParams& P, const double* src, const double* rows,
                                     int k, int i, int j, double inv2a) {
  if (i >= 0 && i < P.nx && j >= 0 && j < P.ny)
    return load_plane4(src + (4 + 4 * k) * P.plane, P.plane, (long long)j * P.pitch + i);
  return load_pop(P, src, rows, k, i, j, inv2a);
}

__global__ void __launch_bounds__(tiled::NT, 2) k_theta_tiled(MarchParams P, int tiles_x) {
  using namespace tiled;
  extern __shared__ double sm[];
  __shared__ int qn;
  const int s = blockIdx.y;
  const SampleCtl* c = P.ctl + s;
  if (!c->active) return;
  double* R = sm;                     // kStaged x NR2
  double* RF = R + kStaged * NR2;     // rfo[NF], pfo[NF]
  double* Q = RF + 2 * NF;            // hard-cell queue, QW x NT (SoA)
  int* qidx = reinterpret_cast<int*>(Q + QW * NT);
  const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * TY;
  const double* src = state_src(P, s, c->parity);
  const double* rows = P.inlet + (long long)s * P.ny * 4;
  const double inv2a = 0.5 / c->a;
  const double gm1 = P.gm1, w = P.w, al = P.alpha;
  if (threadIdx.x == 0) qn = 0;

  // Phase 1: stage u, fluxes and p(u) on the tile + halo 2.
  for (int q = threadIdx.x; q < NR2; q += NT) {
    const int gi = clampi(x0 + q % RX2 - 2, -2, P.nx + 1);
    const int gj = clampi(y0 + q / RX2 - 2, -2, P.ny + 1);
    stage_cell(R, NR2, q, load_u(P, src, rows, gi, gj), inv2a, gm1);
  }
  __syncthreads();

  // Phase 2: first-order candidates (compute_candidates, solver.hpp:301-316)
  // on the tile and its 1-ring (corners are never used).
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
  __syncthreads();

  // Phase 3: gather the limiter inputs of this thread's cell and try theta = 1.
  const int i = x0 + tx, j = y0 + ty;
  const bool valid = i < P.nx && j < P.ny;
  if (valid) {
    cs cf[4];
    {
      const cs P0W = pop_at(P, src, rows, 0, i - 1, j, inv2a);
      const cs P1E = pop_at(P, src, rows, 1, i + 1, j, inv2a);
      const cs P2S = pop_at(P, src, rows, 2, i, j - 1, inv2a);
      const cs P3N = pop_at(P, src, rows, 3, i, j + 1, inv2a);
      const long long off = (long long)j * P.pitch + i;
      const cs P0C = load_plane4(src + 4 * P.plane, P.plane, off);
      const cs P1C = load_plane4(src + 8 * P.plane, P.plane, off);
      const cs P2C = load_plane4(src + 12 * P.plane, P.plane, off);
      const cs P3C = load_plane4(src + 16 * P.plane, P.plane, off);
      const int qc = rq(tx, ty);
      cf[0] = sub(sub(staged_m(R, NR2, rq(tx - 1, ty), 0, w), P0W),
                  sub(staged_m(R, NR2, qc, 1, w), P1C));
      cf[1] = sub(sub(staged_m(R, NR2, rq(tx + 1, ty), 1, w), P1E),
                  sub(staged_m(R, NR2, qc, 0, w), P0C));
      cf[2] = sub(sub(staged_m(R, NR2, rq(tx, ty - 1), 2, w), P2S),
                  sub(staged_m(R, NR2, qc, 3, w), P3C));
      cf[3] = sub(sub(staged_m(R, NR2, rq(tx, ty + 1), 3, w), P3N),
                  sub(staged_m(R, NR2, qc, 2, w), P2C));
    }
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
    const RlmpBounds b = rlmp_bounds(st, P.kappa, P.rho_floor_coef, P.p_floor_coef);
    const cs delta = add(add(cf[0], cf[1]), add(cf[2], cf[3]));
    if (feasible(1.0, foC, delta, cf, b, gm1)) {
      P.theta[(long long)s * P.plane + (long long)j * P.pitch + i] = 1.0;
    } else {
      const int slot = atomicAdd(&qn, 1);
      Q[0 * NT + slot] = foC.r;
      Q[1 * NT + slot] = foC.mx;
      Q[2 * NT + slot] = foC.my;
      Q[3 * NT + slot] = foC.e;
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        Q[(4 + 4 * f) * NT + slot] = cf[f].r;
        Q[(5 + 4 * f) * NT + slot] = cf[f].mx;
        Q[(6 + 4 * f) * NT + slot] = cf[f].my;
        Q[(7 + 4 * f) * NT + slot] = cf[f].e;
      }
      Q[20 * NT + slot] = b.rho_lo;
      Q[21 * NT + slot] = b.rho_hi;
      Q[22 * NT + slot] = b.p_lo;
      Q[23 * NT + slot] = b.p_hi;
      qidx[slot] = j * P.pitch + i;
    }
  }
  __syncthreads();

  // Phase 4: the cells that failed theta = 1 go to the global hard-cell queue
  // (one atomic per CTA), processed by k_theta_hard at full occupancy so the
  // 30-step bisections neither serialise warps of easy cells nor keep this
  // CTA resident.  If the queue is full they are finished here instead.
  const int n = qn;
  if (n == 0) return;
  __shared__ int qbase;
  if (threadIdx.x == 0) qbase = P.hq ? atomicAdd(P.hq_n, n) : P.hq_cap;
  __syncthreads();
  const int base = qbase;
  if (base + n <= P.hq_cap) {
    for (int slot = threadIdx.x; slot < n; slot += NT) {
#pragma unroll 4
      for (int k = 0; k < kHardWords; ++k)
        P.hq[(long long)k * P.hq_cap + base + slot] = Q[k * NT + slot];
      P.hq_idx[base + slot] = (long long)s * P.plane + qidx[slot];
    }
    return;
  }
  for (int slot = base + threadIdx.x; slot < P.hq_cap; slot += NT) P.hq_idx[slot] = -1;
  for (int slot = threadIdx.x; slot < n; slot += NT) {
    const cs fo = {Q[0 * NT + slot], Q[1 * NT + slot], Q[2 * NT + slot], Q[3 * NT + slot]};
    cs cf[4];
#pragma unroll
    for (int f = 0; f < 4; ++f)
      cf[f] = {Q[(4 + 4 * f) * NT + slot], Q[(5 + 4 * f) * NT + slot], Q[(6 + 4 * f) * NT + slot],
               Q[(7 + 4 * f) * NT + slot]};
    RlmpBounds b;
    b.rho_lo = Q[20 * NT + slot];
    b.rho_hi = Q[21 * NT + slot];
    b.p_lo = Q[22 * NT + slot];
    b.p_hi = Q[23 * NT + slot];
    b.rho_floor = P.rho_floor_coef;
    b.p_floor = P.p_floor_coef;
    const double th = rlmp_theta_hard(fo, cf, b, gm1);
    P.theta[(long long)s * P.plane + qidx[slot]] = th;
  }
}

// The limiter's hard cells from the global queue (rlmp_theta after a failed
// feasible(1.0), solver.hpp:462-486), one thread per cell, grid-stride.
__global__ void __launch_bounds__(256, 2) k_theta_hard(MarchParams P) {
  const int n = min(*P.hq_n, P.hq_cap);
  const long long cap = P.hq_cap;
  for (int slot = blockIdx.x * blockDim.x + threadIdx.x; slot < n;
       slot += gridDim.x * blockDim.x) {
    const long long idx = P.hq_idx[slot];
    if (idx < 0) continue;
    const double* q = P.hq + slot;
    const cs fo = {q[0], q[cap], q[2 * cap], q[3 * cap]};
    cs cf[4];
#pragma unroll
    for (int f = 0; f < 4; ++f)
      cf[f] = {q[(4 + 4 * f) * cap], q[(5 + 4 * f) * cap], q[(6 + 4 * f) * cap],
               q[(7 + 4 * f) * cap]};
    RlmpBounds b;
    b.rho_lo = q[20 * cap];
    b.rho_hi = q[21 * cap];
    b.p_lo = q[22 * cap];
    b.p_hi = q[23 * cap];
    b.rho_floor = P.rho_floor_coef;
    b.p_floor = P.p_floor_coef;
    P.theta[idx] = rlmp_theta_hard(fo, cf, b, P.gm1);
  }
}

// Blended stream-collide, tiled: M_k of the tile + 1-ring from shared memory.
template <int kMode>
__global__ void __launch_bounds__(tiled::NT, 2) k_advance_tiled(MarchParams P, double const_theta,
                                                                int tiles_x) {
  using namespace tiled;
  extern __shared__ double sm[];
  const int s = blockIdx.y;
  SampleCtl* c = P.ctl + s;
  if (!c->active) return;
  double* R = sm;
  const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * TY;
  const double* src = state_src(P, s, c->parity);
  double* dst = state_dst(P, s, c->parity);
  const double* rows = P.inlet + (long long)s * P.ny * 4;
  const double inv2a = 0.5 / c->a;
  const double gm1 = P.gm1, w = P.w;
  for (int q = threadIdx.x; q < NR1; q += NT) {
    const int gi = clampi(x0 + q % RX1 - 1, -2, P.nx + 1);
    const int gj = clampi(y0 + q / RX1 - 1, -2, P.ny + 1);
    stage_cell(R, NR1, q, load_u(P, src, rows, gi, gj), inv2a, gm1);
  }
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
    const cs n1 = add(M0W, scale(tw, sub(M0W, pop_at(P, src, rows, 0, i - 1, j, inv2a))));
    const cs n2 = add(M1E, scale(te, sub(M1E, pop_at(P, src, rows, 1, i + 1, j, inv2a))));
    const cs n3 = add(M2S, scale(ts, sub(M2S, pop_at(P, src, rows, 2, i, j - 1, inv2a))));
    const cs n4 = add(M3N, scale(tn, sub(M3N, pop_at(P, src, rows, 3, i, j + 1, inv2a))));
    store_plane4(dst + 4 * P.plane, P.plane, off, n1);
    store_plane4(dst + 8 * P.plane, P.plane, off, n2);
    store_plane4(dst + 12 * P.plane, P.plane, off, n3);
    store_plane4(dst + 16 * P.plane, P.plane, off, n4);
    const cs P0C = load_plane4(src + 4 * P.plane, P.plane, off);
    const cs P1C = load_plane4(src + 8 * P.plane, P.plane, off);
    const cs P2C = load_plane4(src + 12 * P.plane, P.plane, off);
    const cs P3C = load_plane4(src + 16 * P.plane, P.plane, off);
    cs un = add(add(add(n1, n2), add(n3, n4)), scale(P.alpha, staged_u(R, NR1, qc)));
    const cs out = add(add(scale(tw, sub(staged_m(R, NR1, qc, 1, w), P1C)),
                           scale(te, sub(staged_m(R, NR1, qc, 0, w), P0C))),
                       add(scale(ts, sub(staged_m(R, NR1, qc, 3, w), P3C)),
                           scale(tn, sub(staged_m(R, NR1, qc, 2, w), P2C))));
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

template __global__ void k_advance_tiled<0>(MarchParams, double, int);
template __global__ void k_advance_tiled<1>(MarchParams, double, int);
template __global__ void k_advance_tiled<2>(MarchParams, double, int);

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

static cudaError_t smem_attrs() {
  static cudaError_t done = [] {
    cudaError_t e = cudaFuncSetAttribute(k_theta_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tiled::kThetaSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_advance_tiled<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tiled::kAdvanceSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_advance_tiled<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tiled::kAdvanceSmem);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_advance_tiled<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)tiled::kAdvanceSmem);
  }();
  return done;
}

static dim3 tiled_grid(const MarchParams& P, int& tiles_x) {
  tiles_x = (P.nx + tiled::TX - 1) / tiled::TX;
  const int ty = (P.ny + tiled::TY - 1) / tiled::TY;
  return dim3(tiles_x * ty, P.S);
}

cudaError_t launch_theta(const MarchParams& P, cudaStream_t st) {
  if (use_v0()) {
    k_theta<<<tile_grid(P), 256, 0, st>>>(P);
    return cudaGetLastError();
  }
  if (cudaError_t e = smem_attrs()) return e;
  int tx;
  const dim3 g = tiled_grid(P, tx);
  k_theta_tiled<<<g, tiled::NT, tiled::kThetaSmem, st>>>(P, tx);
  if (P.hq) k_theta_hard<<<148 * 8, 256, 0, st>>>(P);
  return cudaGetLastError();
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

cudaError_t launch_set_budget(const MarchParams& P, long long budget, cudaStream_t st) {
  k_set_budget<<<(P.S + 127) / 128, 128, 0, st>>>(P, budget);
  return cudaGetLastError();
}

}  // namespace vlbm_impl
