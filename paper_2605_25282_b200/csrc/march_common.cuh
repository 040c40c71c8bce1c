// march_common.cuh — device helpers shared by the march kernels: boundary-ring
// synthesis on load (fill_ghosts semantics, solver.hpp:230-286), plane
// loads/stores and the per-sample signal-speed reduction.
#pragma once
#include "march.cuh"

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


#ifndef VLBM_STORE_CS
#define VLBM_STORE_CS 1
#endif
__device__ __forceinline__ void store_plane4(double* base, long long plane, long long off,
                                             const cs& v) {
#if VLBM_STORE_CS  // streaming (evict-first) stores: the new state is not re-read
                   // before it leaves L2, the old state's lines stay for the pulls
  __stcs(base + off, v.r);
  __stcs(base + plane + off, v.mx);
  __stcs(base + 2 * plane + off, v.my);
  __stcs(base + 3 * plane + off, v.e);
#else
  base[off] = v.r;
  base[plane + off] = v.mx;
  base[2 * plane + off] = v.my;
  base[3 * plane + off] = v.e;
#endif
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

}  // namespace vlbm_dev
