// post.cu — on-device W1/L1 post-processing of the empirical measures
// (metrics.hpp:29-177), fp64, bit-identical to the reference.
//
//   k_restrict / k_restrict_var   restrict_field (metrics.hpp:29-49)
//   k_strong_partials[_fused]     strong_error's per-sample sums (:69-80) in
//                                 the reference's sequential order; the
//                                 restriction of the fine sample is fused
//   k_w1_*                        wasserstein1's per-cell term (:113-122):
//                                 warp-per-cell sort of M <= 1024
//                                 order-preserving 64-bit keys in registers,
//                                 then the sequential sum over ranks; M > 1024:
//                                 cell-major keys + CUB segmented sort
//   k_ordered_mean                wasserstein1's storage-order acc (:122-124)
//   k_moments                     ensemble_moments (:148-177)
//
// The serial chains (strong_error's num/den, W1's per-cell and per-field
// sums) are evaluated in exactly the reference's order, one dependent DADD
// per term, with the loads staged through shared memory by the other warps
// so only the add latency is on the critical path.
#include <cuda_runtime.h>

#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <type_traits>
#include <cstdint>
#include <cstdlib>

#include "internal.h"

#ifndef VLBM_W1_SORT
// W1 per-cell sort: 2 = 32-bit quantised keys + index through the bitonic
// network, exact order restored among equal quantised keys (default);
// 1 = per-lane sort + merge-path levels on 64-bit keys; 0 = 64-bit bitonic network
#define VLBM_W1_SORT 2
#endif

namespace vlbm_dev {

constexpr unsigned kFull = 0xffffffffu;

// restrict_field: coarse(i,j) = 0.25 * (((f(2i,2j) + f(2i+1,2j)) + f(2i,2j+1)) + f(2i+1,2j+1))
__device__ __forceinline__ double restrict_at(const double* f, int nxf, int i, int j) {
  const double* r0 = f + (long long)(2 * j) * nxf + 2 * i;
  const double* r1 = r0 + nxf;
  const double sum = ((r0[0] + r0[1]) + r1[0]) + r1[1];
  return sum * 0.25;
}
__global__ void k_restrict(int M, int nxc, int nyc, const double* fine, double* coarse) {
  const long long nc = (long long)nxc * nyc, nf = 4 * nc;
  const long long total = (long long)M * 4 * nc;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long mk = idx / nc;  // m * 4 + k
    const long long c = idx - mk * nc;
    const int j = (int)(c / nxc), i = (int)(c - (long long)j * nxc);
    coarse[idx] = restrict_at(fine + mk * nf, 2 * nxc, i, j);
  }
}

__global__ void k_restrict_var(int M, int nxc, int nyc, const double* fine, int var,
                               double* out) {
  const long long nc = (long long)nxc * nyc;
  const long long total = (long long)M * nc;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long m = idx / nc;
    const long long c = idx - m * nc;
    const int j = (int)(c / nxc), i = (int)(c - (long long)j * nxc);
    out[idx] = restrict_at(fine + (m * 4 + var) * 4 * nc, 2 * nxc, i, j);
  }
}

// ---------------------------------------------------------------------------
// strong_error partials.  One CTA per sample; warps 1..3 stage (|a-b|, |b|)
// for a chunk of cells into shared memory (double-buffered) while warp 0
// runs the serial accumulations of the previous chunk in (cell, component)
// order, exactly as metrics.hpp:71-80, one sum per lane.
constexpr int kSpChunk = 256;  // cells per chunk

// Addressing: a(m, k, c) = a[m*as + k*ac + c]; b likewise with (bs, bc), or
// with kFused the restriction of the fine plane at b + m*bs + k*bc.  kNC = 1
// sums one variable only: when the other components are identically zero
// (BASELINE configs[3]) the reference's 4-component sums add only +0.0 terms,
// so the result is bit-identical.
template <bool kFused, int kNC>
__global__ void __launch_bounds__(128) k_strong_partials(int M, long long n, int nxc,
                                                         const double* a, long long as,
                                                         long long ac, const double* b,
                                                         long long bs, long long bc,
                                                         double* partials) {
  __shared__ __align__(16) double sd[2][kSpChunk * kNC];
  __shared__ __align__(16) double sr[2][kSpChunk * kNC];
  const int m = blockIdx.x;
  const double* A = a + (long long)m * as;
  const double* B = b + (long long)m * bs;
  const long long nchunks = (n + kSpChunk - 1) / kSpChunk;
  // Staging: each thread issues the loads of all its items of the chunk
  // before any shared store (kU items per loader thread), so a CTA keeps
  // ~kU * 5 loads in flight per thread.
  constexpr int kLoaders = 96, kU = (kSpChunk * kNC + kLoaders - 1) / kLoaders;
  auto stage = [&](long long ch, int buf, int t0, int nt) {
    const long long c0 = ch * kSpChunk;
    double av[kU], bv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int q = t0 + u * nt;
      const int cl = q / kNC, k = q % kNC;
      const long long c = c0 + cl;
      av[u] = bv[u] = 0.0;
      if (q < kSpChunk * kNC && c < n) {
        if (kFused) {
          const int j = (int)(c / nxc), i = (int)(c - (long long)j * nxc);
          bv[u] = restrict_at(B + (long long)k * bc, 2 * nxc, i, j);
        } else {
          bv[u] = B[(long long)k * bc + c];
        }
        av[u] = A[(long long)k * ac + c];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int q = t0 + u * nt;
      if (q < kSpChunk * kNC && c0 + q / kNC < n) {
        sd[buf][q] = fabs(av[u] - bv[u]);
        sr[buf][q] = fabs(bv[u]);
      }
    }
  };
  // the first chunk is staged by the loader warps too (nt must be kLoaders)
  if (threadIdx.x >= 32) stage(0, 0, threadIdx.x - 32, blockDim.x - 32);
  __syncthreads();
  constexpr int kChains = kNC == 1 ? 2 : 2 + 2 * kNC;
  static_assert(kNC == 1 || kNC == 4, "partials layout: num, den, cnum[4], cden[4]");
  double acc = 0.0;
  for (long long ch = 0; ch < nchunks; ++ch) {
    const int buf = (int)(ch & 1);
    if (threadIdx.x >= 32) {
      if (ch + 1 < nchunks) stage(ch + 1, buf ^ 1, threadIdx.x - 32, blockDim.x - 32);
    } else if (threadIdx.x < kChains) {
      // warp 0, lane l runs chain l: 0 num (every d), 1 den (every r), and
      // with kNC > 1: 2+k cnum[k] (d of component k), 2+kNC+k cden[k].  The
      // lanes issue the same instructions, so one (predicated) DADD per
      // (cell, component) advances every chain in its own order.
      const int l = threadIdx.x;
      const double* src = (l == 0 || (l >= 2 && l < 2 + kNC)) ? sd[buf] : sr[buf];
      const int kk = l < 2 ? -1 : (l - 2) % kNC;
      const long long c0 = ch * kSpChunk;
      const int nc = (int)((n - c0) < kSpChunk ? (n - c0) : kSpChunk);
      for (int cl = 0; cl < nc; ++cl) {
#pragma unroll
        for (int k = 0; k < kNC; ++k) {
          const double v = src[cl * kNC + k];
          if (kk < 0 || kk == k) acc += v;
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < kChains) {
    double* o = partials + (long long)m * 10;
    const int l = threadIdx.x;
    if (kNC == 1) {  // one component: cnum[0] / cden[0] repeat num / den exactly
      o[l] = acc;
      o[l == 0 ? 2 : 6] = acc;
      if (l == 0)
        for (int k = 1; k < 4; ++k) o[2 + k] = o[6 + k] = 0.0;
    } else {
      o[l] = acc;  // 0 num, 1 den, 2..5 cnum, 6..9 cden
    }
  }
}

// ---------------------------------------------------------------------------
// W1.  Order-preserving map of an IEEE double to an unsigned key.
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// Bitonic sort of N = 32*R keys held by one warp, every comparator ascending:
// each merge size k starts with the "flip" step (partner e ^ (k-1), the
// mirror image in the k-block) and continues with half-cleaners (partner
// e ^ j); the lower index always takes the min.  No per-element direction
// logic: 3 instructions per element for an in-register stage, 7 for a
// cross-lane one (2 shuffles, 64-bit compare, xor, 2 selects).  Element
// e = lane*R + r.
template <int R, typename T>
__device__ __forceinline__ void warp_sort_asc(T (&v)[R], int lane) {
  auto cas = [](T& lo, T& hi) {
    const T a = lo, b = hi;
    lo = min(a, b);
    hi = max(a, b);
  };
  // cross-lane step: partner lane ^ m, partner register pr(r); this lane is the
  // upper side iff (lane & topbit) != 0
  auto xlane = [&](int m, int topbit, bool reverse) {
    const bool upper = (lane & topbit) != 0;
    auto upd = [&](T& x, T o) { x = upper ? max(x, o) : min(x, o); };
    if (reverse) {  // partner register R-1-r: exchange mirrored pairs together
#pragma unroll
      for (int r = 0; r < (R + 1) / 2; ++r) {
        const int q = R - 1 - r;
        const T o1 = __shfl_xor_sync(kFull, v[q], m);
        if (q != r) {
          const T o2 = __shfl_xor_sync(kFull, v[r], m);
          upd(v[q], o2);
        }
        upd(v[r], o1);
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) upd(v[r], __shfl_xor_sync(kFull, v[r], m));
    }
  };
#pragma unroll
  for (int k = 2; k <= 32 * R; k <<= 1) {
    // flip step
    if (k <= R) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int r2 = r ^ (k - 1);
        if (r < r2) cas(v[r], v[r2]);
      }
    } else {
      xlane(k / R - 1, k / (2 * R), true);
    }
    // half-cleaners
#pragma unroll
    for (int j = k >> 2; j > 0; j >>= 1) {
      if (j >= R) {
        xlane(j / R, j / R, false);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if ((r & j) == 0) cas(v[r], v[r | j]);
      }
    }
  }
}

// Warp merge sort of N = 32*R keys, element e = lane*R + r on exit (the
// layout of warp_sort_asc).  Each lane sorts its R keys in registers (the
// ascending-only network restricted to in-register stages), then 5 merge
// levels join runs of R, 2R, .., 16R keys: a lane finds where its R outputs
// start on the merge path of its pair of runs (binary search) and merges them
// sequentially into registers; runs live in X (the cell's staging column,
// free once its keys are in registers) at padded positions e + e/32, written
// back after each level.  ~3.9k instructions per 1024 keys against ~7.2k for
// the full network.  Keys are distinct or equal as values, so the merge's tie
// rule does not affect the result.
__device__ __forceinline__ int spos(int e) { return e + (e >> 5); }

template <int R>
__device__ __forceinline__ void warp_merge_sort(unsigned long long (&v)[R], int lane,
                                                unsigned long long* X) {
  auto cas = [](unsigned long long& lo, unsigned long long& hi) {
    const bool lt = hi < lo;
    const unsigned long long a = lo, b = hi;
    lo = lt ? b : a;
    hi = lt ? a : b;
  };
#pragma unroll
  for (int k = 2; k <= R; k <<= 1) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int r2 = r ^ (k - 1);
      if (r < r2) cas(v[r], v[r2]);
    }
#pragma unroll
    for (int j = k >> 2; j > 0; j >>= 1) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((r & j) == 0) cas(v[r], v[r | j]);
    }
  }
  const int e0 = lane * R;
#pragma unroll
  for (int r = 0; r < R; ++r) X[spos(e0 + r)] = v[r];
  __syncwarp();
  constexpr unsigned long long kInf = ~0ull;
#pragma unroll 1
  for (int Lr = R; Lr < 32 * R; Lr <<= 1) {
    const int base = e0 & ~(2 * Lr - 1), d = e0 - base;
    // merge path: i keys from run A = X[base, +Lr), d - i from run B
    int lo = d > Lr ? d - Lr : 0, hi = d < Lr ? d : Lr;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (X[spos(base + mid)] <= X[spos(base + Lr + d - 1 - mid)])
        lo = mid + 1;
      else
        hi = mid;
    }
    int i = lo, j = d - lo;
    unsigned long long ah = i < Lr ? X[spos(base + i)] : kInf;
    unsigned long long bh = j < Lr ? X[spos(base + Lr + j)] : kInf;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool ta = i < Lr && (j >= Lr || ah <= bh);
      v[r] = ta ? ah : bh;
      i += ta;
      j += !ta;
      const bool more = ta ? i < Lr : j < Lr;
      const unsigned long long nv = more ? X[ta ? spos(base + i) : spos(base + Lr + j)] : kInf;
      ah = ta ? nv : ah;
      bh = ta ? bh : nv;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) X[spos(e0 + r)] = v[r];
    __syncwarp();
  }
}

// The same ascending bitonic network on 32-bit keys, laid out for a small
// code footprint: the fully unrolled network is ~2.8 k instructions per sort
// and the kernel then stalls on instruction fetch (ncu: no_instruction 3.9
// cycles per issue), so the cross-lane steps run as runtime loops over the
// partner distance (one shuffle + one min/max per key, 2 R instructions per
// body) and the in-register half-cleaners that end every merge size share one
// body.  Only the in-register stages need compile-time register indices.
template <int R>
__device__ __forceinline__ void warp_sort_u32(unsigned (&v)[R], int lane) {
  auto cas = [](unsigned& lo, unsigned& hi) {
    const unsigned a = lo, b = hi;
    lo = min(a, b);
    hi = max(a, b);
  };
  // the lane's side of a cross-lane compare-exchange: the upper lane keeps the
  // larger key, the lower lane the smaller.  One compare (with the lane's side
  // folded into its predicate) and one select, in place: written as
  // upper ? max : min the runtime loops below carried a max, a predicated min
  // and two register moves per key.
  auto keep = [](unsigned a, unsigned o, bool upper) { return ((o < a) != upper) ? o : a; };
  // runs of R keys sorted inside each lane (merge sizes 2 .. R)
#pragma unroll
  for (int k = 2; k <= R; k <<= 1) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int r2 = r ^ (k - 1);
      if (r < r2) cas(v[r], v[r2]);
    }
#pragma unroll
    for (int j = k >> 2; j > 0; j >>= 1) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((r & j) == 0) cas(v[r], v[r | j]);
    }
  }
  // merge sizes 2R .. 32R: flip across lanes (partner lane ^ (2g - 1), mirrored
  // register), half-cleaners across lanes (partner lane ^ h), then in registers
#pragma unroll 1
  for (int g = 1; g < 32; g <<= 1) {  // g = k / (2R): lanes per half of the merged block
    {
      const int m = 2 * g - 1;
      const bool upper = (lane & g) != 0;
#pragma unroll
      for (int r = 0; r < (R + 1) / 2; ++r) {
        const int q = R - 1 - r;
        const unsigned o1 = __shfl_xor_sync(kFull, v[q], m);
        if (q != r) {
          const unsigned o2 = __shfl_xor_sync(kFull, v[r], m);
          v[q] = keep(v[q], o2, upper);
        }
        v[r] = keep(v[r], o1, upper);
      }
    }
#pragma unroll 1
    for (int h = g >> 1; h > 0; h >>= 1) {
      const bool upper = (lane & h) != 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const unsigned o = __shfl_xor_sync(kFull, v[r], h);
        v[r] = keep(v[r], o, upper);
      }
    }
#pragma unroll
    for (int j = R >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((r & j) == 0) cas(v[r], v[r | j]);
    }
  }
}

// Sorted column by QUANTISED keys: out[r] = the value of rank e = lane*R + r
// among the M values col[0..M) (ranks >= M: unspecified).  The order-
// preserving 64-bit key of each value is reduced to 22 bits relative to the
// cell's own range (q = (key - base) >> sh; base and sh from the smallest and
// largest high words of the keys, warp-uniform) and packed with the value's
// slot as one 32-bit word c = q << 10 | slot, so the bitonic network's
// compare-exchange is one integer min and one max (a 64-bit one costs 6-7
// instructions).  q is monotone in the key, so the network leaves the values
// in exact order except possibly inside runs of EQUAL q, which are contiguous:
// the values are gathered by slot, and only if some adjacent pair of the warp
// shares its q (rare: M <= 1024 values over 4 M buckets) the runs are put in
// exact key order by odd-even transposition passes over the flagged pairs
// until no pass swaps (after 6 passes: the 64-bit merge sort of the gathered
// values, with col as its scratch).  The result is the exact sorted order of
// the keys, as from the 64-bit sorts; col is clobbered.
template <int R>
__device__ __forceinline__ void warp_sort_quantised(int M, int lane, unsigned long long* col,
                                                    unsigned long long (&out)[R]) {
  static_assert(R * 32 <= 1024, "slot index takes 10 bits");
  static_assert(R >= 2, "the exact-order passes pair elements inside a lane");
  unsigned c[R];
  unsigned hmin = 0xffffffffu, hmax = 0u;
#pragma unroll
  for (int r = 0; r < R; ++r) {  // the range of the keys' high words (the column is read twice)
    const int m = r * 32 + lane;
    if (m < M) {
      const unsigned h = (unsigned)(col[m] >> 32);
      hmin = min(hmin, h);
      hmax = max(hmax, h);
    }
  }
  hmin = __reduce_min_sync(kFull, hmin);
  hmax = __reduce_max_sync(kFull, hmax);
  // base and span of the keys: from the high words, or -- when they all agree
  // (a tight cluster) -- from the low words too, so that q is the exact key
  // offset whenever the whole cell spans fewer than 2^22 ulps (no equal-q
  // runs among distinct values then)
  unsigned lbase = 0u;
  unsigned long long span = (((unsigned long long)(hmax - hmin) + 1ull) << 32) - 1ull;
  if (hmin == hmax) {  // warp-uniform
    unsigned lmin = 0xffffffffu, lmax = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int m = r * 32 + lane;
      if (m < M) {
        const unsigned l = (unsigned)col[m];
        lmin = min(lmin, l);
        lmax = max(lmax, l);
      }
    }
    lbase = __reduce_min_sync(kFull, lmin);
    span = __reduce_max_sync(kFull, lmax) - lbase;
  }
  const unsigned long long base = ((unsigned long long)hmin << 32) | lbase;
  // key - base <= span < 2^(64 - clz(span))  ->  q < 2^22
  const int sh = max(0, 42 - __clzll((long long)span));
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int m = r * 32 + lane;
    const unsigned long long d = (m < M ? col[m] : base) - base;
    c[r] = m < M ? ((unsigned)(d >> sh) << 10) | (unsigned)m
                 : 0xffffffffu;  // pads last (slots < M <= 1023 when there are pads)
  }
  warp_sort_u32<R>(c, lane);
  const int e0 = lane * R;
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = e0 + r < M ? col[c[r] & 1023u] : ~0ull;  // pads last
  // adjacent ranks with equal q: bit r = pair (e0 + r, e0 + r + 1), both < M
  const unsigned cnext = __shfl_down_sync(kFull, c[0], 1);
  unsigned eq = 0u;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const unsigned cn = r + 1 < R ? c[r + 1] : cnext;
    const bool in = e0 + r + 1 < M && (r + 1 < R || lane < 31);
    eq |= (in && ((c[r] ^ cn) < 1024u)) ? 1u << r : 0u;
  }
  if (!__any_sync(kFull, eq != 0u)) return;
  bool again = true;
  for (int pass = 0; again; ++pass) {
    if (pass == 6) {  // long runs (values packed far below the cell's range): the 64-bit
                      // merge sort of the gathered values; col is free (every lane gathered)
      __syncwarp();
      warp_merge_sort<R>(out, lane, col);
      return;
    }
    bool sw = false;
#pragma unroll
    for (int par = 0; par < 2; ++par) {
#pragma unroll
      for (int r = par; r + 1 < R; r += 2) {
        if ((eq >> r & 1u) && out[r] > out[r + 1]) {
          const unsigned long long t = out[r];
          out[r] = out[r + 1];
          out[r + 1] = t;
          sw = true;
        }
      }
      if (((R - 1) & 1) == par) {  // the pair across the lane boundary: (lane, R-1) with (lane+1, 0)
        const unsigned long long nx = __shfl_down_sync(kFull, out[0], 1);
        const unsigned long long pv = __shfl_up_sync(kFull, out[R - 1], 1);
        const unsigned eqp = __shfl_up_sync(kFull, eq, 1);
        const bool up = (eq >> (R - 1) & 1u) && out[R - 1] > nx;               // lower side
        const bool dn = lane > 0 && (eqp >> (R - 1) & 1u) && pv > out[0];      // upper side
        if (up) out[R - 1] = nx;
        if (dn) out[0] = pv;
        sw = sw || up || dn;
      }
    }
    again = __any_sync(kFull, sw);
  }
}

// Per-cell term: sum_m |a_(m) - b_(m)| over sorted ranks, sequential in m,
// divided by M (metrics.hpp:118-122).  Loader functors return sample m's
// value of the warp's cell.
// ca / cb: the cell's M values of each ensemble in shared memory (ca is
// overwritten).  One ensemble is sorted at a time (R keys per lane in
// registers); the sorted first column is parked in ca at slot (r, lane) so the
// second sort has the registers to itself.  Rank e = lane*R + r; the chain
// visits lanes in order, each adding its R terms, so the sum is strictly
// sequential in rank as in the reference.
template <int R>
__device__ __forceinline__ double w1_cell(int M, int lane, unsigned long long* ca,
                                          unsigned long long* cb) {
  // The columns hold the values' order-preserving KEYS (dkey, formed once by
  // the staging threads): the sorts compare keys, and dval gives the values
  // back for the terms.
  double sb_[R];
  if constexpr (VLBM_W1_SORT == 2 && R >= 2) {
    unsigned long long kk[R];
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {  // one copy of the network's code for both columns
      warp_sort_quantised<R>(M, lane, pass ? cb : ca, kk);
      if (pass == 0) {
        __syncwarp();  // every lane has gathered from ca
#pragma unroll
        for (int r = 0; r < R; ++r) ca[r * 32 + lane] = kk[r];
        __syncwarp();
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) sb_[r] = dval(kk[r]);
  } else {
  unsigned long long k[R];
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    unsigned long long* col = pass ? cb : ca;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int m = r * 32 + lane;  // load slot order is free: sorting is order-free
      k[r] = m < M ? col[m] : ~0ull;
    }
#if VLBM_W1_SORT == 1
    __syncwarp();  // the column is free once every lane holds its keys
    warp_merge_sort<R>(k, lane, col);
#else
    warp_sort_asc<R>(k, lane);
#endif
    if (pass == 0) {
      __syncwarp();
#pragma unroll
      for (int r = 0; r < R; ++r) ca[r * 32 + lane] = k[r];
      __syncwarp();
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) sb_[r] = dval(k[r]);
  }
  // terms |a_(e) - b_(e)| of the lane's own ranks in registers, all lanes in
  // parallel (padded ranks contribute nothing); then only the dependent adds
  // run lane after lane
  const int valid = M - lane * R;  // ranks of this lane that exist
#pragma unroll
  for (int r = 0; r < R; ++r) sb_[r] = fabs(dval(ca[r * 32 + lane]) - sb_[r]);
  double cell = 0.0;
#pragma unroll 1
  for (int L = 0; L < 32; ++L) {
    if (lane == L) {
      if (valid >= R) {  // a full lane: R unguarded dependent adds
#pragma unroll
        for (int r = 0; r < R; ++r) cell += sb_[r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (r < valid) cell += sb_[r];
      }
    }
    cell = __shfl_sync(kFull, cell, L);
  }
  return cell / static_cast<double>(M);
}

// A CTA of kW1Cells warps owns kW1Cells consecutive cells, one warp per cell.
// The M values of both ensembles for its cells are staged into shared memory
// [cell][m] with sector-efficient loads, then each warp reduces its cell.
//   kKind 0: sample-major planes, value(m, c) = a[m*as + c], b[m*bs + c]
//   kKind 1: coarse planes vs the restriction of fine planes (b = fine,
//            bs = fine sample stride; 32-byte coarse and two 64-byte fine
//            segments per sample, every fetched sector fully used)
//   kKind 2: cell-major columns after the sample->cell re-shard, a[c*M + m]
//   kKind 3: row tables (peer memory): a, b are device arrays of M row
//            pointers (const double* const*) -- sample m's coarse plane and
//            fine plane, each on whichever GPU holds the sample (NVLink peer
//            mapping); as = the first global cell of this launch; the
//            restriction is fused as in kind 1
#ifndef VLBM_W1_CELLS
#define VLBM_W1_CELLS 4
#endif
constexpr int kW1Cells = VLBM_W1_CELLS;
#ifndef VLBM_W1_STAGE
#define VLBM_W1_STAGE 8  // samples whose loads a staging thread keeps in flight
#endif
#ifndef VLBM_W1_MINB
#define VLBM_W1_MINB 4  // register budget: 65536 / (128 threads x this)
#endif

// Sample m's value pair of (launch-local) cell c for the W1 kernels; (i, j):
// the cell's coarse coordinates (kinds 1 and 3), found once per thread.
template <int kKind>
__device__ __forceinline__ void w1_load(int M, long long c, int m, int nxc, int i, int j,
                                        const double* a, long long as, const double* b,
                                        long long bs, double& va, double& vb) {
  if (kKind == 2) {
    va = a[c * M + m];
    vb = b[c * M + m];
  } else if (kKind == 3) {
    va = reinterpret_cast<const double* const*>(a)[m][as + c];
    vb = restrict_at(reinterpret_cast<const double* const*>(b)[m], 2 * nxc, i, j);
  } else {
    va = a[(long long)m * as + c];
    vb = kKind == 1 ? restrict_at(b + (long long)m * bs, 2 * nxc, i, j) : b[(long long)m * bs + c];
  }
}

template <int R, int kKind>
__global__ void __launch_bounds__(32 * kW1Cells, kW1Cells <= 4 ? VLBM_W1_MINB : 1) k_w1_tile(int M, long long n, int nxc,
                                                           const double* a, long long as,
                                                           const double* b, long long bs,
                                                           double* terms) {
  extern __shared__ unsigned long long smw[];  // the values' keys (dkey), [column][cell][m]
  constexpr int LD = 32 * R + 32;  // column stride: transposed stores, merge scratch e + e/32
  unsigned long long* sa = smw;
  unsigned long long* sb = smw + kW1Cells * LD;
  const long long c0 = (long long)blockIdx.x * kW1Cells;
  if (kKind == 2) {
#pragma unroll 4
    for (int e = threadIdx.x; e < M * kW1Cells; e += blockDim.x) {
      const int cl = e / M, m = e - cl * M;
      const long long c = c0 + cl;
      double va = 0.0, vb = 0.0;
      if (c < n) w1_load<kKind>(M, c, m, nxc, 0, 0, a, as, b, bs, va, vb);
      sa[cl * LD + m] = dkey(va);
      sb[cl * LD + m] = dkey(vb);
    }
    __syncthreads();
  } else {
    // element e = m * kW1Cells + cl with e = threadIdx.x + k * blockDim.x: a
    // thread keeps ONE cell (cl) for all its samples, so the cell's coarse
    // coordinates (a 64-bit division) are found once; kStage samples' loads
    // are issued before the first is stored (the staging is latency-bound).
    // (Measured and dropped: the CTAs of a thread-block cluster staging 8 - 32
    // consecutive cells together -- each CTA loading a share of the samples for
    // all the cluster's cells in 64 - 512 B runs and writing the keys into the
    // owners' columns through distributed shared memory: 20.7 / 24.0 / 26.0 ms
    // with 2 / 4 / 8 CTAs per cluster against 20.4 ms.)
    constexpr int kStage = VLBM_W1_STAGE, kStep = 32;  // kStep = blockDim.x / kW1Cells samples apart
    const int cl = (int)threadIdx.x % kW1Cells;
    const long long c = c0 + cl;
    int i = 0, j = 0;
    if (kKind != 0 && c < n) {
      const long long cg_ = (kKind == 3 ? as : 0) + c;
      j = (int)(cg_ / nxc);
      i = (int)(cg_ - (long long)j * nxc);
    }
    unsigned long long* da = sa + cl * LD;
    unsigned long long* db = sb + cl * LD;
    // kVec: each fine row's pair as one 128-bit load (16-byte aligned pairs:
    // an aligned plane and even strides -- every torch / cudaMalloc buffer),
    // so neighbouring lanes read one contiguous run per row
    auto stage = [&](auto vec_tag) {
      constexpr bool kVec = decltype(vec_tag)::value;
      for (int m0 = (int)threadIdx.x / kW1Cells; m0 < M; m0 += kStage * kStep) {
        double va[kStage];
        double2 f0[kStage], f1[kStage];  // the fine rows' pairs (kinds 1, 3); kind 0: b in f0.x
#pragma unroll
        for (int q = 0; q < kStage; ++q) {
          const int m = m0 + q * kStep;
          va[q] = 0.0;
          f0[q] = f1[q] = make_double2(0.0, 0.0);
          if (m < M && c < n) {
            if (kKind == 0) {
              va[q] = a[(long long)m * as + c];
              f0[q].x = b[(long long)m * bs + c];
            } else {
              const double* fb = kKind == 3 ? reinterpret_cast<const double* const*>(b)[m]
                                            : b + (long long)m * bs;
              va[q] = kKind == 3 ? reinterpret_cast<const double* const*>(a)[m][as + c]
                                 : a[(long long)m * as + c];
              const double* r0 = fb + (long long)(2 * j) * (2 * nxc) + 2 * i;
              const double* r1 = r0 + 2 * nxc;
              if (kVec) {
                f0[q] = *reinterpret_cast<const double2*>(r0);
                f1[q] = *reinterpret_cast<const double2*>(r1);
              } else {
                f0[q] = make_double2(r0[0], r0[1]);
                f1[q] = make_double2(r1[0], r1[1]);
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kStage; ++q) {
          const int m = m0 + q * kStep;
          if (m < M) {
            // restrict_field's sum, operation by operation (restrict_at)
            const double vb =
                kKind == 0 ? f0[q].x : (((f0[q].x + f0[q].y) + f1[q].x) + f1[q].y) * 0.25;
            da[m] = dkey(va[q]);
            db[m] = dkey(vb);
          }
        }
      }
    };
    if (kKind == 1 && (reinterpret_cast<unsigned long long>(b) & 15ull) == 0ull && (bs & 1) == 0)
      stage(std::true_type{});
    else
      stage(std::false_type{});
    __syncthreads();
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long c = c0 + w;
  if (c >= n) return;
#ifdef VLBM_W1_EXP_NOSORT  // timing experiment only (WRONG results): the staging alone
  const double t = dval(sa[w * LD + lane]) + dval(sb[w * LD + lane]);
#else
  const double t = w1_cell<R>(M, lane, sa + w * LD, sb + w * LD);
#endif
  if (lane == 0) terms[c] = t;
}

// acc = sum_c terms[c] in storage order; result = acc / n (metrics.hpp:112-124).
constexpr int kOmChunk = 2048;
// acc continues from *acc_io unless first; writes acc back to *acc_io (if
// given) and acc / n_total to *result (if given): a storage-order sum can be
// run in pieces, each piece continuing the previous one's chain exactly.
__global__ void __launch_bounds__(256) k_ordered_sum(long long n, const double* terms,
                                                    double* acc_io, int first, long long n_total,
                                                    double* result) {
  __shared__ __align__(16) double buf[2][kOmChunk];
  const long long nchunks = (n + kOmChunk - 1) / kOmChunk;
  auto stage = [&](long long ch, int bi, int t0, int nt) {
    const long long c0 = ch * kOmChunk;
    for (int q = t0; q < kOmChunk; q += nt)
      if (c0 + q < n) buf[bi][q] = terms[c0 + q];
  };
  stage(0, 0, threadIdx.x, blockDim.x);
  __syncthreads();
  double acc = first ? 0.0 : *acc_io;
  for (long long ch = 0; ch < nchunks; ++ch) {
    const int bi = (int)(ch & 1);
    if (threadIdx.x >= 32) {
      if (ch + 1 < nchunks) stage(ch + 1, bi ^ 1, threadIdx.x - 32, blockDim.x - 32);
    } else if (threadIdx.x == 0) {
      const long long c0 = ch * kOmChunk;
      const int nc = (int)((n - c0) < kOmChunk ? (n - c0) : kOmChunk);
      if (nc == kOmChunk) {
        // software-pipelined: 16 values in registers while the next 16 load;
        // the adds stay one dependent chain in storage order
        const double2* b2 = reinterpret_cast<const double2*>(buf[bi]);
        double2 x[8], y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = b2[i];
        for (int base = 0; base < kOmChunk / 2; base += 8) {
          if (base + 8 < kOmChunk / 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) y[i] = b2[base + 8 + i];
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            acc += x[i].x;
            acc += x[i].y;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = y[i];
        }
      } else {
        for (int q = 0; q < nc; ++q) acc += buf[bi][q];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (acc_io) *acc_io = acc;
    if (result) *result = acc / static_cast<double>(n_total);
  }
}

// ensemble_moments per (component, cell) on sample-major blocks: x(m, q) =
// x[m * stride + q], q over 4*n entries.
__global__ void k_moments(int M, long long nq, const double* x, long long stride, double* mean,
                          double* sd) {
  const double inv_m = 1.0 / M;
  const double inv_m1 = 1.0 / (M - 1.0);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int m = 0; m < M; ++m) s += x[(long long)m * stride + q];
    const double mu = s * inv_m;
    double ss = 0.0;
    for (int m = 0; m < M; ++m) {
      const double d = x[(long long)m * stride + q] - mu;
      ss += d * d;
    }
    mean[q] = mu;
    sd[q] = sqrt(ss * inv_m1);
  }
}

}  // namespace vlbm_dev

namespace vlbm_impl {
using namespace vlbm_dev;

static int grid_for(long long total, int threads = 256, int cap = 148 * 32) {
  long long b = (total + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b > cap ? cap : b);
}

cudaError_t launch_restrict(int M, int nxc, int nyc, const double* fine, double* coarse,
                            cudaStream_t st) {
  k_restrict<<<grid_for((long long)M * 4 * nxc * nyc), 256, 0, st>>>(M, nxc, nyc, fine, coarse);
  return cudaGetLastError();
}

cudaError_t launch_restrict_var(int M, int nxc, int nyc, const double* fine, int var, double* out,
                                cudaStream_t st) {
  k_restrict_var<<<grid_for((long long)M * nxc * nyc), 256, 0, st>>>(M, nxc, nyc, fine, var, out);
  return cudaGetLastError();
}

cudaError_t launch_strong_partials(int M, int64_t n, const double* a, const double* b,
                                   double* partials, cudaStream_t st) {
  k_strong_partials<false, 4><<<M, 128, 0, st>>>(M, n, 0, a, 4 * n, n, b, 4 * n, n, partials);
  return cudaGetLastError();
}

cudaError_t launch_strong_partials_fused(int M, int nxc, int nyc, const double* coarse,
                                         const double* fine, double* partials, cudaStream_t st) {
  const long long n = (long long)nxc * nyc;
  k_strong_partials<true, 4><<<M, 128, 0, st>>>(M, n, nxc, coarse, 4 * n, n, fine, 16 * n, 4 * n,
                                                partials);
  return cudaGetLastError();
}

cudaError_t launch_strong_partials_var(int M, int nxc, int nyc, const double* coarse,
                                       int64_t c_stride, const double* fine, int64_t f_stride,
                                       double* partials, cudaStream_t st) {
  const long long n = (long long)nxc * nyc;
  k_strong_partials<true, 1><<<M, 128, 0, st>>>(M, n, nxc, coarse, c_stride, 0, fine, f_stride,
                                                0, partials);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// W1 for M > 1024 (any ensemble size): cells in batches; both ensembles of a
// batch transposed to cell-major order-preserving keys (32x32 tiles through
// shared memory: coalesced reads along cells, writes along samples; the
// restriction of the fine ensemble fused as in k_w1_tile), each cell's M keys
// sorted by CUB's segmented sort, then one thread per cell adds
// |a_(m) - b_(m)| strictly in rank order (metrics.hpp:118-122).
template <int kKind>
__global__ void k_w1_keys(int M, long long c0, long long nb, int nxc, const double* a,
                          long long as, const double* b, long long bs, unsigned long long* ka,
                          unsigned long long* kb) {
  __shared__ unsigned long long ta[32][33], tb[32][33];
  const long long cb = (long long)blockIdx.x * 32;  // batch-local cell tile
  const int mb = blockIdx.y * 32;                    // sample tile
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  int ci = 0, cj = 0;  // coarse coordinates of this thread's cell (kinds 1 and 3)
  if ((kKind == 1 || kKind == 3) && cb + tx < nb) {
    const long long cg = (kKind == 3 ? as : 0) + c0 + cb + tx;
    cj = (int)(cg / nxc);
    ci = (int)(cg - (long long)cj * nxc);
  }
  for (int r = ty; r < 32; r += 8) {  // read: sample mb + r, cell cb + tx
    const int m = mb + r;
    const long long cl = cb + tx, c = c0 + cl;
    unsigned long long va = 0, vb = 0;
    if (m < M && cl < nb) {
      double x, y;
      w1_load<kKind>(M, c, m, nxc, ci, cj, a, as, b, bs, x, y);
      va = dkey(x);
      vb = dkey(y);
    }
    ta[r][tx] = va;
    tb[r][tx] = vb;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {  // write: cell cb + r, sample mb + tx
    const long long cl = cb + r;
    const int m = mb + tx;
    if (m < M && cl < nb) {
      ka[cl * M + m] = ta[tx][r];
      kb[cl * M + m] = tb[tx][r];
    }
  }
}

__global__ void k_w1_sorted_terms(int M, long long nb, const unsigned long long* ka,
                                  const unsigned long long* kb, double* terms) {
  for (long long cl = (long long)blockIdx.x * blockDim.x + threadIdx.x; cl < nb;
       cl += (long long)gridDim.x * blockDim.x) {
    const unsigned long long* pa = ka + cl * M;
    const unsigned long long* pb = kb + cl * M;
    double cell = 0.0;
    for (int m = 0; m < M; ++m) cell += fabs(dval(pa[m]) - dval(pb[m]));
    terms[cl] = cell / static_cast<double>(M);
  }
}

__global__ void k_seg_offsets(int M, long long nb, int* off) {  // segment c starts at c * M
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c <= nb;
       c += (long long)gridDim.x * blockDim.x)
    off[c] = (int)(c * M);
}

template <int kKind>
static cudaError_t launch_w1_large(int M, long long n, int nxc, const double* a, long long as,
                                   const double* b, long long bs, double* terms,
                                   cudaStream_t st) {
  // batch: 4 key arrays (two ensembles, sorted copies) of M x nb keys within
  // ~4 GB and under CUB's 32-bit item count
  long long nb_max = (4ll << 30) / (32ll * M);
  nb_max = nb_max < (0x7fffffffll / M) ? nb_max : (0x7fffffffll / M);
  nb_max = nb_max < n ? nb_max : n;
  if (const char* e = getenv("VLBM_W1_BATCH_CELLS"))  // test hook: force several batches
    nb_max = std::max(1ll, std::min(nb_max, atoll(e)));
  if (nb_max < 1) return cudaErrorInvalidValue;
  const size_t items = (size_t)M * nb_max;
  unsigned long long *ka = nullptr, *kb = nullptr, *sa = nullptr, *sb = nullptr;
  void* tmp = nullptr;
  int* off = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, ka, sa, (int)items,
                                                     (int)nb_max, off, off + 1, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&off, sizeof(int) * (nb_max + 1), st);
  if (e == cudaSuccess) {
    k_seg_offsets<<<(unsigned)((nb_max + 256) / 256), 256, 0, st>>>(M, nb_max, off);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMallocAsync(&ka, items * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&kb, items * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&sa, items * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&sb, items * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tmp_bytes, st);
  for (long long c0 = 0; e == cudaSuccess && c0 < n; c0 += nb_max) {
    const long long nb = (n - c0) < nb_max ? (n - c0) : nb_max;
    const int nitems = (int)(M * nb);
    const dim3 g((unsigned)((nb + 31) / 32), (unsigned)((M + 31) / 32));
    k_w1_keys<kKind><<<g, 256, 0, st>>>(M, c0, nb, nxc, a, as, b, bs, ka, kb);
    e = cudaGetLastError();
    size_t tb = tmp_bytes;
    if (e == cudaSuccess)
      e = cub::DeviceSegmentedSort::SortKeys(tmp, tb, ka, sa, nitems, (int)nb, off, off + 1, st);
    if (e == cudaSuccess)
      e = cub::DeviceSegmentedSort::SortKeys(tmp, tb, kb, sb, nitems, (int)nb, off, off + 1, st);
    if (e == cudaSuccess) {
      k_w1_sorted_terms<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(M, nb, sa, sb, terms + c0);
      e = cudaGetLastError();
    }
  }
  for (void* p : {(void*)ka, (void*)kb, (void*)sa, (void*)sb, tmp, (void*)off})
    if (p) cudaFreeAsync(p, st);
  return e;
}

// W1 launch for M <= 1024: R = keys per lane (next power of two of M/32).
template <int kKind>
static cudaError_t launch_w1(int M, long long n, int nxc, const double* a, long long as,
                             const double* b, long long bs, double* terms, cudaStream_t st) {
  if (M < 1) return cudaErrorInvalidValue;
  if (M > 1024) return launch_w1_large<kKind>(M, n, nxc, a, as, b, bs, terms, st);
  const int grid = (int)((n + kW1Cells - 1) / kW1Cells);
  auto go = [&](auto kernel, int R, int nbuf) {
    const size_t smem = sizeof(double) * nbuf * kW1Cells * (32 * R + 32);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel<<<grid, 32 * kW1Cells, smem, st>>>(M, n, nxc, a, as, b, bs, terms);
  };
#define VLBM_W1_K(R) go(k_w1_tile<R, kKind>, R, 2)
  if (M <= 32)
    VLBM_W1_K(1);
  else if (M <= 64)
    VLBM_W1_K(2);
  else if (M <= 128)
    VLBM_W1_K(4);
  else if (M <= 256)
    VLBM_W1_K(8);
  else if (M <= 512)
    VLBM_W1_K(16);
  else
    VLBM_W1_K(32);
#undef VLBM_W1_K
  return cudaGetLastError();
}

cudaError_t launch_w1_planes(int M, int64_t n, const double* a, int64_t as, const double* b,
                             int64_t bs, double* terms, cudaStream_t st) {
  return launch_w1<0>(M, n, 0, a, as, b, bs, terms, st);
}

cudaError_t launch_w1_restrict(int M, int nxc, int nyc, const double* a, int64_t as,
                               const double* f, int64_t fs, double* terms, cudaStream_t st) {
  return launch_w1<1>(M, (long long)nxc * nyc, nxc, a, as, f, fs, terms, st);
}

cudaError_t launch_w1_cells(int M, int64_t n, const double* a, const double* b, double* terms,
                            cudaStream_t st) {
  return launch_w1<2>(M, n, 0, a, 0, b, 0, terms, st);
}

cudaError_t launch_w1_rows(int M, int nxc, int64_t cell0, int64_t n, const double* const* a_rows,
                           const double* const* f_rows, double* terms, cudaStream_t st) {
  return launch_w1<3>(M, n, nxc, reinterpret_cast<const double*>(a_rows), cell0,
                      reinterpret_cast<const double*>(f_rows), 0, terms, st);
}

cudaError_t launch_ordered_mean(int64_t n, const double* terms, double* result, cudaStream_t st) {
  k_ordered_sum<<<1, 256, 0, st>>>(n, terms, nullptr, 1, n, result);
  return cudaGetLastError();
}

// W1 of coarse planes vs the restricted fine planes with the storage-order
// mean overlapped: the cells are processed in K chunks of whole coarse rows
// on `st`; each chunk's part of the sequential sum runs on a second stream
// as soon as its terms exist, continuing the chain of the previous chunk
// (the same additions in the same order), so only the last chunk's part of
// the chain follows the last W1 launch.  result: device scalar.
cudaError_t launch_w1_restrict_mean(int M, int nxc, int nyc, const double* a, int64_t as,
                                    const double* f, int64_t fs, double* terms, double* acc,
                                    double* result, cudaStream_t st) {
  const long long n = (long long)nxc * nyc;
  // chunks of whole rows: 16 by default (VLBM_W1_CHUNKS: 1..16, measurement hook)
  static const int k_env = [] {
    const char* e = getenv("VLBM_W1_CHUNKS");
    const int v = e ? atoi(e) : 16;
    return v >= 1 && v <= 16 ? v : 16;
  }();
  const int K = nyc >= k_env ? k_env : nyc;
  // the second stream and its events: one set per host thread and device
  // (concurrent callers on several GPUs each get their own)
  struct Aux {
    int dev = -1;
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev[17] = {};
  };
  thread_local Aux aux[16];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess && (dev < 0 || dev >= 16)) e = cudaErrorInvalidDevice;
  Aux* ax = e == cudaSuccess ? &aux[dev] : nullptr;
  if (e == cudaSuccess && ax->dev != dev) {
    e = cudaStreamCreateWithFlags(&ax->s2, cudaStreamNonBlocking);
    for (int k = 0; e == cudaSuccess && k < 17; ++k)
      e = cudaEventCreateWithFlags(&ax->ev[k], cudaEventDisableTiming);
    if (e == cudaSuccess) ax->dev = dev;
  }
  cudaStream_t s2 = ax ? ax->s2 : nullptr;
  cudaEvent_t* ev = ax ? ax->ev : nullptr;
  for (int k = 0; e == cudaSuccess && k < K; ++k) {
    const int r0 = (int)((long long)nyc * k / K), r1 = (int)((long long)nyc * (k + 1) / K);
    const long long c0 = (long long)r0 * nxc, cn = (long long)(r1 - r0) * nxc;
    e = launch_w1<1>(M, cn, nxc, a + c0, as, f + 4 * c0, fs, terms + c0, st);
    if (e == cudaSuccess) e = cudaEventRecord(ev[k], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s2, ev[k], 0);
    if (e == cudaSuccess) {
      k_ordered_sum<<<1, 256, 0, s2>>>(cn, terms + c0, acc, k == 0, n,
                                       k == K - 1 ? result : nullptr);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) e = cudaEventRecord(ev[16], s2);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[16], 0);
  return e;
}

cudaError_t launch_moments(int M, int64_t nq, const double* x, int64_t stride, double* mean,
                           double* sd, cudaStream_t st) {
  k_moments<<<grid_for(nq), 256, 0, st>>>(M, nq, x, stride, mean, sd);
  return cudaGetLastError();
}

}  // namespace vlbm_impl
