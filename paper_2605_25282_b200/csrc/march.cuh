// march.cuh — device-side layout and control blocks of a batched VLBM march.
//
// HBM layout (one batch = S independent samples of one nx x ny grid):
//   state[buf][s][20][ny][pitch]  f64, buf in {0,1} (ping-pong per sample):
//       planes 0..3  u        (rho, mom_x, mom_y, E)       solver.hpp:589
//       planes 4+4k+c pops[k] component c, k = 0..3         solver.hpp:590
//   theta[s][ny][pitch]           f64 cell theta of the current step
//   inlet[s][ny][4]               f64 inlet profile rows (host libm)
//   ctl[s]                        per-sample control block (below)
// No ghost cells are stored: the boundary ring is synthesised on load from
// the interior (fill_ghosts semantics, solver.hpp:230-286).
#pragma once
#include <cuda.h>

#include <cstdint>

#include "vlbm_device.cuh"

namespace vlbm_dev {

enum { BC_INLET = 0, BC_OUTFLOW = 1, BC_WALL = 2, BC_PERIODIC = 3 };
enum { LIM_FIRST = 0, LIM_SECOND = 1, LIM_RLMP = 2 };
enum { ST_RUNNING = 0, ST_DIVERGED = 2 };
constexpr int kPlanes = 20;
constexpr int kHardWords = 24;  // u_FO (4), c_w/c_e/c_s/c_n (16), rho_lo/hi, p_lo/hi
constexpr int kBisWords = 13;
constexpr int kUncWords = 28;

// Per-sample control block.  Written by k_sched (one thread per sample) and
// by the advance epilogue (atomics on smax_bits / flags).
struct SampleCtl {
  double t;             // Simulation::time_
  double dt;            // dt of the scheduled step
  double a;             // a = dx / dt of the scheduled step
  double inv2a;         // 0.5 / a, formed once by k_sched (the kernels' per-thread division)
  double smax_inlet;    // max signal speed over the inlet rows (constant)
  unsigned long long smax_bits;  // max interior signal speed (bits; >0 doubles order as u64)
  int bad_signal;       // some cell had a non-finite signal speed (rho<=0, p<=0, NaN)
  int nonfinite;        // some component non-finite after the step
  long long steps;      // Simulation::steps_
  long long budget;     // steps still allowed in this call
  int status;           // ST_RUNNING / ST_DIVERGED
  int active;           // scheduled to step in the current iteration
  int parity;           // buffer holding the current state
  int pad;
};

struct MarchParams {
  int nx, ny, pitch, S;
  long long plane;          // ny * pitch
  long long sample_stride;  // kPlanes * plane
  double* buf0;
  double* buf1;
  double* theta;            // S * plane
  const double* inlet;      // S * ny * 4
  const double* face_tx;    // optional prescribed blending (S x ny x (nx+1))
  const double* face_ty;    // (S x (ny+1) x nx)
  SampleCtl* ctl;
  int* n_active;
  // Global hard-cell queue of the limiter (cells that fail theta = 1): SoA,
  // kHardWords doubles per entry, capacity hq_cap; hq_n is reset by k_sched.
  double* hq;
  long long* hq_idx;  // s * plane + j * pitch + i
  int* hq_n;
  int* hq_next;  // unused slot (hq_n[1]); hq_n[2], hq_n[3]: bisection queue counts
  int hq_cap;
  // Bisection queues (capacity hq_cap each), filled by k_theta_hard:
  //   bq: vertices all certified -- u_FO(4), delta(4), rho_lo/hi, p_lo/hi, thc  (kBisWords);
  //   cq: some uncertified -- u_FO(4), c_f(16), rho_lo/hi, p_lo/hi, thc, p0, err, er (kUncWords)
  //   *_idx: cell index; cq_idx packs the uncertified-vertex mask in bits 40..55
  double* bq;
  long long* bq_idx;
  // Tail queue of k_bisect_unc: lo, hi (2 x hq_cap doubles); tq_idx = cq
  // slot | step << 40.  It aliases the first two word planes of hq and hq_idx
  // (dead once k_theta_hard has run; k_bisect_cert, which may run beside
  // k_bisect_unc on `side`, reads only bq).
  double* tq;
  long long* tq_idx;
  cudaStream_t side;               // k_bisect_cert's stream (joined before the advance)
  cudaEvent_t ev_fork, ev_join;    // fork after k_theta_hard / join after k_bisect_cert
  double* cq;
  long long* cq_idx;
  // Queue statistics (cumulative, never reset): [0] cells finished in place
  // because a queue was full, [1] peak hard cells of one pass, [2] hard cells
  // summed over passes, [3] passes.  Updated by the limiter kernels / k_sched.
  unsigned long long* qstats;
  AuditCtr* audit;    // optional: disagreements of the certified bisection (must stay 0)
  int cert1;     // decide the theta = 1 vertex floors by the quadratic form (rlmp.cuh;
                 // A/B switch VLBM_CERT1, default on; 0: always the exact checks)
  int replay;    // k_bisect_unc replays its bisections from certified classifications
                 // (rlmp_replay.cuh; A/B switch VLBM_REPLAY, default on)
  int persist_ctas;  // grid of the persistent limiter tile pass (this group's share of the GPU)
  // TMA tensor maps [x, y, plane, sample] of buffer 0/1 with the tile boxes of
  // the advance (34x10x20), the limiter's u (36x12x4) and populations (34x10x16).
  CUtensorMap tm_adv[2], tm_thu[2], tm_thp[2];
  double dx, gamma, gm1, alpha, w, safety, kappa, rho_floor_coef, p_floor_coef;
  double rho_ref, p_ref;
  int bc[4];
  int limiter;
  int conservative;
};

}  // namespace vlbm_dev
