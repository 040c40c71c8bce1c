// internal.h — shared declarations between the C-ABI (capi.cu), the host IC
// (host_ic.cpp) and the kernel launchers (march.cu, post.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "vlbm_b200.h"

namespace vlbm_dev {
struct MarchParams;
}

namespace vlbm_impl {

int set_error(int code, const std::string& msg);

// ---- host IC (host_ic.cpp): same libm as the reference on this image ----
double grid_dx(const vlbm_grid& g);
double y_center(const vlbm_grid& g, int j);
int validate_grid(const vlbm_grid& g);
int validate_params(const vlbm_params& p);
int validate_perturbation(const vlbm_perturbation& pp);
void inlet_state(double y, int K, const double* yc, const double* zc,
                 const vlbm_perturbation& pp, double gamma, double* out);
// initial_field (perturbation.hpp:106-122) into 4 planes of ny x nx.
void initial_field(const vlbm_grid& g, int K, const double* yc, const double* zc,
                   const vlbm_perturbation& pp, double gamma, double strip, double* out);
// Leading wedge cells of initial_field per row (counts[ny]).
void wedge_counts(const vlbm_grid& g, double strip, int* counts);

// ---- march launchers (march.cu) -------------------------------------------
cudaError_t launch_signal(const vlbm_dev::MarchParams& P, cudaStream_t st);
cudaError_t launch_init(const vlbm_dev::MarchParams& P, double* d_a0, cudaStream_t st);
// initial_field on the device from the uploaded inlet rows and wedge counts
// (state buffer 0): ambient amb[4] except u_in(y_j) on cells i < counts[j].
cudaError_t launch_init_field(const vlbm_dev::MarchParams& P, const int* counts,
                              const double* amb4, cudaStream_t st);
cudaError_t launch_sched(const vlbm_dev::MarchParams& P, double target, double fixed_dt,
                         cudaStream_t st);
// part 0: the tile pass (u_FO, bounds, feasible(1), hard-cell queue);
// part 1: the hard cells (closed-form cap, certified bisections).
cudaError_t launch_theta(const vlbm_dev::MarchParams& P, cudaStream_t st, int part);
// mode 0: cell theta plane, 1: constant theta, 2: prescribed faces
cudaError_t launch_advance(const vlbm_dev::MarchParams& P, int mode, double const_theta,
                           cudaStream_t st);
// tiled production kernels (march_tiled.cu)
int encode_tensor_maps(vlbm_dev::MarchParams& P);
cudaError_t launch_theta_tiled(const vlbm_dev::MarchParams& P, cudaStream_t st);
cudaError_t launch_theta_hard(const vlbm_dev::MarchParams& P, cudaStream_t st);
// Resident k_theta_tiled CTAs per SM (occupancy of the persistent tile pass).
int theta_ctas_per_sm();
// Tiles of k_theta_tiled's grid (32 x VLBM_THETA_TY cells, one warp per row)
// per sample.
#ifndef VLBM_THETA_TY
#define VLBM_THETA_TY 8
#endif
inline int theta_tiles(int nx, int ny) {
  return ((nx + 31) / 32) * ((ny + VLBM_THETA_TY - 1) / VLBM_THETA_TY);
}
cudaError_t launch_advance_tiled(const vlbm_dev::MarchParams& P, int mode, double const_theta,
                                 cudaStream_t st);
cudaError_t launch_set_budget(const vlbm_dev::MarchParams& P, long long budget,
                              cudaStream_t st);

// ---- post-processing launchers (post.cu) ----------------------------------
cudaError_t launch_restrict(int M, int nxc, int nyc, const double* fine, double* coarse,
                            cudaStream_t st);
cudaError_t launch_restrict_var(int M, int nxc, int nyc, const double* fine, int var, double* out,
                                cudaStream_t st);
// per-sample sequential L1 partials (num, den, cnum[4], cden[4]) -> M x 10
cudaError_t launch_strong_partials(int M, int64_t n, const double* a, const double* b,
                                   double* partials, cudaStream_t st);
// one variable, fused restriction: coarse(m, c) = coarse[m*c_stride + c],
// fine plane of sample m at fine + m*f_stride
cudaError_t launch_strong_partials_var(int M, int nxc, int nyc, const double* coarse,
                                       int64_t c_stride, const double* fine, int64_t f_stride,
                                       double* partials, cudaStream_t st);
cudaError_t launch_strong_partials_fused(int M, int nxc, int nyc, const double* coarse,
                                         const double* fine, double* partials, cudaStream_t st);
cudaError_t launch_w1_planes(int M, int64_t n, const double* a, int64_t a_sample_stride,
                             const double* b, int64_t b_sample_stride, double* terms,
                             cudaStream_t st);
cudaError_t launch_w1_restrict(int M, int nxc, int nyc, const double* coarse,
                               int64_t c_sample_stride, const double* fine,
                               int64_t f_sample_stride, double* terms, cudaStream_t st);
cudaError_t launch_w1_cells(int M, int64_t n, const double* a, const double* b, double* terms,
                            cudaStream_t st);
// row tables: sample m's coarse plane at a_rows[m], fine plane at f_rows[m]
// (any GPU, peer-mapped), cells [cell0, cell0 + n) of the coarse grid
cudaError_t launch_w1_rows(int M, int nxc, int64_t cell0, int64_t n, const double* const* a_rows,
                           const double* const* f_rows, double* terms, cudaStream_t st);
cudaError_t launch_ordered_mean(int64_t n, const double* terms, double* result, cudaStream_t st);
// W1 (fused restriction) with the storage-order mean overlapped chunk by chunk
// on an internal stream; terms: n cells, acc: one device double of scratch
cudaError_t launch_w1_restrict_mean(int M, int nxc, int nyc, const double* coarse,
                                    int64_t c_sample_stride, const double* fine,
                                    int64_t f_sample_stride, double* terms, double* acc,
                                    double* result, cudaStream_t st);
// nq entries per sample: x(m, q) = x[m * sample_stride + q]
cudaError_t launch_moments(int M, int64_t nq, const double* x, int64_t sample_stride,
                           double* mean, double* stddev, cudaStream_t st);

}  // namespace vlbm_impl
