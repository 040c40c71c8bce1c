// metrics_ctx.cu — compute_metrics' per (pair, time) reductions with each
// ensemble uploaded ONCE and everything after on the device
// (metrics.hpp:284-300: restrict_field of every fine snapshot, wasserstein1
// of the metric variable, strong_error over all four components).
//
// The caller streams the jointly valid samples in (any batches, sample
// order): each batch's coarse and fine fields are copied to the device once,
// the per-sample strong_error partials (restriction fused, the reference's
// sequential sums) are taken right there, and the metric variable's planes
// are kept in a device store.  finish() then runs W1 over the whole store
// (restriction fused, storage-order mean overlapped: vlbm_d_w1_restrict_mean)
// and the host tail of strong_error.  The fine ensemble is never restricted
// on the host and nothing is uploaded twice.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using vlbm_impl::set_error;

#define CUM(call)                                                                  \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return set_error(VLBM_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

struct vlbm_metrics {
  int M = 0, nxc = 0, nyc = 0, var = 0, device = 0;
  long long nc = 0, nf = 0;
  int B = 0;  // samples per device staging batch
  cudaStream_t st = nullptr;
  double *d_rc = nullptr, *d_rf = nullptr;  // metric-variable planes [M][nc], [M][nf]
  double *d_part = nullptr;                 // strong_error partials [M][10]
  double *d_c = nullptr, *d_f = nullptr;    // staging [B][4][nc], [B][4][nf]
  double *d_terms = nullptr, *d_acc = nullptr, *d_res = nullptr;
  std::vector<char> seen;
};

static void metrics_free(vlbm_metrics* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  for (double* p : {m->d_rc, m->d_rf, m->d_part, m->d_c, m->d_f, m->d_terms, m->d_acc, m->d_res})
    cudaFree(p);
  if (m->st) cudaStreamDestroy(m->st);
  delete m;
}

extern "C" {

int vlbm_metrics_begin(int M, int nxc, int nyc, int var, int device, vlbm_metrics** out) {
  if (!out || M < 1) return set_error(VLBM_E_INVALID, "metrics: no jointly valid samples for pair");
  if (nxc < 1 || nyc < 1) return set_error(VLBM_E_INVALID, "metrics: empty grid");
  if (var < 0 || var > 3) return set_error(VLBM_E_INVALID, "variable must be 0..3");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return set_error(VLBM_E_CUDA, "no CUDA device available (the VLBM path has no CPU fallback)");
  if (device < 0 || device >= n) return set_error(VLBM_E_INVALID, "device index out of range");
  CUM(cudaSetDevice(device));
  auto* m = new vlbm_metrics;
  m->M = M, m->nxc = nxc, m->nyc = nyc, m->var = var, m->device = device;
  m->nc = (long long)nxc * nyc;
  m->nf = 4 * m->nc;
  m->seen.assign(M, 0);
  // staging batch: ~1 GiB of coarse + fine fields
  const long long per = 4 * (m->nc + m->nf) * (long long)sizeof(double);
  m->B = (int)std::max(1ll, std::min((long long)M, (1ll << 30) / per));
  cudaError_t e = cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking);
  auto alloc = [&](double** p, long long n_doubles) {
    if (e == cudaSuccess) e = cudaMalloc(p, sizeof(double) * (size_t)std::max(1ll, n_doubles));
  };
  alloc(&m->d_rc, (long long)M * m->nc);
  alloc(&m->d_rf, (long long)M * m->nf);
  alloc(&m->d_part, 10ll * M);
  alloc(&m->d_c, 4ll * m->B * m->nc);
  alloc(&m->d_f, 4ll * m->B * m->nf);
  alloc(&m->d_terms, m->nc);
  alloc(&m->d_acc, 1);
  alloc(&m->d_res, 1);
  if (e != cudaSuccess) {
    metrics_free(m);
    return set_error(VLBM_E_NOMEM, std::string("metrics: device buffers: ") + cudaGetErrorString(e));
  }
  *out = m;
  return VLBM_OK;
}

// Samples first .. first+count-1 of the jointly valid set: coarse fields
// [count][4][nyc][nxc] and fine fields [count][4][2nyc][2nxc] (host).
int vlbm_metrics_add(vlbm_metrics* m, int first, int count, const double* coarse,
                     const double* fine) {
  if (!m || !coarse || !fine) return set_error(VLBM_E_INVALID, "null argument");
  if (first < 0 || count < 0 || first + count > m->M)
    return set_error(VLBM_E_INVALID, "metrics: sample range out of bounds");
  CUM(cudaSetDevice(m->device));
  for (int b0 = 0; b0 < count; b0 += m->B) {
    const int nb = std::min(m->B, count - b0);
    CUM(cudaMemcpyAsync(m->d_c, coarse + 4 * m->nc * (long long)b0, sizeof(double) * 4 * m->nc * nb,
                        cudaMemcpyHostToDevice, m->st));
    CUM(cudaMemcpyAsync(m->d_f, fine + 4 * m->nf * (long long)b0, sizeof(double) * 4 * m->nf * nb,
                        cudaMemcpyHostToDevice, m->st));
    CUM(vlbm_impl::launch_strong_partials_fused(nb, m->nxc, m->nyc, m->d_c, m->d_f,
                                                m->d_part + 10ll * (first + b0), m->st));
    // the metric variable's planes into the W1 store (plane var of each sample)
    CUM(cudaMemcpy2DAsync(m->d_rc + m->nc * (long long)(first + b0), sizeof(double) * m->nc,
                          m->d_c + m->var * m->nc, sizeof(double) * 4 * m->nc,
                          sizeof(double) * m->nc, nb, cudaMemcpyDeviceToDevice, m->st));
    CUM(cudaMemcpy2DAsync(m->d_rf + m->nf * (long long)(first + b0), sizeof(double) * m->nf,
                          m->d_f + m->var * m->nf, sizeof(double) * 4 * m->nf,
                          sizeof(double) * m->nf, nb, cudaMemcpyDeviceToDevice, m->st));
    for (int s = 0; s < nb; ++s) m->seen[first + b0 + s] = 1;
  }
  CUM(cudaStreamSynchronize(m->st));  // the caller may reuse its buffers
  return VLBM_OK;
}

int vlbm_metrics_finish(vlbm_metrics* m, double* w1, double* e_strong, double* per_component) {
  if (!m || !w1 || !e_strong) return set_error(VLBM_E_INVALID, "null argument");
  for (char c : m->seen)
    if (!c) return set_error(VLBM_E_INVALID, "metrics: not every sample was added");
  CUM(cudaSetDevice(m->device));
  CUM(vlbm_impl::launch_w1_restrict_mean(m->M, m->nxc, m->nyc, m->d_rc, m->nc, m->d_rf, m->nf,
                                         m->d_terms, m->d_acc, m->d_res, m->st));
  std::vector<double> part(10 * (size_t)m->M);
  CUM(cudaMemcpyAsync(part.data(), m->d_part, sizeof(double) * part.size(),
                      cudaMemcpyDeviceToHost, m->st));
  CUM(cudaMemcpyAsync(w1, m->d_res, sizeof(double), cudaMemcpyDeviceToHost, m->st));
  CUM(cudaStreamSynchronize(m->st));
  return vlbm_strong_finish(m->M, part.data(), e_strong, per_component);
}

void vlbm_metrics_destroy(vlbm_metrics* m) { metrics_free(m); }

}  // extern "C"
