// capi.cu — the C ABI of include/vlbm_b200.h: batch lifecycle, the host
// side of the run_sample loop (device-resident scheduling, host polls one
// int per chunk of steps), and the post-processing entry points.
//
// There is no CPU fallback: every numeric result below is produced by the
// sm_100a kernels in march.cu / post.cu; a CUDA failure is reported as
// VLBM_E_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "march.cuh"

using vlbm_dev::MarchParams;
using vlbm_dev::SampleCtl;

namespace vlbm_impl {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace vlbm_impl

using vlbm_impl::set_error;

#define CU(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return set_error(VLBM_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

struct vlbm_batch {
  vlbm_grid g{};
  vlbm_params p{};
  int S = 0;
  int device = 0;
  MarchParams P{};
  cudaStream_t stream = nullptr;
  int* h_active = nullptr;  // pinned
  double* d_a0 = nullptr;
  double* d_face_tx = nullptr;
  double* d_face_ty = nullptr;
  // stats
  bool timing = false;
  long long launches = 0;
  double ms_kind[4] = {0, 0, 0, 0};  // sched, limiter tile pass, advance, limiter hard path
  std::vector<cudaEvent_t> ev;  // pool of events, pairs per timed launch
  std::vector<int> ev_kind;     // index into ms_kind
  std::vector<cudaStream_t> ev_stream;
  int ev_used = 0;
  // sample groups (march views), see alloc_batch
  int G = 1;
  std::vector<MarchParams> Pg;
  std::vector<cudaStream_t> sg;  // sg[0] == stream
  std::vector<int> g0;           // first sample of each group
  int* d_active_g = nullptr;
  int* h_active_g = nullptr;     // pinned
  cudaEvent_t ev_fork = nullptr;
  bool cert_side = true;  // k_bisect_cert on a side stream (VLBM_CERT_SIDE=0: in line)
  // serial sample groups: the groups share the batch's stream and ONE set of
  // limiter queues (allocated by group 0), marched one after another
  bool serial = false;
  unsigned long long* d_qstats = nullptr;
  bool graphs = true;  // chunks after the first replay as a CUDA graph (VLBM_GRAPHS=0: off)
};

namespace {

int check_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return set_error(VLBM_E_CUDA, std::string("no CUDA device available (the VLBM path has no "
                                              "CPU fallback): ") +
                                      cudaGetErrorString(e));
  if (device < 0 || device >= n) return set_error(VLBM_E_INVALID, "device index out of range");
  CU(cudaSetDevice(device));
  return VLBM_OK;
}

void free_batch(vlbm_batch* b) {
  if (!b) return;
  cudaSetDevice(b->device);
  cudaFree(b->P.buf0);
  cudaFree(b->P.buf1);
  cudaFree(b->P.theta);
  cudaFree(const_cast<double*>(b->P.inlet));
  cudaFree(b->P.ctl);
  cudaFree(b->P.n_active);
  cudaFree(b->d_a0);
  for (size_t g = 0; g < b->Pg.size(); ++g) {
    MarchParams& Q = b->Pg[g];
    if (b->serial && g > 0) continue;  // queues, side stream and events belong to group 0
    cudaFree(Q.hq);
    cudaFree(Q.hq_idx);
    cudaFree(Q.hq_n);
    cudaFree(Q.bq);
    cudaFree(Q.bq_idx);
    if (Q.side) cudaStreamDestroy(Q.side);
    if (Q.ev_fork) cudaEventDestroy(Q.ev_fork);
    if (Q.ev_join) cudaEventDestroy(Q.ev_join);
    cudaFree(Q.cq);
    cudaFree(Q.cq_idx);
    if (g > 0 && b->sg[g]) cudaStreamDestroy(b->sg[g]);
  }
  cudaFree(b->d_active_g);
  cudaFree(b->d_qstats);
  if (b->h_active_g) cudaFreeHost(b->h_active_g);
  if (b->ev_fork) cudaEventDestroy(b->ev_fork);
  cudaFree(b->d_face_tx);
  cudaFree(b->d_face_ty);
  cudaFree(b->P.audit);
  if (b->h_active) cudaFreeHost(b->h_active);
  for (cudaEvent_t e : b->ev) cudaEventDestroy(e);
  if (b->stream) cudaStreamDestroy(b->stream);
  delete b;
}

// Allocates the batch and its device arrays; fields/inlet uploaded by caller.
int alloc_batch(const vlbm_grid* g, const vlbm_params* p, int S, int device, vlbm_batch** out) {
  if (!g || !p || !out) return set_error(VLBM_E_INVALID, "null argument");
  if (S < 1) return set_error(VLBM_E_INVALID, "n_samples must be >= 1");
  if (int rc = vlbm_impl::validate_grid(*g)) return rc;
  if (int rc = vlbm_impl::validate_params(*p)) return rc;
  if (int rc = check_device(device)) return rc;
  auto* b = new vlbm_batch;
  b->g = *g;
  b->p = *p;
  b->S = S;
  b->device = device;
  MarchParams& P = b->P;
  P.nx = g->nx;
  P.ny = g->ny;
  P.pitch = (g->nx + 15) / 16 * 16;  // 128-byte rows: TMA strides and coalescing
  P.S = S;
  P.plane = (long long)P.ny * P.pitch;
  P.sample_stride = vlbm_dev::kPlanes * P.plane;
  P.dx = vlbm_impl::grid_dx(*g);
  P.gamma = p->gamma;
  P.gm1 = p->gamma - 1.0;
  P.alpha = p->alpha;
  P.w = 0.25 * (1.0 - p->alpha);
  P.safety = p->safety;
  P.kappa = p->rlmp_relaxation;
  P.rho_ref = p->rho_ref;
  P.p_ref = p->p_ref;
  P.rho_floor_coef = p->positivity_floor * p->rho_ref;  // rlmp_bounds, solver.hpp:413-414
  P.p_floor_coef = p->positivity_floor * p->p_ref;
  for (int k = 0; k < 4; ++k) P.bc[k] = p->bc[k];
  P.limiter = p->limiter;
  P.conservative = p->conservative_bound;
  const size_t state_bytes = sizeof(double) * (size_t)S * P.sample_stride;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t need = 2 * state_bytes + sizeof(double) * (size_t)S * P.plane +
                      sizeof(double) * (size_t)S * P.ny * 4 + sizeof(SampleCtl) * S;
  if (need + (size_t)(256ull << 20) > free_b) {
    delete b;
    return set_error(VLBM_E_NOMEM, "batch needs " + std::to_string(need >> 20) + " MiB, " +
                                       std::to_string(free_b >> 20) + " MiB free");
  }
  int rc = VLBM_OK;
  auto chk = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == VLBM_OK)
      rc = set_error(VLBM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  chk(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking), "stream");
  chk(cudaMalloc(&P.buf0, state_bytes), "malloc state0");
  chk(cudaMalloc(&P.buf1, state_bytes), "malloc state1");
  chk(cudaMalloc(&P.theta, sizeof(double) * (size_t)S * P.plane), "malloc theta");
  double* inlet = nullptr;
  chk(cudaMalloc(&inlet, sizeof(double) * (size_t)S * P.ny * 4), "malloc inlet");
  P.inlet = inlet;
  chk(cudaMalloc(&P.ctl, sizeof(SampleCtl) * S), "malloc ctl");
  chk(cudaMalloc(&P.n_active, sizeof(int)), "malloc n_active");
  chk(cudaMalloc(&b->d_a0, sizeof(double) * S), "malloc a0");
  chk(cudaMallocHost(&b->h_active, sizeof(int)), "malloc host");
  // Sample groups (below): the march runs G views of the batch (disjoint
  // sample ranges: offset pointers, own control slice, tensor maps, counter).
  P.cert1 = 1;
  if (const char* e = getenv("VLBM_CERT1")) P.cert1 = atoi(e) != 0;
  P.replay = 1;
  if (const char* e = getenv("VLBM_REPLAY")) P.replay = atoi(e) != 0;
  if ((size_t)S * vlbm_impl::theta_tiles(P.nx, P.ny) > (size_t)INT_MAX)
    rc = set_error(VLBM_E_INVALID, "too many tiles for one batch");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (const char* e = getenv("VLBM_GRAPHS")) b->graphs = atoi(e) != 0;
  if (const char* e = getenv("VLBM_CERT_SIDE")) b->cert_side = atoi(e) != 0;
  const bool rlmp = p->limiter == VLBM_LIMITER_RLMP;
  // Limiter queues: per hard cell kHardWords (hq) + kBisWords (bq) +
  // kUncWords (cq) doubles and three indices; the tail queue aliases hq.
  const size_t entry =
      sizeof(double) * (vlbm_dev::kHardWords + vlbm_dev::kBisWords + vlbm_dev::kUncWords) +
      3 * sizeof(long long);
  const size_t avail =
      free_b > need + (size_t)(2ull << 30) ? free_b - need - (size_t)(2ull << 30) : 0;
  const size_t qbudget = avail / 2;  // the other half stays free for the caller
  const size_t cells_per_sample = (size_t)P.nx * P.ny;
  // Sample groups.  Serial (the default when needed): when one set of queues
  // covering every cell of the batch does not fit in qbudget, the batch is
  // marched as G groups of samples, one after another on the batch's stream,
  // sharing one set of queues that covers every cell of a group -- so no
  // hard cell ever overflows (configs[2]: 125 samples of 4000x800).
  // VLBM_SERIAL_GROUPS forces G (tests).  Concurrent (VLBM_GROUPS, an A/B
  // switch: 2-4 groups measured 0.7-1.6 % slower since the replay): each
  // group on its own stream with its own share of the queues.
  int G = 1;
  if (rlmp) {
    if (const char* e = getenv("VLBM_SERIAL_GROUPS")) {
      G = std::max(1, std::min(S, atoi(e)));
    } else {
      while (G < S && (size_t)((S + G - 1) / G) * cells_per_sample * entry > qbudget) ++G;
    }
    b->serial = G > 1;
  }
  if (!b->serial)
    if (const char* e = getenv("VLBM_GROUPS")) G = std::max(1, std::min(S, atoi(e)));
  b->G = G;
  chk(cudaMalloc(&b->d_active_g, sizeof(int) * G), "malloc active_g");
  chk(cudaMallocHost(&b->h_active_g, sizeof(int) * G), "malloc host active_g");
  chk(cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming), "event");
  chk(cudaMalloc(&b->d_qstats, 4 * sizeof(unsigned long long)), "malloc qstats");
  if (rc == VLBM_OK) chk(cudaMemset(b->d_qstats, 0, 4 * sizeof(unsigned long long)), "memset");
  P.qstats = b->d_qstats;
  for (int g = 0; g < G && rc == VLBM_OK; ++g) {
    const int s0 = (int)((long long)S * g / G), s1 = (int)((long long)S * (g + 1) / G);
    MarchParams Q = P;
    Q.S = s1 - s0;
    Q.ctl = P.ctl + s0;
    Q.buf0 = P.buf0 + (size_t)s0 * P.sample_stride;
    Q.buf1 = P.buf1 + (size_t)s0 * P.sample_stride;
    Q.theta = P.theta + (size_t)s0 * P.plane;
    Q.inlet = P.inlet + (size_t)s0 * P.ny * 4;
    Q.n_active = b->d_active_g + g;
    Q.persist_ctas = std::max(1, sms * vlbm_impl::theta_ctas_per_sm() / (b->serial ? 1 : G));
    cudaStream_t sg = b->stream;
    if (g > 0 && !b->serial) chk(cudaStreamCreateWithFlags(&sg, cudaStreamNonBlocking), "stream g");
    if (rlmp && b->serial && g > 0) {
      const MarchParams& Q0 = b->Pg[0];  // the shared queues
      Q.hq = Q0.hq, Q.hq_idx = Q0.hq_idx, Q.hq_n = Q0.hq_n, Q.hq_next = Q0.hq_next;
      Q.hq_cap = Q0.hq_cap;
      Q.bq = Q0.bq, Q.bq_idx = Q0.bq_idx, Q.tq = Q0.tq, Q.tq_idx = Q0.tq_idx;
      Q.cq = Q0.cq, Q.cq_idx = Q0.cq_idx;
      Q.side = Q0.side, Q.ev_fork = Q0.ev_fork, Q.ev_join = Q0.ev_join;
    } else if (rlmp) {
      const int Sg = b->serial ? (S + G - 1) / G : Q.S;
      size_t cap = (size_t)Sg * cells_per_sample;
      const size_t share = b->serial ? qbudget : qbudget / G;
      if (cap * entry > share) cap = share / entry;
      if (cap > (size_t)INT_MAX / 2) cap = (size_t)INT_MAX / 2;
      if (const char* e = getenv("VLBM_HQ_CAP"))  // test hook: exercise the overflow paths
        cap = std::min(cap, (size_t)std::max(0ll, atoll(e)));
      // even thirds of whole kHB chunks (16-B aligned bulk copies): rounded up
      // when memory allows, so a queue meant to cover a group's cells does
      cap = (cap + 767) / 768 * 768 * entry <= share ? (cap + 767) / 768 * 768 : cap / 768 * 768;
      if (cap >= 1024) {
        Q.hq_cap = (int)cap;
        chk(cudaMalloc(&Q.hq, sizeof(double) * vlbm_dev::kHardWords * cap), "malloc hq");
        chk(cudaMalloc(&Q.hq_idx, sizeof(long long) * cap), "malloc hq_idx");
        chk(cudaMalloc(&Q.bq, sizeof(double) * vlbm_dev::kBisWords * cap), "malloc bq");
        chk(cudaMalloc(&Q.bq_idx, sizeof(long long) * cap), "malloc bq_idx");
        Q.tq = Q.hq;  // aliases: hq is dead once k_theta_hard has run
        Q.tq_idx = Q.hq_idx;
        if (b->cert_side) {
          chk(cudaStreamCreateWithFlags(&Q.side, cudaStreamNonBlocking), "stream side");
          chk(cudaEventCreateWithFlags(&Q.ev_fork, cudaEventDisableTiming), "event");
          chk(cudaEventCreateWithFlags(&Q.ev_join, cudaEventDisableTiming), "event");
        }
        chk(cudaMalloc(&Q.cq, sizeof(double) * vlbm_dev::kUncWords * cap), "malloc cq");
        chk(cudaMalloc(&Q.cq_idx, sizeof(long long) * cap), "malloc cq_idx");
        // counters: [0] hard cells, [2] bq, [3..5] cq bins, [6] limiter tile claims, [7] tail
        chk(cudaMalloc(&Q.hq_n, 8 * sizeof(int)), "malloc hq_n");
        Q.hq_next = Q.hq_n + 1;
        if (rc == VLBM_OK) chk(cudaMemset(Q.hq_n, 0, 8 * sizeof(int)), "memset hq_n");
      }
    }
    if (rc == VLBM_OK) rc = vlbm_impl::encode_tensor_maps(Q);
    b->Pg.push_back(Q);
    b->sg.push_back(sg);
    b->g0.push_back(s0);
  }
  if (rc == VLBM_OK) rc = vlbm_impl::encode_tensor_maps(P);
  if (rc == VLBM_OK) {
    chk(cudaMemsetAsync(P.buf0, 0, state_bytes, b->stream), "memset");
    chk(cudaMemsetAsync(P.buf1, 0, state_bytes, b->stream), "memset");
    chk(cudaMemsetAsync(P.theta, 0, sizeof(double) * (size_t)S * P.plane, b->stream), "memset");
    chk(cudaMemsetAsync(inlet, 0, sizeof(double) * (size_t)S * P.ny * 4, b->stream), "memset");
    std::vector<SampleCtl> ctl(S);
    std::memset(ctl.data(), 0, sizeof(SampleCtl) * S);
    for (auto& c : ctl) c.status = vlbm_dev::ST_RUNNING;
    chk(cudaMemcpyAsync(P.ctl, ctl.data(), sizeof(SampleCtl) * S, cudaMemcpyHostToDevice,
                        b->stream),
        "upload ctl");
    chk(cudaStreamSynchronize(b->stream), "sync");
  }
  if (rc != VLBM_OK) {
    free_batch(b);
    return rc;
  }
  *out = b;
  return VLBM_OK;
}

int upload_sample(vlbm_batch* b, int s, const double* field, const double* inlet_rows) {
  const MarchParams& P = b->P;
  const size_t n = (size_t)P.nx * P.ny;
  double* dst = P.buf0 + (size_t)s * P.sample_stride;
  for (int k = 0; k < 4; ++k)
    CU(cudaMemcpy2DAsync(dst + k * P.plane, sizeof(double) * P.pitch, field + k * n,
                         sizeof(double) * P.nx, sizeof(double) * P.nx, P.ny,
                         cudaMemcpyHostToDevice, b->stream));
  if (inlet_rows)
    CU(cudaMemcpyAsync(const_cast<double*>(P.inlet) + (size_t)s * P.ny * 4, inlet_rows,
                       sizeof(double) * P.ny * 4, cudaMemcpyHostToDevice, b->stream));
  return VLBM_OK;
}

// Constructor tail: kinetic speed of the initial field, a0, pops = M(u, a0).
int finish_create(vlbm_batch* b) {
  CU(vlbm_impl::launch_signal(b->P, b->stream));
  CU(vlbm_impl::launch_init(b->P, b->d_a0, b->stream));
  b->launches += 3;
  CU(cudaStreamSynchronize(b->stream));
  return VLBM_OK;
}

// Kernel timing (CUDA events around each launch on its own stream).  With
// several sample groups the per-kind sums add the groups' (overlapping)
// kernel times.
void record(vlbm_batch* b, int kind, cudaStream_t st) {
  if (!b->timing) return;
  while ((int)b->ev.size() < 2 * (b->ev_used + 1)) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    b->ev.push_back(e);
  }
  if ((int)b->ev_kind.size() < b->ev_used + 1) {
    b->ev_kind.resize(b->ev_used + 1);
    b->ev_stream.resize(b->ev_used + 1);
  }
  b->ev_kind[b->ev_used] = kind;
  b->ev_stream[b->ev_used] = st;
  cudaEventRecord(b->ev[2 * b->ev_used], st);
}
void record_end(vlbm_batch* b) {
  if (!b->timing) return;
  cudaEventRecord(b->ev[2 * b->ev_used + 1], b->ev_stream[b->ev_used]);
  ++b->ev_used;
}
void harvest(vlbm_batch* b) {
  for (int q = 0; q < b->ev_used; ++q) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, b->ev[2 * q], b->ev[2 * q + 1]);
    b->ms_kind[b->ev_kind[q]] += ms;
  }
  b->ev_used = 0;
}

// The run_sample while-loop for every sample (solver.hpp:645-658), device
// scheduled: chunks of `chunk` iterations [sched, theta, advance] are issued,
// then the host reads the number of samples the last k_sched scheduled; 0
// means every sample has reached the target (or diverged / used its budget)
// and every step taken is finalised.
int march_loop(vlbm_batch* b, double target, double fixed_dt, int mode, int chunk) {
  const bool rlmp = b->p.limiter == VLBM_LIMITER_RLMP && mode == 0;
  const int adv_mode = mode == 2 ? 2 : (rlmp ? 0 : 1);
  const double const_theta = b->p.limiter == VLBM_LIMITER_SECOND_ORDER ? 1.0 : 0.0;
  const int G = b->G;
  auto issue = [&](int n) -> int {
    // fork: the group streams start after everything queued on the main stream
    if (G > 1 && !b->serial) {
      CU(cudaEventRecord(b->ev_fork, b->stream));
      for (int g = 1; g < G; ++g) CU(cudaStreamWaitEvent(b->sg[g], b->ev_fork, 0));
    }
    for (int it = 0; it < n; ++it) {
      for (int g = 0; g < G; ++g) {  // groups interleaved: their kernels overlap
        const MarchParams& Q = b->Pg[g];
        cudaStream_t st = b->sg[g];
        record(b, 0, st);
        CU(vlbm_impl::launch_sched(Q, target, fixed_dt, st));
        record_end(b);
        if (rlmp) {
          record(b, 1, st);
          CU(vlbm_impl::launch_theta(Q, st, 0));
          record_end(b);
          record(b, 3, st);
          CU(vlbm_impl::launch_theta(Q, st, 1));
          record_end(b);
        }
        record(b, 2, st);
        CU(vlbm_impl::launch_advance(Q, adv_mode, const_theta, st));
        record_end(b);
        b->launches += rlmp ? (Q.hq ? (Q.replay ? 7 : 6) : 3) : 2;
      }
    }
    return VLBM_OK;
  };
  // From the second chunk of a call on, the chunk's launches replay as one
  // CUDA graph (captured once per call: the kernel arguments are fixed for
  // the call, the per-step state lives on the device). Not while per-launch
  // timing is on (its events are harvested on the host) or with several
  // sample groups.
  const bool use_graph = b->graphs && !b->timing && (G == 1 || b->serial);
  cudaGraphExec_t exec = nullptr;
  int exec_chunk = -1;
  long long exec_launches = 0;
  int rc = VLBM_OK;
  for (int pass = 0;; ++pass) {
    if (use_graph && pass > 0) {
      if (exec_chunk != chunk) {
        if (exec) cudaGraphExecDestroy(exec);
        exec = nullptr;
        const long long l0 = b->launches;
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamBeginCapture(b->stream, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) {
          rc = set_error(VLBM_E_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
          break;
        }
        const int ri = issue(chunk);
        e = cudaStreamEndCapture(b->stream, &graph);
        if (ri != VLBM_OK) {
          if (graph) cudaGraphDestroy(graph);
          rc = ri;
          break;
        }
        if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
        if (graph) cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
          exec = nullptr;
          rc = set_error(VLBM_E_CUDA, std::string("CUDA graph capture: ") + cudaGetErrorString(e));
          break;
        }
        exec_launches = b->launches - l0;
        b->launches = l0;
        exec_chunk = chunk;
      }
      cudaError_t e = cudaGraphLaunch(exec, b->stream);
      if (e != cudaSuccess) {
        rc = set_error(VLBM_E_CUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
        break;
      }
      b->launches += exec_launches;
    } else if ((rc = issue(chunk)) != VLBM_OK) {
      break;
    }
    cudaError_t e = cudaSuccess;
    for (int g = 0; g < G && e == cudaSuccess; ++g)
      e = cudaMemcpyAsync(b->h_active_g + g, b->Pg[g].n_active, sizeof(int),
                          cudaMemcpyDeviceToHost, b->sg[g]);
    for (int g = 0; g < G && e == cudaSuccess; ++g)
      if (g == 0 || !b->serial) e = cudaStreamSynchronize(b->sg[g]);
    if (e != cudaSuccess) {
      rc = set_error(VLBM_E_CUDA, std::string("march poll: ") + cudaGetErrorString(e));
      break;
    }
    if (b->timing) harvest(b);
    int active = 0;
    for (int g = 0; g < G; ++g) active += b->h_active_g[g];
    if (active == 0) break;
    if (mode == 2) chunk = 1;
  }
  if (exec) cudaGraphExecDestroy(exec);
  return rc;
}

int read_ctl(vlbm_batch* b, std::vector<SampleCtl>& ctl) {
  ctl.resize(b->S);
  CU(cudaMemcpyAsync(ctl.data(), b->P.ctl, sizeof(SampleCtl) * b->S, cudaMemcpyDeviceToHost,
                     b->stream));
  CU(cudaStreamSynchronize(b->stream));
  return VLBM_OK;
}

}  // namespace

extern "C" {

int vlbm_abi_version(void) { return VLBM_ABI_VERSION; }
int vlbm_device_count(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}
const char* vlbm_last_error(void) { return vlbm_impl::g_last_error.c_str(); }

int vlbm_batch_create(const vlbm_grid* g, const vlbm_params* p, const vlbm_perturbation* pp,
                      uint64_t base_seed, int64_t m0, int n_samples, double strip_width,
                      int device, vlbm_batch** out) {
  if (!pp) return set_error(VLBM_E_INVALID, "null perturbation");
  if (int rc = vlbm_impl::validate_perturbation(*pp)) return rc;
  if (n_samples < 1) return set_error(VLBM_E_INVALID, "n_samples must be >= 1");
  const int K = pp->modes;
  std::vector<double> yc((size_t)K * n_samples), zc((size_t)K * n_samples);
  for (int s = 0; s < n_samples; ++s)
    vlbm_draw_coefficients(base_seed, (uint64_t)(m0 + s), K, yc.data() + (size_t)K * s,
                           zc.data() + (size_t)K * s);
  return vlbm_batch_create_coeffs(g, p, pp, n_samples, yc.data(), zc.data(), strip_width, device,
                                  out);
}

int vlbm_batch_create_coeffs(const vlbm_grid* g, const vlbm_params* p,
                             const vlbm_perturbation* pp, int n_samples, const double* y_all,
                             const double* z_all, double strip_width, int device,
                             vlbm_batch** out) {
  if (!pp || !y_all || !z_all) return set_error(VLBM_E_INVALID, "null argument");
  if (int rc = vlbm_impl::validate_perturbation(*pp)) return rc;
  if (strip_width < 0.0) return set_error(VLBM_E_INVALID, "config: inlet_strip_width must be >= 0");
  // run_sample's construction (solver.hpp:633-640): jet boundaries and
  // set_reference(rho_amb, p_amb).
  vlbm_params q = *p;
  q.bc[0] = VLBM_BC_INLET;
  q.bc[1] = VLBM_BC_OUTFLOW;
  q.bc[2] = VLBM_BC_WALL;
  q.bc[3] = VLBM_BC_WALL;
  q.rho_ref = pp->rho_amb;
  q.p_ref = pp->p_amb;
  vlbm_batch* b = nullptr;
  if (int rc = alloc_batch(g, &q, n_samples, device, &b)) return rc;
  // The inlet rows u_in(y_j) of every sample on the host (the reference's
  // libm: perturbation.hpp:87-95), threads over samples; the initial field
  // (ambient + the wedge of those rows) is then laid out on the device.
  const int K = pp->modes;
  const size_t nrow = 4 * (size_t)g->ny;
  double* rows = nullptr;
  if (cudaMallocHost(&rows, sizeof(double) * nrow * n_samples) != cudaSuccess) {
    free_batch(b);
    return set_error(VLBM_E_NOMEM, "pinned staging buffer");
  }
  auto fill = [&](int s0, int s1) {
    for (int s = s0; s < s1; ++s)
      for (int j = 0; j < g->ny; ++j)
        vlbm_impl::inlet_state(vlbm_impl::y_center(*g, j), K, y_all + (size_t)K * s,
                               z_all + (size_t)K * s, *pp, q.gamma, rows + nrow * s + 4 * j);
  };
  const long long work = (long long)n_samples * g->ny;
  int nt = work < 20000 ? 1
                        : (int)std::min(std::max(1u, std::thread::hardware_concurrency()), 16u);
  nt = std::min(nt, n_samples);
  if (nt <= 1) {
    fill(0, n_samples);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back(fill, (int)((long long)n_samples * t / nt),
                      (int)((long long)n_samples * (t + 1) / nt));
    for (auto& x : th) x.join();
  }
  std::vector<int> counts(g->ny);
  vlbm_impl::wedge_counts(*g, strip_width, counts.data());
  const double amb[4] = {pp->rho_amb, 0.0, 0.0, pp->p_amb / (q.gamma - 1.0)};  // ambient_state
  int* d_counts = nullptr;
  int rc = VLBM_OK;
  auto chk = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == VLBM_OK)
      rc = set_error(VLBM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  chk(cudaMemcpyAsync(const_cast<double*>(b->P.inlet), rows, sizeof(double) * nrow * n_samples,
                      cudaMemcpyHostToDevice, b->stream),
      "upload inlet rows");
  chk(cudaMalloc(&d_counts, sizeof(int) * g->ny), "malloc counts");
  if (rc == VLBM_OK)
    chk(cudaMemcpyAsync(d_counts, counts.data(), sizeof(int) * g->ny, cudaMemcpyHostToDevice,
                        b->stream),
        "upload counts");
  if (rc == VLBM_OK) chk(vlbm_impl::launch_init_field(b->P, d_counts, amb, b->stream), "init field");
  if (rc == VLBM_OK) chk(cudaStreamSynchronize(b->stream), "initial field");
  cudaFree(d_counts);
  cudaFreeHost(rows);
  if (rc == VLBM_OK) rc = finish_create(b);
  if (rc != VLBM_OK) {
    free_batch(b);
    return rc;
  }
  *out = b;
  return VLBM_OK;
}

int vlbm_batch_create_fields(const vlbm_grid* g, const vlbm_params* p, int n_samples,
                             const double* init_fields, const double* inlet_rows,
                             const uint64_t* seeds, int device, vlbm_batch** out) {
  (void)seeds;
  if (!init_fields) return set_error(VLBM_E_INVALID, "Simulation: initial field size mismatch");
  if (p && p->bc[0] == VLBM_BC_INLET && !inlet_rows)
    return set_error(VLBM_E_INVALID, "Simulation: inlet boundary requires a profile");
  vlbm_batch* b = nullptr;
  if (int rc = alloc_batch(g, p, n_samples, device, &b)) return rc;
  const size_t n = (size_t)g->nx * g->ny;
  int rc = VLBM_OK;
  for (int s = 0; s < n_samples && rc == VLBM_OK; ++s)
    rc = upload_sample(b, s, init_fields + 4 * n * s,
                       inlet_rows ? inlet_rows + (size_t)4 * g->ny * s : nullptr);
  if (rc == VLBM_OK) rc = finish_create(b);
  if (rc != VLBM_OK) {
    free_batch(b);
    return rc;
  }
  *out = b;
  return VLBM_OK;
}

void vlbm_batch_destroy(vlbm_batch* b) { free_batch(b); }
int vlbm_batch_size(const vlbm_batch* b) { return b ? b->S : 0; }

int vlbm_batch_run_to(vlbm_batch* b, double target) {
  if (!b) return set_error(VLBM_E_INVALID, "null batch");
  CU(cudaSetDevice(b->device));
  CU(vlbm_impl::launch_set_budget(b->P, LLONG_MAX, b->stream));
  ++b->launches;
  return march_loop(b, target, 0.0, 0, 16);
}

int vlbm_batch_step(vlbm_batch* b, int n, double fixed_dt) {
  if (!b) return set_error(VLBM_E_INVALID, "null batch");
  if (n <= 0) return VLBM_OK;
  CU(cudaSetDevice(b->device));
  CU(vlbm_impl::launch_set_budget(b->P, n, b->stream));
  ++b->launches;
  const double inf = std::numeric_limits<double>::infinity();
  return march_loop(b, inf, fixed_dt > 0.0 ? fixed_dt : 0.0, 0, n < 16 ? n + 1 : 16);
}

int vlbm_batch_step_with_blending(vlbm_batch* b, double dt, const double* theta_x,
                                  const double* theta_y) {
  if (!b || !theta_x || !theta_y) return set_error(VLBM_E_INVALID, "null argument");
  CU(cudaSetDevice(b->device));
  const size_t ntx = (size_t)b->S * b->g.ny * (b->g.nx + 1);
  const size_t nty = (size_t)b->S * (b->g.ny + 1) * b->g.nx;
  if (!b->d_face_tx) {
    CU(cudaMalloc(&b->d_face_tx, sizeof(double) * ntx));
    CU(cudaMalloc(&b->d_face_ty, sizeof(double) * nty));
  }
  CU(cudaMemcpyAsync(b->d_face_tx, theta_x, sizeof(double) * ntx, cudaMemcpyHostToDevice,
                     b->stream));
  CU(cudaMemcpyAsync(b->d_face_ty, theta_y, sizeof(double) * nty, cudaMemcpyHostToDevice,
                     b->stream));
  b->P.face_tx = b->d_face_tx;
  b->P.face_ty = b->d_face_ty;
  for (int g = 0; g < b->G; ++g) {
    b->Pg[g].face_tx = b->d_face_tx + (size_t)b->g0[g] * b->g.ny * (b->g.nx + 1);
    b->Pg[g].face_ty = b->d_face_ty + (size_t)b->g0[g] * (b->g.ny + 1) * b->g.nx;
  }
  CU(vlbm_impl::launch_set_budget(b->P, 1, b->stream));
  ++b->launches;
  const double inf = std::numeric_limits<double>::infinity();
  return march_loop(b, inf, dt > 0.0 ? dt : 0.0, 2, 2);
}

int vlbm_batch_get(vlbm_batch* b, int s, double* u, double* pops, double* time, int64_t* steps,
                   int* status) {
  if (!b) return set_error(VLBM_E_INVALID, "null batch");
  if (s < 0 || s >= b->S) return set_error(VLBM_E_INVALID, "sample index out of range");
  CU(cudaSetDevice(b->device));
  std::vector<SampleCtl> ctl;
  if (int rc = read_ctl(b, ctl)) return rc;
  const MarchParams& P = b->P;
  const double* src = (ctl[s].parity ? P.buf1 : P.buf0) + (size_t)s * P.sample_stride;
  const size_t n = (size_t)P.nx * P.ny;
  if (u)
    for (int k = 0; k < 4; ++k)
      CU(cudaMemcpy2DAsync(u + k * n, sizeof(double) * P.nx, src + k * P.plane,
                           sizeof(double) * P.pitch, sizeof(double) * P.nx, P.ny,
                           cudaMemcpyDeviceToHost, b->stream));
  if (pops)
    for (int k = 0; k < 16; ++k)
      CU(cudaMemcpy2DAsync(pops + k * n, sizeof(double) * P.nx, src + (4 + k) * P.plane,
                           sizeof(double) * P.pitch, sizeof(double) * P.nx, P.ny,
                           cudaMemcpyDeviceToHost, b->stream));
  CU(cudaStreamSynchronize(b->stream));
  if (time) *time = ctl[s].t;
  if (steps) *steps = ctl[s].steps;
  if (status) *status = ctl[s].status;
  return VLBM_OK;
}

int vlbm_batch_get_fields(vlbm_batch* b, double* u_all) {
  if (!b || !u_all) return set_error(VLBM_E_INVALID, "null argument");
  CU(cudaSetDevice(b->device));
  std::vector<SampleCtl> ctl;
  if (int rc = read_ctl(b, ctl)) return rc;
  const MarchParams& P = b->P;
  const size_t n = (size_t)P.nx * P.ny;
  for (int s = 0; s < b->S; ++s) {
    const double* src = (ctl[s].parity ? P.buf1 : P.buf0) + (size_t)s * P.sample_stride;
    for (int k = 0; k < 4; ++k)
      CU(cudaMemcpy2DAsync(u_all + (4 * (size_t)s + k) * n, sizeof(double) * P.nx,
                           src + k * P.plane, sizeof(double) * P.pitch, sizeof(double) * P.nx,
                           P.ny, cudaMemcpyDeviceToHost, b->stream));
  }
  CU(cudaStreamSynchronize(b->stream));
  return VLBM_OK;
}

int vlbm_batch_copy_fields_device(vlbm_batch* b, double* d_u_all) {
  if (!b || !d_u_all) return set_error(VLBM_E_INVALID, "null argument");
  CU(cudaSetDevice(b->device));
  std::vector<SampleCtl> ctl;
  if (int rc = read_ctl(b, ctl)) return rc;
  const MarchParams& P = b->P;
  const size_t n = (size_t)P.nx * P.ny;
  for (int s = 0; s < b->S; ++s) {
    const double* src = (ctl[s].parity ? P.buf1 : P.buf0) + (size_t)s * P.sample_stride;
    for (int k = 0; k < 4; ++k)
      CU(cudaMemcpy2DAsync(d_u_all + (4 * (size_t)s + k) * n, sizeof(double) * P.nx,
                           src + k * P.plane, sizeof(double) * P.pitch, sizeof(double) * P.nx,
                           P.ny, cudaMemcpyDeviceToDevice, b->stream));
  }
  CU(cudaStreamSynchronize(b->stream));
  return VLBM_OK;
}

int vlbm_batch_get_scalars(vlbm_batch* b, double* time, int64_t* steps, int* status) {
  if (!b) return set_error(VLBM_E_INVALID, "null batch");
  CU(cudaSetDevice(b->device));
  std::vector<SampleCtl> ctl;
  if (int rc = read_ctl(b, ctl)) return rc;
  for (int s = 0; s < b->S; ++s) {
    if (time) time[s] = ctl[s].t;
    if (steps) steps[s] = ctl[s].steps;
    if (status) status[s] = ctl[s].status;
  }
  return VLBM_OK;
}

int vlbm_batch_get_theta(vlbm_batch* b, int s, double* theta) {
  if (!b || !theta) return set_error(VLBM_E_INVALID, "null argument");
  if (s < 0 || s >= b->S) return set_error(VLBM_E_INVALID, "sample index out of range");
  CU(cudaSetDevice(b->device));
  const MarchParams& P = b->P;
  CU(cudaMemcpy2DAsync(theta, sizeof(double) * P.nx, P.theta + (size_t)s * P.plane,
                       sizeof(double) * P.pitch, sizeof(double) * P.nx, P.ny,
                       cudaMemcpyDeviceToHost, b->stream));
  CU(cudaStreamSynchronize(b->stream));
  return VLBM_OK;
}

int vlbm_batch_device_u(vlbm_batch* b, int s, double** d_u) {
  if (!b || !d_u) return set_error(VLBM_E_INVALID, "null argument");
  if (s < 0 || s >= b->S) return set_error(VLBM_E_INVALID, "sample index out of range");
  std::vector<SampleCtl> ctl;
  if (int rc = read_ctl(b, ctl)) return rc;
  *d_u = (ctl[s].parity ? b->P.buf1 : b->P.buf0) + (size_t)s * b->P.sample_stride;
  return VLBM_OK;
}

void* vlbm_batch_stream(vlbm_batch* b) { return b ? (void*)b->stream : nullptr; }

int vlbm_batch_set_timing(vlbm_batch* b, int enable) {
  if (!b) return set_error(VLBM_E_INVALID, "null batch");
  b->timing = enable != 0;
  for (double& m : b->ms_kind) m = 0;
  return VLBM_OK;
}

int vlbm_batch_set_audit(vlbm_batch* b, int enable) {
  if (!b) return set_error(VLBM_E_INVALID, "null batch");
  CU(cudaSetDevice(b->device));
  if (enable && !b->P.audit) {
    CU(cudaMalloc(&b->P.audit, VLBM_AUDIT_COUNTERS * sizeof(vlbm_dev::AuditCtr)));
    CU(cudaMemset(b->P.audit, 0, VLBM_AUDIT_COUNTERS * sizeof(vlbm_dev::AuditCtr)));
  } else if (!enable && b->P.audit) {
    CU(cudaFree(b->P.audit));
    b->P.audit = nullptr;
  }
  for (auto& Q : b->Pg) Q.audit = b->P.audit;
  return VLBM_OK;
}

int vlbm_batch_audit(vlbm_batch* b, int64_t* counters) {
  if (!b || !counters) return set_error(VLBM_E_INVALID, "null argument");
  vlbm_dev::AuditCtr h[VLBM_AUDIT_COUNTERS] = {};
  if (b->P.audit) {
    CU(cudaMemcpyAsync(h, b->P.audit, sizeof(h), cudaMemcpyDeviceToHost, b->stream));
    CU(cudaStreamSynchronize(b->stream));
  }
  for (int k = 0; k < VLBM_AUDIT_COUNTERS; ++k) counters[k] = (int64_t)h[k];
  return VLBM_OK;
}

int vlbm_batch_queue_stats(vlbm_batch* b, int64_t* out) {
  if (!b || !out) return set_error(VLBM_E_INVALID, "null argument");
  CU(cudaSetDevice(b->device));
  unsigned long long h[4] = {0, 0, 0, 0};
  CU(cudaMemcpyAsync(h, b->d_qstats, sizeof(h), cudaMemcpyDeviceToHost, b->stream));
  CU(cudaStreamSynchronize(b->stream));
  out[0] = b->Pg.empty() ? 0 : b->Pg[0].hq_cap;
  out[1] = b->G;
  for (int k = 0; k < 4; ++k) out[2 + k] = (int64_t)h[k];
  return VLBM_OK;
}

int vlbm_batch_kernel_ms(vlbm_batch* b, double* ms) {
  if (!b || !ms) return set_error(VLBM_E_INVALID, "null argument");
  ms[0] = b->ms_kind[1];
  ms[1] = b->ms_kind[3];
  ms[2] = b->ms_kind[2];
  ms[3] = b->ms_kind[0];
  return VLBM_OK;
}

int vlbm_batch_stats(vlbm_batch* b, int64_t* launches, double* ms_theta, double* ms_advance,
                     double* ms_sched, int64_t* cell_updates) {
  if (!b) return set_error(VLBM_E_INVALID, "null batch");
  if (launches) *launches = b->launches;
  if (ms_theta) *ms_theta = b->ms_kind[1] + b->ms_kind[3];
  if (ms_advance) *ms_advance = b->ms_kind[2];
  if (ms_sched) *ms_sched = b->ms_kind[0];
  if (cell_updates) {
    std::vector<SampleCtl> ctl;
    if (int rc = read_ctl(b, ctl)) return rc;
    long long tot = 0;
    for (auto& c : ctl) tot += c.steps;
    *cell_updates = tot * (long long)b->g.nx * b->g.ny;
  }
  return VLBM_OK;
}

// ---- post-processing, host buffers -------------------------------------------

namespace {
struct DevBuf {
  double* p = nullptr;
  ~DevBuf() { cudaFree(p); }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, sizeof(double) * (n ? n : 1)); }
};
int upload(DevBuf& d, const double* h, size_t n) {
  CU(d.alloc(n));
  CU(cudaMemcpy(d.p, h, sizeof(double) * n, cudaMemcpyHostToDevice));
  return VLBM_OK;
}
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return check_device(dev);
}
}  // namespace

int vlbm_restrict_field(int nx, int ny, const double* fine, double* coarse) {
  if (nx % 2 != 0 || ny % 2 != 0)
    return set_error(VLBM_E_INVALID, "restrict_field: fine dimensions must be even");
  if (int rc = current_device()) return rc;
  const size_t nf = (size_t)4 * nx * ny, nc = nf / 4;
  DevBuf df, dc;
  if (int rc = upload(df, fine, nf)) return rc;
  CU(dc.alloc(nc));
  CU(vlbm_impl::launch_restrict(1, nx / 2, ny / 2, df.p, dc.p, 0));
  CU(cudaMemcpy(coarse, dc.p, sizeof(double) * nc, cudaMemcpyDeviceToHost));
  return VLBM_OK;
}

// Host tail of strong_error (metrics.hpp:81-89) over the device partials.
static int strong_finish(int M, const std::vector<double>& part, double* result, double* pc) {
  double acc = 0.0;
  double comp_acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int m = 0; m < M; ++m) {
    const double* o = part.data() + 10 * (size_t)m;
    if (o[1] == 0.0) return set_error(VLBM_E_DOMAIN, "strong_error: zero reference norm");
    acc += o[0] / o[1];
    for (int k = 0; k < 4; ++k) comp_acc[k] += o[6 + k] > 0.0 ? o[2 + k] / o[6 + k] : 0.0;
  }
  if (pc)
    for (int k = 0; k < 4; ++k) pc[k] = comp_acc[k] / static_cast<double>(M);
  *result = acc / static_cast<double>(M);
  return VLBM_OK;
}

int vlbm_strong_error(int M, int64_t n, const double* a, const double* b, double* result,
                      double* pc) {
  if (M < 1 || !a || !b || !result)
    return set_error(VLBM_E_INVALID, "strong_error: sample counts differ or are empty");
  if (int rc = current_device()) return rc;
  DevBuf da, db, dp;
  if (int rc = upload(da, a, (size_t)4 * n * M)) return rc;
  if (int rc = upload(db, b, (size_t)4 * n * M)) return rc;
  CU(dp.alloc(10 * (size_t)M));
  CU(vlbm_impl::launch_strong_partials(M, n, da.p, db.p, dp.p, 0));
  std::vector<double> part(10 * (size_t)M);
  CU(cudaMemcpy(part.data(), dp.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost));
  return strong_finish(M, part, result, pc);
}

int vlbm_wasserstein1(int M, int64_t n, const double* a, const double* b, int var,
                      double* result) {
  if (M < 1 || !a || !b || !result)
    return set_error(VLBM_E_INVALID, "wasserstein1: sample counts differ or are empty");
  if (var < 0 || var > 3) return set_error(VLBM_E_INVALID, "variable must be 0..3");
  if (int rc = current_device()) return rc;
  DevBuf da, db, dt, dr;
  if (int rc = upload(da, a, (size_t)4 * n * M)) return rc;
  if (int rc = upload(db, b, (size_t)4 * n * M)) return rc;
  CU(dt.alloc(n));
  CU(dr.alloc(1));
  CU(vlbm_impl::launch_w1_planes(M, n, da.p + var * n, 4 * n, db.p + var * n, 4 * n, dt.p, 0));
  CU(vlbm_impl::launch_ordered_mean(n, dt.p, dr.p, 0));
  CU(cudaMemcpy(result, dr.p, sizeof(double), cudaMemcpyDeviceToHost));
  return VLBM_OK;
}

int vlbm_ensemble_moments(int M, int64_t n, const double* x, double* mean, double* sd) {
  if (M < 1 || !x) return set_error(VLBM_E_INVALID, "ensemble_moments: no samples");
  if (M < 2)
    return set_error(VLBM_E_INVALID, "ensemble_moments: std requires at least 2 samples");
  if (int rc = current_device()) return rc;
  DevBuf dx, dm, ds;
  if (int rc = upload(dx, x, (size_t)4 * n * M)) return rc;
  CU(dm.alloc(4 * n));
  CU(ds.alloc(4 * n));
  CU(vlbm_impl::launch_moments(M, 4 * n, dx.p, 4 * n, dm.p, ds.p, 0));
  CU(cudaMemcpy(mean, dm.p, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(sd, ds.p, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
  return VLBM_OK;
}

// ---- post-processing, device buffers (stream-ordered) ------------------------

int vlbm_d_strong_partials(int M, int nxc, int nyc, const double* d_coarse, const double* d_fine,
                           double* d_partials, void* stream) {
  CU(vlbm_impl::launch_strong_partials_fused(M, nxc, nyc, d_coarse, d_fine, d_partials,
                                             (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_d_strong_partials_var(int M, int nxc, int nyc, const double* d_coarse, int64_t c_stride,
                               const double* d_fine, int64_t f_stride, double* d_partials,
                               void* stream) {
  if (M < 1) return set_error(VLBM_E_INVALID, "strong_error: sample counts differ or are empty");
  CU(vlbm_impl::launch_strong_partials_var(M, nxc, nyc, d_coarse, c_stride, d_fine, f_stride,
                                           d_partials, (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_strong_finish(int M, const double* partials, double* result, double* per_component) {
  if (M < 1 || !partials || !result)
    return set_error(VLBM_E_INVALID, "strong_error: sample counts differ or are empty");
  std::vector<double> part(partials, partials + 10 * (size_t)M);
  return strong_finish(M, part, result, per_component);
}

int vlbm_d_w1_restrict(int M, int nxc, int nyc, const double* d_coarse, int64_t c_stride,
                       const double* d_fine, int64_t f_stride, double* d_terms, void* stream) {
  if (M < 1) return set_error(VLBM_E_INVALID, "wasserstein1: sample counts differ or are empty");
  CU(vlbm_impl::launch_w1_restrict(M, nxc, nyc, d_coarse, c_stride, d_fine, f_stride, d_terms,
                                   (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_d_w1_restrict_mean(int M, int nxc, int nyc, const double* d_coarse, int64_t c_stride,
                            const double* d_fine, int64_t f_stride, double* d_terms,
                            double* d_scratch, double* d_result, void* stream) {
  if (M < 1) return set_error(VLBM_E_INVALID, "wasserstein1: sample counts differ or are empty");
  if (nxc < 1 || nyc < 1) return set_error(VLBM_E_INVALID, "wasserstein1: empty grid");
  CU(vlbm_impl::launch_w1_restrict_mean(M, nxc, nyc, d_coarse, c_stride, d_fine, f_stride, d_terms,
                                        d_scratch, d_result, (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_d_restrict_var(int M, int nxc, int nyc, const double* d_fine, int var, double* d_out,
                        void* stream) {
  CU(vlbm_impl::launch_restrict_var(M, nxc, nyc, d_fine, var, d_out, (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_d_w1_cells(int M, int64_t n, const double* d_a, const double* d_b, double* d_terms,
                    void* stream) {
  if (M < 1) return set_error(VLBM_E_INVALID, "wasserstein1: sample counts differ or are empty");
  CU(vlbm_impl::launch_w1_cells(M, n, d_a, d_b, d_terms, (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_d_w1_cells_planes(int M, int64_t n, const double* d_a, const double* d_b,
                           double* d_terms, void* stream) {
  if (M < 1) return set_error(VLBM_E_INVALID, "wasserstein1: sample counts differ or are empty");
  CU(vlbm_impl::launch_w1_planes(M, n, d_a, n, d_b, n, d_terms, (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_d_w1_rows(int M, int nxc, int64_t cell0, int64_t n, const double* const* d_coarse_rows,
                   const double* const* d_fine_rows, double* d_terms, void* stream) {
  if (M < 1) return set_error(VLBM_E_INVALID, "wasserstein1: sample counts differ or are empty");
  if (nxc < 1 || cell0 < 0 || n < 0 || !d_coarse_rows || !d_fine_rows)
    return set_error(VLBM_E_INVALID, "wasserstein1: invalid row tables");
  if (n == 0) return VLBM_OK;
  CU(vlbm_impl::launch_w1_rows(M, nxc, cell0, n, d_coarse_rows, d_fine_rows, d_terms,
                               (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_ipc_handle(const void* d_ptr, unsigned char handle[64], uint64_t* offset) {
  if (!d_ptr || !handle || !offset) return set_error(VLBM_E_INVALID, "ipc: null argument");
  using Range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Range range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !fn)
      return set_error(VLBM_E_CUDA, "ipc: cuMemGetAddressRange unavailable");
    range = reinterpret_cast<Range>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)d_ptr) != CUDA_SUCCESS)
    return set_error(VLBM_E_CUDA, "ipc: not a device allocation");
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, (void*)base));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  *offset = (uint64_t)((CUdeviceptr)d_ptr - base);
  return VLBM_OK;
}

int vlbm_ipc_open(const unsigned char handle[64], void** d_base) {
  if (!handle || !d_base) return set_error(VLBM_E_INVALID, "ipc: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  CU(cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess));
  return VLBM_OK;
}

int vlbm_ipc_close(void* d_base) {
  CU(cudaIpcCloseMemHandle(d_base));
  return VLBM_OK;
}

int vlbm_d_ordered_mean(int64_t n, const double* d_terms, double* d_result, void* stream) {
  CU(vlbm_impl::launch_ordered_mean(n, d_terms, d_result, (cudaStream_t)stream));
  return VLBM_OK;
}

int vlbm_d_moments_planes(int M, int64_t n, const double* d_x, double* d_mean, double* d_std,
                          void* stream) {
  // one variable: x(m, c) = d_x[m * n + c]
  if (M < 2) return set_error(VLBM_E_INVALID, "ensemble_moments: std requires at least 2 samples");
  CU(vlbm_impl::launch_moments(M, n, d_x, n, d_mean, d_std, (cudaStream_t)stream));
  return VLBM_OK;
}

}  // extern "C"
