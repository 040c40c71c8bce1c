/*
 * vlbm_b200.h — C ABI of the B200-native probabilistic VLBM hot path.
 *
 * This is the drop-in boundary between the reference's host C++ (config,
 * manifest, .vlbm snapshots: /root/reference/proj/include/vlbm/{config,
 * ensemble,snapshot_io}.hpp) and the sm_100a kernels.  Plain C types only:
 * pointers, sizes, ints and doubles; no torch or C++ types cross it.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/vlbm/):
 *
 *   vlbm_batch_create        Simulation::Simulation         solver.hpp:61-100
 *                            + initial_field / inlet_state  perturbation.hpp:87-122
 *                            (as built by run_sample        solver.hpp:633-640)
 *   vlbm_batch_create_fields Simulation::Simulation on caller fields (tests)
 *   vlbm_batch_run_to        run_sample's inner while loop  solver.hpp:645-658
 *   vlbm_batch_step          Simulation::step(suggest_dt()) solver.hpp:157-170
 *   vlbm_batch_step_with_blending
 *                            Simulation::step_with_blending solver.hpp:173-181
 *   vlbm_batch_get           Simulation::state/population/time/steps,
 *                            snapshot()                     solver.hpp:103-120
 *   vlbm_batch_get_theta     Simulation::compute_blending   solver.hpp:184-191
 *                            (cell theta of the last limiter pass)
 *   vlbm_draw_coefficients   draw_coefficients              perturbation.hpp:42-54
 *   vlbm_inlet_rows          inlet_state at y_center(j)     perturbation.hpp:87-95
 *   vlbm_restrict_field      restrict_field                 metrics.hpp:29-49
 *   vlbm_strong_error        strong_error                   metrics.hpp:55-90
 *   vlbm_wasserstein1        wasserstein1                   metrics.hpp:97-125
 *   vlbm_ensemble_moments    ensemble_moments               metrics.hpp:148-177
 *   vlbm_d_w1_restrict_mean  wasserstein1 on device planes  metrics.hpp:97-125
 *                            (restriction fused, storage-order mean overlapped)
 *   vlbm_metrics_*           compute_metrics' per (pair, time) W1 + E_strong
 *                            with one upload per ensemble   metrics.hpp:259-327
 *   vlbm_d_w1_rows           wasserstein1's per-cell terms over samples held on
 *                            several GPUs (row tables, CUDA-IPC peer mappings):
 *                            compute_metrics' W1 across a sample-sharded node
 *   vlbm_batch_copy_fields_device
 *                            the snapshots of run_sample kept on the device
 *                            (compute_metrics without the .vlbm round trip)
 *   vlbm_device_count        run_ensemble's worker count    ensemble.hpp:294-300
 *                            (one worker per GPU)
 *
 * Layouts.  A "field" is the reference FieldSnapshot data in the .vlbm
 * on-disk plane order (snapshot_io.hpp:311-315): 4 contiguous f64 planes
 * (rho, rho*v1, rho*v2, E), each ny rows of nx values, x fastest.  An
 * ensemble of M fields is M such blocks back to back.  "pops" are 4 such
 * field blocks, population k = 0..3 (paper's u_1..u_4), 16 planes.
 *
 * Errors: every call returns 0 on success or a negative vlbm_status; the
 * message is available from vlbm_last_error() (thread-local).  The C++
 * wrapper maps VLBM_E_INVALID -> std::invalid_argument, VLBM_E_DOMAIN ->
 * std::domain_error, VLBM_E_RUNTIME -> std::runtime_error, mirroring the
 * reference's throw sites.
 *
 * Functions whose pointer arguments are named d_* take DEVICE pointers and
 * run on the caller's stream (cudaStream_t passed as void*); all others take
 * host pointers and are synchronous.
 */
#ifndef VLBM_B200_H_
#define VLBM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VLBM_ABI_VERSION 1

typedef enum vlbm_status {
  VLBM_OK = 0,
  VLBM_E_INVALID = -1, /* std::invalid_argument in the reference */
  VLBM_E_DOMAIN = -2,  /* std::domain_error */
  VLBM_E_RUNTIME = -3, /* std::runtime_error */
  VLBM_E_CUDA = -4,    /* CUDA runtime failure (no CPU fallback exists) */
  VLBM_E_NOMEM = -5
} vlbm_status;

/* BcType, solver.hpp:20 (same numbering). */
typedef enum vlbm_bc {
  VLBM_BC_INLET = 0,
  VLBM_BC_OUTFLOW = 1,
  VLBM_BC_WALL = 2,
  VLBM_BC_PERIODIC = 3
} vlbm_bc;

/* Limiter, lattice.hpp:10 (same numbering). */
typedef enum vlbm_limiter {
  VLBM_LIMITER_FIRST_ORDER = 0,
  VLBM_LIMITER_SECOND_ORDER = 1,
  VLBM_LIMITER_RLMP = 2
} vlbm_limiter;

/* Sample status (RunStatus, ensemble.hpp:23, plus the in-flight state). */
typedef enum vlbm_sample_status {
  VLBM_SAMPLE_RUNNING = 0,
  VLBM_SAMPLE_DIVERGED = 2
} vlbm_sample_status;

/* Grid, grid.hpp:14-38. */
typedef struct vlbm_grid {
  int nx, ny;
  double x_max, y_min, y_max;
} vlbm_grid;

/* GasParams (euler.hpp:9) + LatticeParams (lattice.hpp:13-35) +
 * Boundaries side types (solver.hpp:25-31) + set_reference (solver.hpp:599). */
typedef struct vlbm_params {
  double gamma;
  double alpha;
  double safety;
  double rlmp_relaxation;
  double positivity_floor;
  int limiter;            /* vlbm_limiter */
  int conservative_bound; /* 0/1 */
  double rho_ref, p_ref;  /* positivity reference (run_sample: rho_amb, p_amb) */
  int bc[4];              /* x_min, x_max, y_min, y_max: vlbm_bc */
} vlbm_params;

/* PerturbationParams, perturbation.hpp:16-31. */
typedef struct vlbm_perturbation {
  double amplitude;
  int modes;
  double decay_exponent;
  double r_jet;
  double rho_jet_bar;
  double rho_amb;
  double p_amb;
  double v_jet;
} vlbm_perturbation;

typedef struct vlbm_batch vlbm_batch;

/* ---- library ---------------------------------------------------------- */
int vlbm_abi_version(void);
/* Visible CUDA devices (0 without a GPU). */
int vlbm_device_count(void);
const char* vlbm_last_error(void);
/* Fills the reference defaults (lattice.hpp:13-35, euler.hpp:10,
 * perturbation.hpp:16-31, config.hpp:27-29) and the jet boundaries. */
void vlbm_default_params(vlbm_params* p);
void vlbm_default_perturbation(vlbm_perturbation* pp);
void vlbm_default_grid(vlbm_grid* g, int nx, int ny);

/* ---- initial conditions (host; integer-exact splitmix64 + host libm) -- */
/* Returns the per-sample seed (ModeCoefficients::seed); y,z get K values. */
uint64_t vlbm_draw_coefficients(uint64_t base_seed, uint64_t m, int K, double* y_coeffs,
                                double* z_coeffs);
/* out[j*4 + k] = inlet_state(grid.y_center(j), coeffs, pp, gamma)[k]. */
int vlbm_inlet_rows(const vlbm_grid* g, const vlbm_perturbation* pp, double gamma,
                    const double* y_coeffs, const double* z_coeffs, double* out);

/* ---- the march: a batch of independent samples on one grid, one GPU -- */
/* Jet-case batch: samples m = m0 .. m0+n_samples-1 of base_seed, built
 * exactly as run_sample builds them (inlet profile, initial_field with the
 * wedge strip, set_reference(rho_amb, p_amb)). */
int vlbm_batch_create(const vlbm_grid* g, const vlbm_params* p, const vlbm_perturbation* pp,
                      uint64_t base_seed, int64_t m0, int n_samples, double strip_width,
                      int device, vlbm_batch** out);
/* Jet-case batch from explicit mode coefficients (SampleSpec::coeffs,
 * solver.hpp:611-619; e.g. read back from a manifest): y_coeffs, z_coeffs
 * are n_samples x pp->modes; seeds (ModeCoefficients::seed) may be NULL. */
int vlbm_batch_create_coeffs(const vlbm_grid* g, const vlbm_params* p,
                             const vlbm_perturbation* pp, int n_samples, const double* y_coeffs,
                             const double* z_coeffs, double strip_width, int device,
                             vlbm_batch** out);
/* Generic batch on caller-provided initial fields (n_samples field blocks)
 * and optional inlet rows (n_samples x ny x 4; required iff bc[0] is
 * Inlet).  seeds may be NULL. */
int vlbm_batch_create_fields(const vlbm_grid* g, const vlbm_params* p, int n_samples,
                             const double* init_fields, const double* inlet_rows,
                             const uint64_t* seeds, int device, vlbm_batch** out);
void vlbm_batch_destroy(vlbm_batch* b);
int vlbm_batch_size(const vlbm_batch* b);

/* Marches every running sample until t >= target - 1e-12, clamping the last
 * dt to hit target exactly; divergence (non-finite dt or state) stops a
 * sample as run_sample does.  max_steps_per_sample < 0 = unlimited. */
int vlbm_batch_run_to(vlbm_batch* b, double target);
/* n steps of step(suggest_dt()) for every running sample (no clamp);
 * fixed_dt > 0 instead uses step(fixed_dt) (reference tests' fixed-dt
 * loops).  Divergence handling as run_to. */
int vlbm_batch_step(vlbm_batch* b, int n, double fixed_dt);
/* One step with a prescribed interface blending (test hook).  theta_x is
 * n_samples x ny x (nx+1), theta_y n_samples x (ny+1) x nx (BlendingField
 * layout, solver.hpp:35-51).  dt <= 0 uses suggest_dt(). */
int vlbm_batch_step_with_blending(vlbm_batch* b, double dt, const double* theta_x,
                                  const double* theta_y);

/* Copy out sample s.  Any pointer may be NULL.  u: 1 field block; pops: 4
 * field blocks.  status: vlbm_sample_status. */
int vlbm_batch_get(vlbm_batch* b, int s, double* u, double* pops, double* time, int64_t* steps,
                   int* status);
/* All samples' u into n_samples field blocks (snapshot of the batch). */
int vlbm_batch_get_fields(vlbm_batch* b, double* u_all);
/* The same dense (S x 4 x ny x nx) fields into DEVICE memory of the batch's
 * GPU (snapshots kept on the device for the on-device metrics; no host copy). */
int vlbm_batch_copy_fields_device(vlbm_batch* b, double* d_u_all);
/* Per-sample scalars: time, steps, status (arrays of n_samples; any NULL). */
int vlbm_batch_get_scalars(vlbm_batch* b, double* time, int64_t* steps, int* status);
/* Cell theta (ny x nx) of sample s from the last limiter pass. */
int vlbm_batch_get_theta(vlbm_batch* b, int s, double* theta_cell);
/* Device views for zero-copy consumers (torch/NCCL plumbing): u planes of
 * sample s in the current buffer, cudaStream_t of the batch. */
int vlbm_batch_device_u(vlbm_batch* b, int s, double** d_u);
void* vlbm_batch_stream(vlbm_batch* b);
/* Kernel-launch counter (for the bench's gpu_launches claim) and the
 * accumulated device time of the limiter / advance kernels (ms, CUDA
 * events) when timing is enabled. */
int vlbm_batch_set_timing(vlbm_batch* b, int enable);
int vlbm_batch_stats(vlbm_batch* b, int64_t* launches, double* ms_theta, double* ms_advance,
                     double* ms_sched, int64_t* cell_updates);
/* The timed device ms by kernel group: ms[0] limiter tile pass (u_FO, bounds,
 * feasible(1)), ms[1] limiter hard cells (cap + bisections), ms[2] advance,
 * ms[3] scheduler.  With several sample groups the groups' overlapping
 * launches are each timed on their own stream. */
int vlbm_batch_kernel_ms(vlbm_batch* b, double* ms);
/* Audit of the limiter's certificates (test hook): when enabled, every
 * certified decision (the theta = 1 vertex certificate and each certified
 * bisection step) is re-checked with the full 16-check feasible() and
 * disagreements are counted.  vlbm_batch_audit fills
 * counters[VLBM_AUDIT_COUNTERS]: disagreements (must be 0), bisections
 * entered, fully certified at the closed-form theta, uncertified, not
 * certifiable, no margin at theta = 0, uncertified vertices at the start
 * (sum), vertex evaluations in the bisections (sum), cells whose diagonal
 * passes at theta = 1, of those vertex-certified, of those feasible(1),
 * warps with vertex checks left, and three certificate statistics
 * (uncertified-but-feasible; of those with the true vertex minimum above
 * p_FO / 2; of those with the quadratic part dominant). */
/* Limiter-queue statistics (cumulative since creation): out[0] queue
 * capacity (entries, per sample group), out[1] sample groups (the queues
 * are shared by groups marched one after another on the batch's stream when
 * one set covering every cell of the batch does not fit in memory),
 * out[2] cells finished in place because a queue was full (overflows; 0
 * when the capacity covers a group's cells), out[3] the largest number of
 * hard cells (theta = 1 infeasible) of one group in one step, out[4] hard
 * cells summed over steps and groups, out[5] limiter passes counted. */
int vlbm_batch_queue_stats(vlbm_batch* b, int64_t* out6);
#define VLBM_AUDIT_COUNTERS 16
int vlbm_batch_set_audit(vlbm_batch* b, int enable);
int vlbm_batch_audit(vlbm_batch* b, int64_t* counters);

/* ---- post-processing (host buffers, synchronous) ---------------------- */
/* restrict_field: fine nx x ny (even) field block -> (nx/2) x (ny/2). */
int vlbm_restrict_field(int nx, int ny, const double* fine, double* coarse);
/* strong_error over M coarse / M restricted-fine field blocks of n_cells;
 * per_component (4) may be NULL. */
int vlbm_strong_error(int M, int64_t n_cells, const double* coarse, const double* restricted,
                      double* result, double* per_component);
/* wasserstein1 over M field blocks each (var = 0..3 component). */
int vlbm_wasserstein1(int M, int64_t n_cells, const double* a, const double* b, int var,
                      double* result);
/* ensemble_moments: mean and std (each one field block). */
int vlbm_ensemble_moments(int M, int64_t n_cells, const double* samples, double* mean,
                          double* stddev);

/* ---- post-processing on device arrays (stream-ordered) ---------------- */
/* Fused restriction + per-sample L1 partials: coarse (M x 4 x nyc x nxc)
 * and fine (M x 4 x 2nyc x 2nxc) field blocks; writes per-sample num, den
 * and per-component cnum[4], cden[4] (M x 10 doubles) in the reference's
 * sequential summation order (bit-exact). */
int vlbm_d_strong_partials(int M, int nxc, int nyc, const double* d_coarse, const double* d_fine,
                           double* d_partials, void* stream);
/* One variable (e.g. rho planes only, BASELINE configs[3]): coarse(m, c) =
 * d_coarse[m*c_stride + c]; the fine plane of sample m (2nxc x 2nyc) starts
 * at d_fine + m*f_stride and is restricted on the fly.  Writes M x 10
 * partials like vlbm_d_strong_partials (components 1..3 zero): equal to the
 * 4-component sums when the other components are identically zero. */
int vlbm_d_strong_partials_var(int M, int nxc, int nyc, const double* d_coarse, int64_t c_stride,
                               const double* d_fine, int64_t f_stride, double* d_partials,
                               void* stream);
/* strong_error's host tail (metrics.hpp:81-89) over M x 10 partials (host
 * copy): throws-equivalent VLBM_E_DOMAIN on a zero reference norm. */
int vlbm_strong_finish(int M, const double* partials, double* result, double* per_component);

/* compute_metrics' reductions for one (grid pair, snapshot time) with each
 * ensemble uploaded once (metrics.hpp:284-300): begin with the number of
 * jointly valid samples M (M* of the pair), the coarse grid and the metric
 * variable; add the samples in order, in any batches (host fields: coarse
 * [count][4][nyc][nxc], fine [count][4][2nyc][2nxc]) -- each batch's
 * strong_error partials are taken on the device at once and the metric
 * variable's planes kept there; finish runs wasserstein1 (restriction fused)
 * and the strong_error tail.  Results bit-identical to wasserstein1 and
 * strong_error on the restricted fields. */
typedef struct vlbm_metrics vlbm_metrics;
int vlbm_metrics_begin(int M, int nxc, int nyc, int var, int device, vlbm_metrics** out);
int vlbm_metrics_add(vlbm_metrics* m, int first, int count, const double* coarse,
                     const double* fine);
int vlbm_metrics_finish(vlbm_metrics* m, double* w1, double* e_strong, double* per_component);
void vlbm_metrics_destroy(vlbm_metrics* m);
/* W1 per-cell terms of coarse planes vs the on-the-fly restriction of fine
 * planes (one variable, addressing as vlbm_d_strong_partials_var). */
int vlbm_d_w1_restrict(int M, int nxc, int nyc, const double* d_coarse, int64_t c_stride,
                       const double* d_fine, int64_t f_stride, double* d_cell_terms,
                       void* stream);
/* vlbm_d_w1_restrict + vlbm_d_ordered_mean in one call, the storage-order
 * mean overlapped with the per-cell terms (cells in chunks of whole coarse
 * rows; each chunk's part of the sequential sum runs on an internal stream
 * once its terms exist).  d_terms: n_cells doubles, d_scratch: 1 double,
 * d_result: W1 (wasserstein1's return value, bit-identical). */
int vlbm_d_w1_restrict_mean(int M, int nxc, int nyc, const double* d_coarse, int64_t c_stride,
                            const double* d_fine, int64_t f_stride, double* d_terms,
                            double* d_scratch, double* d_result, void* stream);
/* Restricted-fine plane of one variable into a (M x n_cells) array. */
int vlbm_d_restrict_var(int M, int nxc, int nyc, const double* d_fine, int var, double* d_out,
                        void* stream);
/* Per-cell W1 terms cell_c = sum_m |a_(m) - b_(m)| / M on cell-major
 * columns: d_a, d_b are (n_cells x M), one column per cell. */
int vlbm_d_w1_cells(int M, int64_t n_cells, const double* d_a, const double* d_b,
                    double* d_cell_terms, void* stream);
/* Same on sample-major planes (M x n_cells, one variable): the kernel
 * gathers the per-cell columns itself. */
int vlbm_d_w1_cells_planes(int M, int64_t n_cells, const double* d_a, const double* d_b,
                           double* d_cell_terms, void* stream);
/* Per-cell W1 terms of cells [cell0, cell0 + n_cells) of an nxc-wide coarse
 * grid over M samples given as ROW TABLES: d_coarse_rows / d_fine_rows are
 * device arrays of M device pointers, sample m's coarse density plane and
 * its fine (2nxc-wide) plane, which may live on any GPU of the node
 * (peer-mapped through vlbm_ipc_open).  The restriction is fused; the kernel
 * reads the remote samples over NVLink while it sorts (the fused alternative
 * to the all-to-all re-shard; wasserstein1's per-cell term, metrics.hpp:113-122). */
int vlbm_d_w1_rows(int M, int nxc, int64_t cell0, int64_t n_cells,
                   const double* const* d_coarse_rows, const double* const* d_fine_rows,
                   double* d_cell_terms, void* stream);
/* CUDA IPC for the row tables: the 64-byte handle of the allocation holding
 * d_ptr and d_ptr's byte offset in it; open a peer process's handle (the
 * base of its allocation, mapped with peer access) and close it. */
int vlbm_ipc_handle(const void* d_ptr, unsigned char handle[64], uint64_t* offset);
int vlbm_ipc_open(const unsigned char handle[64], void** d_base);
int vlbm_ipc_close(void* d_base);
/* Storage-order sequential sum of n terms, then / n (wasserstein1's acc). */
int vlbm_d_ordered_mean(int64_t n, const double* d_terms, double* d_result, void* stream);
/* Per-cell moments on sample-major planes (M x n_cells, one variable). */
int vlbm_d_moments_planes(int M, int64_t n_cells, const double* d_x, double* d_mean,
                          double* d_std, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VLBM_B200_H_ */
