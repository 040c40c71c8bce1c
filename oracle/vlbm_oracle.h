/* oracle/vlbm_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path (the VLBM march and the
 * W1/L1 post-processing of /root/reference/proj/include/vlbm/).  It is the
 * checker the CUDA path is compared against; it is pinned bit-for-bit to the
 * reference itself (oracle/_ref, built from the unmodified headers) and to
 * the reference tests' known-answer values by tests/test_oracle_pin.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  Field layout: include/vlbm_b200.h (4 planes, x fastest).
 */
#ifndef VLBM_ORACLE_H_
#define VLBM_ORACLE_H_
#include <stdint.h>

#include "vlbm_b200.h"

typedef struct vo_sim vo_sim;

uint64_t vo_mix64(uint64_t z);
uint64_t vo_sample_seed(uint64_t base, uint64_t m);
uint64_t vo_draw_coefficients(uint64_t base, uint64_t m, int K, double* y, double* z);
double vo_density_perturbation(double y, int K, const double* yc, const double* zc,
                               const vlbm_perturbation* pp);
void vo_inlet_state(double y, int K, const double* yc, const double* zc,
                    const vlbm_perturbation* pp, double gamma, double* out);
int vo_initial_field(const vlbm_grid* g, int K, const double* yc, const double* zc,
                     const vlbm_perturbation* pp, double gamma, double strip, double* out);
double vo_pressure(const double* u, double gamma);
void vo_maxwellians(const double* u, double a, double alpha, double gamma, double* out16);

int vo_sim_create(const vlbm_grid* g, const vlbm_params* p, const double* init,
                  const double* inlet_rows, uint64_t seed, vo_sim** out);
void vo_sim_destroy(vo_sim* s);
int vo_sim_step(vo_sim* s, double dt);
double vo_sim_suggest_dt(vo_sim* s);
double vo_sim_time(vo_sim* s);
long vo_sim_steps(vo_sim* s);
int vo_sim_state_finite(vo_sim* s);
void vo_sim_get(vo_sim* s, double* u, double* pops);
int vo_sim_compute_blending(vo_sim* s, double a, double* tx, double* ty);
int vo_sim_step_with_blending(vo_sim* s, double dt, const double* tx, const double* ty);
void vo_sim_theta_cell(vo_sim* s, double* theta);
int vo_sim_limiter_cells(vo_sim* s, double a, double* out);

int vo_run_sample(const vlbm_grid* g, const vlbm_params* p, const vlbm_perturbation* pp, int K,
                  const double* yc, const double* zc, uint64_t seed, double strip,
                  const double* times, int n_times, double* out_fields, double* out_time,
                  int* out_div, long* out_steps, int* out_admissible);

int vo_restrict_field(int nx, int ny, const double* fine, double* coarse);
int vo_strong_error(int M, int64_t n, const double* a, const double* b, double* result,
                    double* per_comp);
int vo_wasserstein1(int M, int64_t n, const double* a, const double* b, int var, double* result);
int vo_ensemble_moments(int M, int64_t n, const double* x, double* mean, double* stddev);
const char* vo_last_error(void);

#endif
