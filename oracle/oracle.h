/*
 * oracle.h -- CPU restatement of the reference MF-CIM (MFZ) L0RBCS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This code is the parity checker for the CUDA
 * product path in paper_2405_00366_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * never links, imports or falls back to it.
 *
 * Every function restates a reference routine (paths relative to
 * /root/reference/proj) and keeps its exact elementwise association:
 *   rng.hpp:21-64            mt19937_64 + Box-Muller           -> orc_rng_*
 *   datagen.cpp:11-55        gen_instance                      -> orc_gen_instance
 *   orchestrator.cpp:12-20   pump / eta schedules              -> orc_pump_*, orc_eta_schedule
 *   orchestrator.cpp:45-47,80-99  apply_coupling / make_problem -> orc_problem_*, orc_apply_*
 *   solver_mfz.cpp:24-124    init / fields / step / run        -> orc_local_field_*, orc_mfz_step, orc_run_mfz
 *   cdp.cpp:17-64,66-148     subproblem, Jacobi, CG, scatter   -> orc_cdp_minimize
 *   model.cpp:18-52,128-153  hamiltonian/objective/rmse/hamming -> orc_hamiltonian, orc_rmse, ...
 *   orchestrator.cpp:163-235 median + alternating_minimize     -> orc_alternating_minimize
 *   tools/main.cpp:263-268   mix_seed                          -> orc_mix_seed
 *
 * Coupling modes (the self-sensitivity experiment):
 *   ORC_LITERAL   apply_gram(w) = A^T (A w), two sequential GEMVs, no FMA
 *                 (orchestrator.cpp:86-88 -- the reference's main path).
 *   ORC_CANON     G = A^T A built with a sequential-k fma chain; G w summed in
 *                 the GPU's documented segmented fma order (nseg, gran).  This
 *                 is the order the fp64 CUDA path reproduces bit for bit.
 *   ORC_EXPLICIT  G = A^T A built sequentially without FMA; G w sequential.
 * Eigen's own GEMV/GEMM summation order cannot be reproduced without Eigen
 * (absent in this image), so bitwise parity with the original binary is
 * unpinned; the three modes bound how much the reduction order matters.
 *
 * Builder extensions (marked ⊕ there), implemented identically
 * in the GPU host runtime:
 *   pump_kind = ORC_PUMP_LINEAR: p(t) = (p_end * t) / (n_steps * dt) at the
 *   accumulated t (t += dt per step, solver_mfz.cpp:86).
 */
#ifndef CIMCS_ORACLE_H
#define CIMCS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- RNG */
typedef struct {
    uint64_t mt[312];
    int mti;
    uint64_t n_gauss;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_raw(orc_rng* r);
double orc_uniform_open(orc_rng* r);
uint64_t orc_uniform_below(orc_rng* r, uint64_t bound);
double orc_gauss(orc_rng* r);
uint64_t orc_mix_seed(uint64_t base, uint64_t salt);
long long orc_round_half_away(double v);

/* ------------------------------------------------------------ datagen */
/* returns 0 ok, 1 input_error */
int orc_gen_dims(int N, double alpha, double a, int* M, int* K);
/* A is M x N column-major (Eigen default, as in ProblemInstance::A). */
int orc_gen_instance(int N, double alpha, double a, double nu, uint64_t seed,
                     double* A, double* y, double* x, int32_t* xi);

/* ---------------------------------------------------------- schedules */
enum { ORC_PUMP_SIGMOID = 0, ORC_PUMP_LINEAR = 1 };
double orc_pump_sigmoid(double t, double p_thr, double d);
double orc_pump_linear(double t, double p_end, double T);
double orc_eta_schedule(int i, double eta_init, double eta_end, int velo);
int orc_trace_stride(int n_steps, int cap);

typedef struct {
    double g2, j, K, beta, tau, dt;
    int n_steps;
    double p_thr, d, eta_init, eta_end;
    int velo;
    double dt_c;
    int jacobi_iters, cg_max_iters;
    double cg_tol, gamma;
    int mfz_loss_minus_j;
    double mu_abort;
    int pump_kind;     /* ⊕ ORC_PUMP_SIGMOID (reference) | ORC_PUMP_LINEAR */
    double pump_end;   /* ⊕ linear ramp end value (1.2 in BASELINE configs) */
} orc_hyper;

void orc_hyper_default(orc_hyper* h);       /* types.hpp:77-96 */
int orc_hyper_validate(const orc_hyper* h); /* types.hpp:98-106; 0 ok, 2 config_error */
/* p[k] = pump at the accumulated t of step k, k < n_steps. */
void orc_pump_table(const orc_hyper* h, double* p);

/* ------------------------------------------------------------ problem */
enum { ORC_LITERAL = 0, ORC_CANON = 1, ORC_EXPLICIT = 2 };

typedef struct {
    int N, M, mode, nseg, gran;
    const double* A; /* M x N col-major, caller-owned */
    const double* y; /* M */
    double* G;       /* N x N row-major (modes CANON/EXPLICIT) */
    double* hz;      /* N */
    double* D;       /* N : gram_diag */
    double* work;    /* max(M, N) scratch */
    const double* x_true;  /* optional */
    const int32_t* xi_true;
} orc_problem;

int orc_problem_init_gram(orc_problem* p, int N, const double* G, const double* hz);
int orc_problem_init(orc_problem* p, int N, int M, const double* A, const double* y,
                     int mode, int nseg, int gran);
void orc_problem_free(orc_problem* p);
/* canonical segmented dot of row i of G with v (exposed for unit tests) */
double orc_canon_dot(const double* g, const double* v, int N, int nseg, int gran);
void orc_gram_apply(const orc_problem* p, const double* w, double* out);     /* G w   */
void orc_coupling_apply(const orc_problem* p, const double* w, double* out); /* D∘w - G w */

void orc_local_field_cn(const orc_problem* p, const double* R, const double* c,
                        double tau, double* h);
void orc_local_field_bn(const orc_problem* p, const double* R, const int32_t* sigma,
                        double tau, double* h);
/* returns -1 ok, >=0 offending spin (divergence_error), -2 non-finite pump (input_error) */
int orc_mfz_step(int N, const double* c, const double* e, double p, const orc_hyper* h,
                 double eta, const double* R, const double* hfield, double* c_out,
                 double* e_out);

enum { ORC_MFZ_CN = 0, ORC_MFZ_BN = 1, ORC_PP = 2 }; /* == Backend, orchestrator.hpp:28 */

/* Positive-P SDE backend (solver_pp.cpp:9-132): measured_amplitude,
 * local_field_pp, pp_step (mu, n, m, e from the pre-step state; returns -1 or
 * the first spin with a non-finite value), run_pp (N deviates per step from
 * rng; returns -1, the offending spin (non-finite: kind 0, |mu| > mu_abort:
 * kind 1), -3 config_error). */
int orc_measured_amplitude(int N, const double* mu, const double* noise, const orc_hyper* h,
                           double* mt);
void orc_local_field_pp(const orc_problem* p, const double* R, const double* mt, double tau,
                        double* out);
int orc_pp_step(int N, const double* mu, const double* n, const double* m, const double* e,
                double p, const orc_hyper* h, double eta, const double* R, const double* hf,
                const double* noise, double* mu_o, double* n_o, double* m_o, double* e_o);
int orc_run_pp(const orc_problem* p, const double* R, const orc_hyper* h, double eta,
               orc_rng* rng, double* mu_out, double* n_out, double* m_out, double* e_out,
               double* mt_out, int32_t* sigma_out, double* min_e, int* kind);

/* One CIM call (run_mfz).  c0 drawn from rng.  trace_* optional (NULL).
 * Returns -1 ok, >=0 offending spin index, -2 input_error, -3 config_error. */
void orc_set_perturb(int mode); /* sensitivity study knob, see oracle.c */
int orc_run_mfz(const orc_problem* p, const double* R, const orc_hyper* h, double eta,
                int backend, orc_rng* rng, double* c_out, double* e_out,
                int32_t* sigma_out, double* min_e, int trace_mode, int* trace_count,
                int32_t* trace_steps, double* trace_c, double* trace_e, int trace_cap);

enum { ORC_CDP_JACOBI = 0, ORC_CDP_CG = 1 };
/* returns 0 ok, 1 input_error (singular diagonal; *bad_index = active spin) */
int orc_cdp_minimize(const orc_problem* p, const int32_t* sigma, const double* R_prev,
                     int method, const orc_hyper* h, double* R_out, int* bad_index);

double orc_objective_at(const orc_problem* p, const double* R, const int32_t* sigma,
                        double lambda);
double orc_hamiltonian_at(const orc_problem* p, const double* R, const int32_t* sigma,
                          double lambda);
double orc_hamiltonian(int N, int M, const double* A, const double* y, const double* R,
                       const int32_t* sigma, double lambda);
double orc_objective(int N, int M, const double* A, const double* y, const double* R,
                     const int32_t* sigma, double lambda);
double orc_rmse(int N, const double* R, const int32_t* sigma, const double* x,
                const int32_t* xi);
double orc_hamming(int N, const int32_t* sigma, const int32_t* xi);
double orc_median(int n, const double* v);

typedef struct {
    int32_t i, support;
    double eta, hamiltonian, rmse, hamming, min_e, median_e;
} orc_record;

/* alternating_minimize.  hist must hold velo+1 records; hist_R / hist_sigma
 * ((velo+1) x N) optional.  Returns 0 ok (trial may still have failed: see
 * *fail_alt >= 0), 1 input_error, 2 config_error. */
int orc_alternating_minimize(const orc_problem* p, int backend, const orc_hyper* h,
                             const double* R_init, orc_rng* rng, int cdp_method,
                             int track_best, double* R_out, int32_t* sigma_out,
                             orc_record* hist, int* n_hist, double* hist_R,
                             int32_t* hist_sigma, int* fail_alt, int* fail_index);

/* Convenience for the batch harness: one (instance, replica) trial whose
 * solver stream is seeded with `seed` (caller applies mix_seed). */
int orc_solve_trial(int N, int M, const double* A, const double* y, const double* x,
                    const int32_t* xi, int mode, int nseg, int gran, int backend,
                    const orc_hyper* h, uint64_t seed, int cdp_method, int track_best,
                    double* R_out, int32_t* sigma_out, orc_record* hist, int* n_hist,
                    int* fail_alt, int* fail_index);

/* Multithreaded batch of independent trials (the run_jobs pool model,
 * tools/main.cpp:305-321).  A/y/x/xi are arrays of per-trial pointers.
 * Returns wall seconds. */
double orc_solve_batch(int ntrials, int nthreads, int N, const int* M, const double* const* A,
                       const double* const* y, const double* const* x,
                       const int32_t* const* xi, int mode, int nseg, int gran, int backend,
                       const orc_hyper* h, const uint64_t* seeds, int cdp_method,
                       double* R_out, int32_t* sigma_out, int* fail_alt);

/* Bounded CPU-baseline sample: the first alt_limit alternations per trial. */
double orc_solve_batch_limited(int ntrials, int nthreads, int alt_limit, int N, const int* M,
                               const double* const* A, const double* const* y, int mode,
                               int backend, const orc_hyper* h, const uint64_t* seeds,
                               double* R_out, int32_t* sigma_out);

#ifdef __cplusplus
}
#endif
#endif
