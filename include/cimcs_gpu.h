/*
 * cimcs_gpu.h -- C ABI of the B200 MFZ-CIM L0RBCS hot path (libcimcs_gpu.so).
 *
 * The reference (arXiv 2405.00366, /root/reference/proj) is CPU-only C++;
 * its solver seams are C++ (std::function closures, Eigen vectors).  This
 * header is the thin C layer the reference's solver API calls into so the
 * GPU path is a drop-in.  Every entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj).  Plain pointers and
 * sizes only; all host buffers are caller-owned; every call is synchronous
 * on return.  Host vectors are trajectory-major: element (b, r, i) of a
 * B x R x N array is at ((b * R) + r) * N + i, where b = instance,
 * r = replica, i = spin.
 *
 * Status codes mirror the reference's exception types (types.hpp:16-33):
 *   0 ok, 1 input_error, 2 config_error, 3 divergence_error, 4 cuda error.
 * The message of the last failing call on this thread: cimcs_last_error().
 */
#ifndef CIMCS_GPU_H
#define CIMCS_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CIMCS_ABI_VERSION 1

enum { CIMCS_OK = 0, CIMCS_INPUT_ERROR = 1, CIMCS_CONFIG_ERROR = 2,
       CIMCS_DIVERGENCE = 3, CIMCS_CUDA_ERROR = 4 };
/* Context arithmetic.  F64: every quantity in fp64, in the documented
 * canonical order (bitwise-reproducible; cimcs_canon_order).  F32: fp32 state,
 * coupling on the tcgen05 tensor cores (N > 512) or fp32 CUDA cores. */
enum { CIMCS_F32 = 0, CIMCS_F64 = 1 };
/* == Backend {MfzCN, MfzBN, PositiveP}, orchestrator.hpp:28 */
enum { CIMCS_MFZ_CN = 0, CIMCS_MFZ_BN = 1, CIMCS_PP = 2 };
/* == CdpMethod {Jacobi, ConjugateGradient}, cdp.hpp:60 */
enum { CIMCS_CDP_JACOBI = 0, CIMCS_CDP_CG = 1 };
enum { CIMCS_PUMP_SIGMOID = 0, CIMCS_PUMP_LINEAR = 1 };

/* HyperParams, types.hpp:77-96, plus the two BASELINE-config extensions
 * (linear pump ramp).  Field order is part of the ABI. */
typedef struct cimcs_hyper {
    double g2, j, K, beta, tau, dt;
    int32_t n_steps;
    double p_thr, d, eta_init, eta_end;
    int32_t velo;
    double dt_c;
    int32_t jacobi_iters, cg_max_iters;
    double cg_tol, gamma;
    int32_t mfz_loss_minus_j;
    double mu_abort;
    int32_t pump_kind;   /* CIMCS_PUMP_SIGMOID (reference, orchestrator.cpp:12-14) or LINEAR */
    double pump_end;     /* LINEAR: p(t) = (pump_end * t) / (n_steps * dt) */
} cimcs_hyper;

/* AlternationRecord, orchestrator.hpp:100-111 (seconds omitted; support added) */
typedef struct cimcs_record {
    int32_t i, support;
    double eta, hamiltonian, rmse, hamming, min_e, median_e;
} cimcs_record;

/* Device-side timing of the last solve/run_cim, CUDA events on the context
 * stream; launches = number of this library's kernels launched. */
typedef struct cimcs_timing {
    double total_ms;      /* whole call, device time */
    double gram_ms;       /* K1 builder */
    double cim_ms;        /* K2 fused Euler steps (all alternations) */
    double refit_ms;      /* K3 masked Jacobi refit */
    double score_ms;      /* K4 scorer + median */
    double h2d_ms, d2h_ms;
    int64_t step_launches, refit_launches, other_launches;
    double step_bytes;    /* algorithmic bytes of one step launch (G share, dense) */
    double step_flops;    /* algorithmic flops of one step launch (2 N^2 R B) */
    double tile_kernel_ms;        /* option "kernel_timing" (eager launches only): summed  */
    int64_t tile_kernel_launches; /*   CUDA-event time of the step-mode tile-kernel launches */
} cimcs_timing;

typedef struct cimcs_ctx cimcs_ctx;

/* ---------------------------------------------------------- utilities */
int cimcs_abi_version(void);
const char* cimcs_last_error(void);
/* types.hpp:77-96 / :98-106 */
void cimcs_hyper_default(cimcs_hyper* h);
int cimcs_hyper_validate(const cimcs_hyper* h);
/* splitmix64 seed mixing, tools/main.cpp:263-268 */
uint64_t cimcs_mix_seed(uint64_t base, uint64_t salt);
/* The fixed summation order of every G*v contraction (fp64 path is bitwise
 * reproducible against the oracle's ORC_CANON mode with these values). */
int cimcs_gemv_order(int dtype, int32_t* nseg, int32_t* gran);
/* The canonical fp64 contraction order of a context's resident problems, as
 * the oracle's ORC_CANON (nseg, gran): (ceil(N/512), 512) on the DMMA symmetric
 * path (unsharded fp64, N > 512), (8, 8) on the grid / cluster kernels.  Replaces
 * nothing in the reference (its Eigen GEMV order is unpinnable); it is the
 * reproducibility contract of the fp64 path. */
int cimcs_canon_order(const cimcs_ctx* ctx, int32_t* nseg, int32_t* gran);

/* Host instance generator: gen_instance, datagen.cpp:15-55 (same seeded
 * stream and draw order; std::mt19937_64 + Box-Muller as rng.hpp:21-64).
 * A is M x N column-major (ProblemInstance::A layout). */
int cimcs_gen_dims(int32_t N, double alpha, double a, int32_t* M, int32_t* K);
int cimcs_gen_instance(int32_t N, double alpha, double a, double nu, uint64_t seed,
                       double* A, double* y, double* x_true, int32_t* xi_true);
/* Batch of instances on `threads` host threads (instance_grid/run_jobs,
 * tools/main.cpp:305-344).  Arrays of per-instance pointers. */
int cimcs_gen_instances(int32_t B, int32_t N, const double* alpha, const double* a,
                        const double* nu, const uint64_t* seeds, double* const* A,
                        double* const* y, double* const* x_true, int32_t* const* xi_true,
                        int32_t threads);

/* ----------------------------------------- bundles and CSV (host, io.hpp) */
/* format_double, io.hpp:13 / io.cpp:18-25: shortest text that round-trips. */
int cimcs_format_double(double v, char* buf, int32_t cap);
/* fnv1a64, io.hpp:16 / io.cpp:27-34 */
uint64_t cimcs_fnv1a64(const char* bytes, uint64_t n);
/* save_instance, io.hpp:20-28 / io.cpp:86-125.  A is M x N column-major;
 * x_true / xi_true may be NULL (no truth.csv). */
int cimcs_save_instance(const char* dir, int32_t N, int32_t M, const double* A, const double* y,
                        const double* x_true, const int32_t* xi_true, double a, double alpha,
                        double nu, uint64_t seed);
/* load_instance, io.hpp:29 / io.cpp:127-167, in two calls: A == NULL reads
 * meta.json (N, M, has_truth, a, alpha, nu, seed); then, with *N / *M as
 * returned and caller-sized arrays, the CSVs (x_true / xi_true filled only
 * when has_truth).  Row / column count mismatches are input errors. */
int cimcs_load_instance(const char* dir, int32_t* N, int32_t* M, int32_t* has_truth, double* a,
                        double* alpha, double* nu, uint64_t* seed, double* A, double* y,
                        double* x_true, int32_t* xi_true);
/* CsvWriter, io.hpp:31-48 / io.cpp:169-196: "# " comment lines, header,
 * rows of exactly ncols cells (else input_error); written on close. */
typedef struct cimcs_csv cimcs_csv;
int cimcs_csv_open(const char* path, const char* const* comments, int32_t ncomments,
                   const char* const* columns, int32_t ncols, cimcs_csv** out);
int cimcs_csv_row(cimcs_csv* w, const char* const* cells, int32_t n);
int cimcs_csv_close(cimcs_csv* w);

/* Tile sharding of the symmetric path (sharded contexts, option "tile_shard"):
 * the super-rows [P0, P1) (4 row blocks of 128 each) whose upper-triangle gram
 * tiles rank `rank` of `world` streams, contiguous and balanced by tile count. */
int cimcs_tile_shard(int32_t nRB, int32_t world, int32_t rank, int32_t* P0, int32_t* P1);
/* make_mask, mri.hpp:45 / mri.cpp:185-207: M distinct k-space positions of an
 * H x W grid (reference Rng, partial Fisher-Yates), sorted into out[M]. */
int cimcs_make_mask(int32_t H, int32_t W, int32_t M, uint64_t seed, int32_t* out);

/* ------------------------------------------------------------ context */
/* One per host thread; owns device buffers, one CUDA stream and graphs. */
int cimcs_create(int32_t device, int32_t dtype, cimcs_ctx** out);
/* Row-sharded context (one process per GPU, config 4): rank owns whole
 * 128-spin row blocks [rank*per, (rank+1)*per) of every instance's gram and
 * the state of those spins; the contraction input is all-gathered (NCCL)
 * after every Euler step and Jacobi sweep inside the CUDA graphs.  No C ABI
 * call changes meaning; every rank receives full result vectors.
 * cimcs_nccl_unique_id fills 128 bytes on one rank, to be broadcast. */
int cimcs_nccl_unique_id(uint8_t* out, int32_t nbytes);
int cimcs_create_sharded(int32_t device, int32_t dtype, int32_t world, int32_t rank,
                         const uint8_t* nccl_id, cimcs_ctx** out);
void cimcs_destroy(cimcs_ctx* ctx);
/* key: "host_threads" (c0 generator pool), "use_graphs" (0/1), "tensor_cores" (0/1,
 * fp32 contexts, before cimcs_set_problems). */
int cimcs_set_option(cimcs_ctx* ctx, const char* key, int64_t value);

/* B problems of equal N (make_problem(inst), orchestrator.cpp:80-99).
 * A[b]: M[b] x N column-major, y[b]: M[b].  x_true/xi_true may be NULL
 * (metrics then NaN, as SolverProblem::rmse_at, orchestrator.cpp:70-78). */
int cimcs_set_problems(cimcs_ctx* ctx, int32_t B, int32_t N, const int32_t* M,
                       const double* const* A, const double* const* y,
                       const double* const* x_true, const int32_t* const* xi_true);
/* K1: G = A^T A (gram, full diagonal), hz = A^T y, D = diag(G), device
 * resident.  Replaces coupling_from_observation (model.cpp:54-63) and the
 * per-step matrix-free A^T(A w) (orchestrator.cpp:86-88): J w = D∘w - G w. */
/* a DOCUMENTED DEVIATION for config-4-scale runs: B
 * instances with gen_instance's recipe and shapes (datagen.cpp:15-55) drawn on
 * the GPU from counter-based Philox4x32-10 streams instead of the reference's
 * sequential mt19937_64 stream, so they are NOT the reference's instances
 * (never used for parity).  Replaces cimcs_set_problems (A, y, x, xi resident). */
int cimcs_set_generated_problems(cimcs_ctx* ctx, int32_t B, int32_t N, const double* alpha,
                                 const double* a, const double* nu, const uint64_t* seeds);
/* The resident instance b back on the host (A column-major M x N; x/xi when
 * ground truth is set); e.g. to hand a generated instance to save_instance. */
int cimcs_get_instance(cimcs_ctx* ctx, int32_t b, double* A, double* y, double* x_true,
                       int32_t* xi_true);
int cimcs_build_coupling(cimcs_ctx* ctx);
/* Matrix-free transform-chain problem: MriTransform(target_image, mask, gamma)
 * + make_problem(t, &truth) (mri.hpp:46-99, mri.cpp:209-256, 393-411).
 * target is H x W row-major (H, W powers of two in [2, 128]), mask the M
 * sampled k-space indices (unique, in range), x_true the Haar coefficients of
 * the target (nullable; xi = x != 0).  B = 1, fp32 contexts only.  Then
 * cimcs_build_coupling computes hz = Re(A^H y) and diag(G); the quadratic form
 * G = Re(A^H A) + gamma Psi (Dv'Dv + Dh'Dh) Psi' is applied matrix-free every
 * step (mri_kernels.cuh).  Refits always use CG (orchestrator.cpp:128-133);
 * damped Jacobi is a config_error (cdp.cpp:158-159).  get_coupling returns
 * G by applying the chain to every basis vector. */
int cimcs_set_mri_problem(cimcs_ctx* ctx, int32_t H, int32_t W, const double* target,
                          int32_t M, const int32_t* mask, double gamma, const double* x_true);
/* BASELINE config 3 as a matrix-free chain (dct_kernels.cuh): the dense
 * config-3 instance has A = S C2 Psi_L^-1 (row m = the L-level orthonormal
 * Mallat Haar transform -- the reference's average / difference split,
 * mri.cpp:30-48 / 122-165, stopped after L levels -- of the orthonormal 2-D
 * DCT-II basis image of frequency freqs[m] = u * n + v) and observations y[M].
 * The context keeps only the DCT matrix, the frequency mask and y on the
 * frequency grid; every G w is Psi C^T (mask o (C Psi^-1 w C^T)) C, hz = A^T y
 * and D = diag(G) come from the same chain.  n must be 128, 1 <= levels <= 3,
 * fp32 single-GPU contexts.  Unlike the DFT chain, damped Jacobi refits are
 * allowed (this is the dense problem's G).  x_true (N) optional. */
int cimcs_set_dct_problem(cimcs_ctx* ctx, int32_t n, int32_t levels, int32_t M,
                          const int32_t* freqs, const double* y, const double* x_true);
/* lasso_init(t, lambda) (mri.cpp:372-377 -> lasso_normal_form :345-370): FISTA
 * warm start on the built MRI problem with G = Re(A^H A), step `step` (1 in
 * the reference), stop when |f - f_prev| <= tol max(1, |f_prev|) or after
 * max_iters iterations.  x_out[N] (fp32 chain, fp64 objective), the iteration
 * count and the final objective. */
int cimcs_mri_lasso(cimcs_ctx* ctx, double lambda, int32_t max_iters, double tol, double step,
                    double* x_out, int32_t* iterations, double* objective);
/* Copy instance b's coupling back (fp64 host buffers; N*N, N, N).  Test aid. */
int cimcs_get_coupling(cimcs_ctx* ctx, int32_t b, double* G, double* hz, double* D);

/* One Euler step for all B x R trajectories from given (c, e):
 * local_field_{continuous,binarized} (solver_mfz.cpp:33-59) + mfz_step
 * (:61-88).  h_out (optional) receives the local field.  fail_index[b*R+r]
 * = first non-finite spin or -1.  Returns 3 if any trajectory diverged. */
int cimcs_mfz_step(cimcs_ctx* ctx, int32_t R, int32_t backend, const cimcs_hyper* hp,
                   double eta, double p, const double* Rsig, const double* c,
                   const double* e, double* c_out, double* e_out, double* h_out,
                   int32_t* fail_index);

/* One CIM call for all B x R trajectories: run_cim / run_mfz
 * (orchestrator.cpp:140-161, solver_mfz.cpp:90-124).  c0 = the initial
 * amplitudes (0.01 * gauss from each trajectory's stream, init_mfz
 * solver_mfz.cpp:24-31); per-trajectory divergence freezes that
 * trajectory only (fail_index >= 0) and the call returns 3. */
int cimcs_run_cim(cimcs_ctx* ctx, int32_t R, int32_t backend, const cimcs_hyper* hp,
                  double eta, const double* Rsig, const double* c0, double* c_out,
                  double* e_out, int32_t* sigma_out, double* min_e, int32_t* fail_index);

/* One Positive-P CIM call (run_pp, solver_pp.cpp:100-132; backend
 * Backend::PositiveP) for all B x R trajectories.  seeds[b*R+r] seeds the
 * trajectory's reference stream (N unit normals per step, drawn on the host
 * bit-exactly and streamed to the device).  Outputs: final mu, e, the last
 * measured amplitude mu~ and sigma = [mu~ > 0].  fp64 contexts or fp32 with
 * tensor_cores = 0 (config_error otherwise).  Returns 3 on divergence
 * (non-finite value or |mu| > mu_abort; fail_index = offending spin). */
int cimcs_run_pp(cimcs_ctx* ctx, int32_t R, const cimcs_hyper* hp, double eta,
                 const double* Rsig, const uint64_t* seeds, double* mu_out, double* e_out,
                 double* mt_out, int32_t* sigma_out, double* min_e, int32_t* fail_index);

/* Masked refit on each trajectory's support: cdp_minimize with damped
 * Jacobi (cdp.cpp:48-64, 132-139).  Entries with sigma = 0 are returned
 * bitwise untouched.  Singular active diagonal -> input_error. */
int cimcs_refit(cimcs_ctx* ctx, int32_t R, const int32_t* sigma, const double* R_prev,
                double* R_out, const cimcs_hyper* hp);

/* cdp_minimize(inst, sigma, R_prev, method, params) (cdp.cpp:132-139) for all
 * B x R trajectories: method CIMCS_CDP_JACOBI (jacobi_solve, cdp.cpp:48-64;
 * same as cimcs_refit) or CIMCS_CDP_CG (cg_solve, cdp.cpp:66-105: stops at
 * |r| <= cg_tol*|b| or cg_max_iters, breakdown when p.Gp <= 0).  iterations
 * (optional, B x R) receives CgInfo::iterations (jacobi_iters for Jacobi).
 * CG is not available on row-sharded contexts (config_error). */
int cimcs_cdp_minimize(cimcs_ctx* ctx, int32_t R, const int32_t* sigma, const double* R_prev,
                       int32_t method, const cimcs_hyper* hp, double* R_out,
                       int32_t* iterations);

/* K4 scorer: objective_at (orchestrator.cpp:57-62), rmse / hamming_loss
 * (model.cpp:128-153).  Outputs are B x R. */
int cimcs_score(cimcs_ctx* ctx, int32_t R, const double* Rsig, const int32_t* sigma,
                double lambda, double* objective, double* rmse, double* hamming);

/* The whole alternating loop for all B x R trajectories:
 * alternating_minimize (orchestrator.cpp:170-235) with R_init = hz
 * (default_r_init, :138) unless R_init != NULL.  seeds[b*R + r] seeds
 * trajectory (b, r)'s std::mt19937_64 stream (the reference's Rng), which
 * supplies N normals per alternation for c0.  hist holds (velo+1)*B*R
 * records, trajectory-major; n_hist[b*R+r] = recorded alternations;
 * fail_alt = alternation that diverged or -1 (AlternatingResult::failed,
 * orchestrator.hpp:113-124).  cdp: CIMCS_CDP_JACOBI or CIMCS_CDP_CG.
 * backend CIMCS_PP runs run_pp per alternation (see cimcs_run_pp). */
int cimcs_solve(cimcs_ctx* ctx, int32_t R, int32_t backend, const cimcs_hyper* hp,
                int32_t cdp, const uint64_t* seeds, const double* R_init,
                int32_t track_best, double* R_out, int32_t* sigma_out,
                cimcs_record* hist, int32_t* n_hist, int32_t* fail_alt,
                int32_t* fail_index);

int cimcs_get_timing(const cimcs_ctx* ctx, cimcs_timing* out);

/* Measurement aid with no reference counterpart (option "timeline" = 1 first): the
 * %globaltimer stamps (ns) of the LAST symmetric tile / update launch pair, 4 per CTA --
 * tile CTA x at out[4x..] = (entry, past the PDL wait, last item stored, 0), update
 * CTA x of instance b at out[4 (256 + b gridDim.x + x)..] = (entry, past the PDL wait /
 * item flags, exit, 0); tile CTA 0's per-tile stamps at out[4 (8192 + t)..] and
 * out[4 (8320 + t)..] (csrc/sym_kernels.cuh).  *n = the number of values written (<= cap). */
int cimcs_get_timeline(cimcs_ctx* ctx, uint64_t* out, int64_t cap, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif
