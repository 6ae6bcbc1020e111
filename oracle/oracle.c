/*
 * oracle.c -- CPU restatement of the reference MFZ-CIM L0RBCS hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled like the reference:
 * -O3, no -march, -ffp-contract=off (no silent FMA contraction); fma() is
 * called explicitly only where the canonical GPU order uses it.
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ===================================================================== RNG
 * rng.hpp:21-64: std::mt19937_64 (restated from the published MT19937-64
 * algorithm), uniform_open = ((raw >> 11) + 1) * 2^-53, Box-Muller with two
 * uniforms per normal and no pair caching. */
#define MT_N 312
#define MT_M 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void orc_rng_init(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
    r->n_gauss = 0;
}

uint64_t orc_rng_raw(orc_rng* r) {
    if (r->mti >= MT_N) {
        int i;
        for (i = 0; i < MT_N - MT_M; ++i) {
            uint64_t x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
        }
        for (; i < MT_N - 1; ++i) {
            uint64_t x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
        }
        uint64_t x = (r->mt[MT_N - 1] & MT_UM) | (r->mt[0] & MT_LM);
        r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:28-31 */
double orc_uniform_open(orc_rng* r) {
    const uint64_t u = orc_rng_raw(r) >> 11;
    return ((double)u + 1.0) * 0x1.0p-53;
}

/* rng.hpp:34-41 */
uint64_t orc_uniform_below(orc_rng* r, uint64_t bound) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t v;
    do {
        v = orc_rng_raw(r);
    } while (v >= limit);
    return v % bound;
}

/* rng.hpp:44-49 (kPi at :62) */
double orc_gauss(orc_rng* r) {
    static const double kPi = 3.14159265358979323846;
    const double u1 = orc_uniform_open(r);
    const double u2 = orc_uniform_open(r);
    r->n_gauss++;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * kPi * u2);
}

/* tools/main.cpp:263-268 */
uint64_t orc_mix_seed(uint64_t base, uint64_t salt) {
    uint64_t z = base + 0x9E3779B97F4A7C15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* datagen.cpp:11-13 */
long long orc_round_half_away(double v) {
    return (long long)(v < 0 ? ceil(v - 0.5) : floor(v + 0.5));
}

/* ================================================================= datagen */
/* datagen.cpp:17-24 */
int orc_gen_dims(int N, double alpha, double a, int* M, int* K) {
    if (N < 1) return 1;
    if (!(alpha > 0.0) || alpha > 1.0) return 1;
    if (a < 0.0 || a > 1.0) return 1;
    const int m = (int)orc_round_half_away(alpha * (double)N);
    if (m < 1) return 1;
    if (M) *M = m;
    if (K) *K = (int)orc_round_half_away(a * (double)N);
    return 0;
}

/* datagen.cpp:15-55.  Draw order: A row-major (k outer, r inner), x, support
 * positions by partial Fisher-Yates, observation noise. */
int orc_gen_instance(int N, double alpha, double a, double nu, uint64_t seed, double* A,
                     double* y, double* x, int32_t* xi) {
    int M, K;
    if (orc_gen_dims(N, alpha, a, &M, &K)) return 1;
    if (nu < 0.0) return 1;
    orc_rng rng;
    orc_rng_init(&rng, seed);
    const double col_std = 1.0 / sqrt((double)M);
    for (int k = 0; k < M; ++k)
        for (int r = 0; r < N; ++r) A[(size_t)r * M + k] = col_std * orc_gauss(&rng);
    for (int r = 0; r < N; ++r) x[r] = orc_gauss(&rng);
    int* idx = (int*)malloc(sizeof(int) * (size_t)N);
    for (int r = 0; r < N; ++r) {
        idx[r] = r;
        xi[r] = 0;
    }
    for (int i = 0; i < K; ++i) {
        const int pick = i + (int)orc_uniform_below(&rng, (uint64_t)(N - i));
        const int tmp = idx[i];
        idx[i] = idx[pick];
        idx[pick] = tmp;
        xi[idx[i]] = 1;
    }
    free(idx);
    /* y = A w, w = xi o x; per row sequential over columns */
    for (int k = 0; k < M; ++k) y[k] = 0.0;
    for (int r = 0; r < N; ++r) {
        const double w = xi[r] ? x[r] : 0.0;
        const double* col = A + (size_t)r * M;
        for (int k = 0; k < M; ++k) y[k] = y[k] + col[k] * w;
    }
    for (int k = 0; k < M; ++k) y[k] += nu * orc_gauss(&rng);
    return 0;
}

/* =============================================================== schedules */
/* orchestrator.cpp:12-14 */
double orc_pump_sigmoid(double t, double p_thr, double d) {
    return (p_thr - d) + 2.0 * d / (1.0 + exp(-(t - 4.0) / 2.0));
}

/* ⊕ linear ramp 0 -> p_end over T = n_steps*dt (BASELINE configs) */
double orc_pump_linear(double t, double p_end, double T) { return p_end * t / T; }

/* orchestrator.cpp:16-20; std::max(a,b) = (a < b) ? b : a */
double orc_eta_schedule(int i, double eta_init, double eta_end, int velo) {
    if (velo < 1) return NAN;
    const double linear = eta_init * (1.0 - (double)i / velo);
    return (linear < eta_end) ? eta_end : linear;
}

/* solver_mfz.cpp:17-22 */
int orc_trace_stride(int n_steps, int cap) {
    if (n_steps < cap) return 1;
    return (n_steps + cap - 2) / (cap - 1);
}

/* types.hpp:77-96 */
void orc_hyper_default(orc_hyper* h) {
    h->g2 = 1e-7;
    h->j = 1.0;
    h->K = 1.0;
    h->beta = 0.2;
    h->tau = 1.0;
    h->dt = 0.02;
    h->n_steps = 1000;
    h->p_thr = 1.0;
    h->d = 0.4;
    h->eta_init = 0.8;
    h->eta_end = 0.18;
    h->velo = 51;
    h->dt_c = 0.1;
    h->jacobi_iters = 100;
    h->cg_max_iters = 10000;
    h->cg_tol = 1e-10;
    h->gamma = 1e-4;
    h->mfz_loss_minus_j = 0;
    h->mu_abort = 100.0;
    h->pump_kind = ORC_PUMP_SIGMOID;
    h->pump_end = 1.2;
}

/* types.hpp:98-106 */
int orc_hyper_validate(const orc_hyper* h) {
    if (!(h->dt > 0)) return 2;
    if (h->n_steps < 1) return 2;
    if (!(h->tau > 0)) return 2;
    if (h->g2 < 0) return 2;
    if (h->eta_init < h->eta_end || h->eta_end < 0) return 2;
    if (h->velo < 1) return 2;
    if (h->pump_kind != ORC_PUMP_SIGMOID && h->pump_kind != ORC_PUMP_LINEAR) return 2;
    return 0;
}

/* The pump seen at step k is evaluated at the accumulated t (t += dt,
 * solver_mfz.cpp:86,107). */
void orc_pump_table(const orc_hyper* h, double* p) {
    double t = 0.0;
    const double T = (double)h->n_steps * h->dt;
    for (int k = 0; k < h->n_steps; ++k) {
        p[k] = h->pump_kind == ORC_PUMP_LINEAR ? orc_pump_linear(t, h->pump_end, T)
                                               : orc_pump_sigmoid(t, h->p_thr, h->d);
        t = t + h->dt;
    }
}

/* ================================================================= problem */
/* Canonical segmented order: segment s = {j : (j / gran) % nseg == s}; each
 * segment is an fma chain over ascending j starting from +0.0; the segment
 * partials are then added left to right.  fma() is correctly rounded in both
 * the hardware and the libm path, so the dispatch below changes speed only.
 * The GPU uses (nseg, gran) = (8, 8) on its grid / cluster kernels and
 * (ceil(N / 512), 512) -- contiguous 512-column segments -- on the fp64 DMMA
 * symmetric-tile path (cimcs_canon_order; sym64_kernels.cuh derives it). */
#define CANON_BODY                                                                  \
    double P[256];                                                              \
    for (int s = 0; s < nseg; ++s) P[s] = 0.0;                                  \
    int s = 0;                                                                  \
    for (int j0 = 0; j0 < N; j0 += gran) {                                      \
        const int j1 = j0 + gran < N ? j0 + gran : N;                           \
        double acc = P[s];                                                      \
        for (int j = j0; j < j1; ++j) acc = fma(g[j], v[j], acc);               \
        P[s] = acc;                                                             \
        if (++s == nseg) s = 0;                                                 \
    }                                                                           \
    double acc = P[0];                                                          \
    for (int q = 1; q < nseg; ++q) acc = acc + P[q];                            \
    return acc;

__attribute__((target("fma"))) static double canon_dot_hw(const double* g, const double* v,
                                                           int N, int nseg, int gran) {
    CANON_BODY
}

static double canon_dot_sw(const double* g, const double* v, int N, int nseg, int gran) {
    CANON_BODY
}

double orc_canon_dot(const double* g, const double* v, int N, int nseg, int gran) {
    static int have_fma = -1;
    if (have_fma < 0) have_fma = __builtin_cpu_supports("fma") ? 1 : 0;
    return have_fma ? canon_dot_hw(g, v, N, nseg, gran) : canon_dot_sw(g, v, N, nseg, gran);
}

static double seq_dot(const double* a, const double* b, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = s + a[i] * b[i];
    return s;
}

/* sequential-k fma chain (the canonical Gram entry order) */
__attribute__((target("fma"))) static double fma_chain_hw(const double* a, const double* b,
                                                          int n) {
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = fma(a[k], b[k], acc);
    return acc;
}

static double fma_chain_sw(const double* a, const double* b, int n) {
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = fma(a[k], b[k], acc);
    return acc;
}

static double fma_chain(const double* a, const double* b, int n) {
    return __builtin_cpu_supports("fma") ? fma_chain_hw(a, b, n) : fma_chain_sw(a, b, n);
}

/* make_problem(inst) orchestrator.cpp:80-99 / coupling_from_observation
 * model.cpp:54-63 (as G = A^T A; J = D - G is never formed). */
int orc_problem_init(orc_problem* p, int N, int M, const double* A, const double* y,
                     int mode, int nseg, int gran) {
    memset(p, 0, sizeof(*p));
    p->N = N;
    p->M = M;
    p->A = A;
    p->y = y;
    p->mode = mode;
    p->nseg = nseg > 0 ? nseg : 8;
    p->gran = gran > 0 ? gran : 8;
    if (p->nseg > 256) return 1;
    p->hz = (double*)malloc(sizeof(double) * (size_t)N);
    p->D = (double*)malloc(sizeof(double) * (size_t)N);
    p->work = (double*)malloc(sizeof(double) * (size_t)(M > N ? M : N));
    if (mode == ORC_LITERAL) {
        for (int r = 0; r < N; ++r) {
            const double* col = A + (size_t)r * M;
            p->hz[r] = seq_dot(col, y, M);
            p->D[r] = seq_dot(col, col, M);
        }
        return 0;
    }
    p->G = (double*)malloc(sizeof(double) * (size_t)N * N);
    for (int i = 0; i < N; ++i) {
        const double* ci = A + (size_t)i * M;
        for (int j = i; j < N; ++j) {
            const double* cj = A + (size_t)j * M;
            double acc = 0.0;
            if (mode == ORC_CANON)
                acc = fma_chain(ci, cj, M);
            else
                for (int k = 0; k < M; ++k) acc = acc + ci[k] * cj[k];
            p->G[(size_t)i * N + j] = acc;
            p->G[(size_t)j * N + i] = acc;
        }
        double acc = 0.0;
        if (mode == ORC_CANON)
            acc = fma_chain(ci, y, M);
        else
            for (int k = 0; k < M; ++k) acc = acc + ci[k] * y[k];
        p->hz[i] = acc;
        p->D[i] = p->G[(size_t)i * N + i];
    }
    return 0;
}

/* make_problem(G_full, hz), orchestrator.cpp:100-115 (and, restated through the
 * assembled matrix, the operator form make_problem(N, apply, diag, hz) :117-136):
 * mode EXPLICIT with G given (row-major N x N, copied), no A. */
int orc_problem_init_gram(orc_problem* p, int N, const double* G, const double* hz) {
    memset(p, 0, sizeof(*p));
    p->N = N;
    p->M = 0;
    p->mode = ORC_EXPLICIT;
    p->nseg = 8;
    p->gran = 8;
    p->hz = (double*)malloc(sizeof(double) * (size_t)N);
    p->D = (double*)malloc(sizeof(double) * (size_t)N);
    p->work = (double*)malloc(sizeof(double) * (size_t)N);
    p->G = (double*)malloc(sizeof(double) * (size_t)N * N);
    if (!p->hz || !p->D || !p->work || !p->G) return 1;
    memcpy(p->G, G, sizeof(double) * (size_t)N * N);
    memcpy(p->hz, hz, sizeof(double) * (size_t)N);
    for (int i = 0; i < N; ++i) p->D[i] = G[(size_t)i * N + i];
    return 0;
}

void orc_problem_free(orc_problem* p) {
    free(p->G);
    free(p->hz);
    free(p->D);
    free(p->work);
    memset(p, 0, sizeof(*p));
}

/* apply_gram (orchestrator.cpp:86-88 / :333) */
void orc_gram_apply(const orc_problem* p, const double* w, double* out) {
    const int N = p->N, M = p->M;
    if (p->mode == ORC_LITERAL) {
        double* u = p->work;
        for (int k = 0; k < M; ++k) u[k] = 0.0;
        for (int r = 0; r < N; ++r) {
            const double* col = p->A + (size_t)r * M;
            const double wr = w[r];
            for (int k = 0; k < M; ++k) u[k] = u[k] + col[k] * wr;
        }
        for (int r = 0; r < N; ++r) out[r] = seq_dot(p->A + (size_t)r * M, u, M);
    } else if (p->mode == ORC_CANON) {
        for (int i = 0; i < N; ++i)
            out[i] = orc_canon_dot(p->G + (size_t)i * N, w, N, p->nseg, p->gran);
    } else {
        for (int i = 0; i < N; ++i) out[i] = seq_dot(p->G + (size_t)i * N, w, N);
    }
}

/* SolverProblem::apply_coupling orchestrator.cpp:45-47: D∘w - G w */
void orc_coupling_apply(const orc_problem* p, const double* w, double* out) {
    double* g = (double*)malloc(sizeof(double) * (size_t)p->N);
    orc_gram_apply(p, w, g);
    for (int r = 0; r < p->N; ++r) out[r] = p->D[r] * w[r] - g[r];
    free(g);
}

/* solver_mfz.cpp:33-40 */
void orc_local_field_cn(const orc_problem* p, const double* R, const double* c, double tau,
                        double* h) {
    const int N = p->N;
    const double rt = sqrt(tau);
    double* w = (double*)malloc(sizeof(double) * (size_t)N);
    for (int r = 0; r < N; ++r) w[r] = R[r] * 0.25 * (c[r] + rt);
    orc_coupling_apply(p, w, h);
    for (int r = 0; r < N; ++r) h[r] = h[r] + (rt / 2.0) * p->hz[r];
    free(w);
}

/* solver_mfz.cpp:47-54 */
void orc_local_field_bn(const orc_problem* p, const double* R, const int32_t* sigma,
                        double tau, double* h) {
    const int N = p->N;
    const double rt = sqrt(tau);
    double* w = (double*)malloc(sizeof(double) * (size_t)N);
    for (int r = 0; r < N; ++r) w[r] = R[r] * (double)sigma[r];
    orc_coupling_apply(p, w, h);
    for (int r = 0; r < N; ++r) h[r] = (rt / 2.0) * (h[r] + p->hz[r]);
    free(w);
}

/* solver_mfz.cpp:61-88 */
int orc_mfz_step(int N, const double* c_in, const double* e_in, double p, const orc_hyper* h,
                 double eta, const double* R, const double* hf, double* c_out, double* e_out) {
    if (!isfinite(p)) return -2;
    const double rt = sqrt(h->tau);
    const double thresh = eta * eta / 4.0 * rt;
    const double loss = h->mfz_loss_minus_j ? (-1.0 + p - h->j) : (-1.0 + p);
    for (int r = 0; r < N; ++r) {
        const double c = c_in[r];
        const double e = e_in[r];
        const double inj = h->K * h->j * e * (R[r] * hf[r] - thresh);
        c_out[r] = c + h->dt * ((loss - c * c) * c + inj);
        e_out[r] = e + h->dt * (-h->beta * (c * c - h->tau) * e);
        if (!isfinite(c_out[r]) || !isfinite(e_out[r])) return r;
    }
    return -1;
}

/* ============================================================ Positive-P */
/* measured_amplitude solver_pp.cpp:22-29: mu + sqrt(g2/(4 j dt)) w */
int orc_measured_amplitude(int N, const double* mu, const double* noise, const orc_hyper* h,
                           double* mt) {
    if (!(h->j > 0.0)) return 2;
    const double scale = sqrt(h->g2 / (4.0 * h->j * h->dt));
    for (int r = 0; r < N; ++r) mt[r] = mu[r] + scale * noise[r];
    return 0;
}

/* local_field_pp solver_pp.cpp:31-38: w = (R*0.5)*(mt + rt); h = J w + rt*hz */
void orc_local_field_pp(const orc_problem* p, const double* R, const double* mt, double tau,
                        double* out) {
    const int N = p->N;
    const double rt = sqrt(tau);
    double* w = (double*)malloc(sizeof(double) * (size_t)N);
    for (int r = 0; r < N; ++r) w[r] = R[r] * 0.5 * (mt[r] + rt);
    orc_coupling_apply(p, w, out);
    for (int r = 0; r < N; ++r) out[r] = out[r] + rt * p->hz[r];
    free(w);
}

/* pp_step solver_pp.cpp:45-98 (Euler-Maruyama, same association as the source) */
int orc_pp_step(int N, const double* mu_in, const double* n_in, const double* m_in,
                const double* e_in, double p, const orc_hyper* h, double eta, const double* R,
                const double* hf, const double* noise, double* mu_o, double* n_o, double* m_o,
                double* e_o) {
    const double g2 = h->g2, j = h->j, dt = h->dt;
    const double rt = sqrt(h->tau);
    const double thresh = rt * eta * eta / 4.0;
    const double sdt = sqrt(dt);
    const double scale = sqrt(g2 / (4.0 * j * dt));
    for (int r = 0; r < N; ++r) {
        const double mu = mu_in[r], n = n_in[r], m = m_in[r], e = e_in[r];
        const double mu2 = mu * mu;
        const double mn2 = (m + n) * (m + n);
        const double inj = h->K * j * e * (R[r] * hf[r] - thresh);
        const double drift_mu = -(1.0 - p + j) * mu - mu * (mu2 + 2.0 * g2 * n + g2 * m) + inj;
        const double diff_mu = sqrt(j * g2) * (m + n) * noise[r];
        mu_o[r] = mu + dt * drift_mu + sdt * diff_mu;
        n_o[r] = n + dt * (-2.0 * (1.0 + j) * n + 2.0 * p * m - 2.0 * mu2 * (2.0 * n + m) -
                           j * mn2);
        m_o[r] = m + dt * (-2.0 * (1.0 + j) * m + 2.0 * p * n - 2.0 * mu2 * (2.0 * m + n) + p -
                           (mu2 + g2 * m) - j * mn2);
        const double mt = mu + scale * noise[r];
        e_o[r] = e + dt * (-h->beta * (mt * mt - h->tau) * e);
        if (!isfinite(mu_o[r]) || !isfinite(n_o[r]) || !isfinite(m_o[r]) || !isfinite(e_o[r]))
            return r;
    }
    return -1;
}

/* run_pp solver_pp.cpp:100-132 with init_pp :11-20 */
int orc_run_pp(const orc_problem* p, const double* R, const orc_hyper* h, double eta,
               orc_rng* rng, double* mu_out, double* n_out, double* m_out, double* e_out,
               double* mt_out, int32_t* sigma_out, double* min_e, int* kind) {
    if (orc_hyper_validate(h) || !(h->j > 0.0)) return -3;
    const int N = p->N;
    double* st = (double*)calloc((size_t)N * 8, sizeof(double));
    double *mu = st, *n = st + N, *m = st + 2 * N, *e = st + 3 * N;
    double *mu2 = st + 4 * N, *n2 = st + 5 * N, *m2 = st + 6 * N, *e2 = st + 7 * N;
    double* mt = (double*)calloc((size_t)N, sizeof(double));
    double* noise = (double*)malloc(sizeof(double) * (size_t)N);
    double* hf = (double*)malloc(sizeof(double) * (size_t)N);
    for (int r = 0; r < N; ++r) e[r] = 1.0;
    double t = 0.0, me = 1.0;
    const double T = (double)h->n_steps * h->dt;
    int rc = -1;
    if (kind) *kind = 0;
    for (int step = 0; step < h->n_steps; ++step) {
        const double pp = h->pump_kind == ORC_PUMP_LINEAR ? orc_pump_linear(t, h->pump_end, T)
                                                          : orc_pump_sigmoid(t, h->p_thr, h->d);
        for (int r = 0; r < N; ++r) noise[r] = orc_gauss(rng);
        orc_measured_amplitude(N, mu, noise, h, mt);
        orc_local_field_pp(p, R, mt, h->tau, hf);
        rc = orc_pp_step(N, mu, n, m, e, pp, h, eta, R, hf, noise, mu2, n2, m2, e2);
        if (rc != -1) break;
        double* tmp;
        tmp = mu; mu = mu2; mu2 = tmp;
        tmp = n; n = n2; n2 = tmp;
        tmp = m; m = m2; m2 = tmp;
        tmp = e; e = e2; e2 = tmp;
        t = t + h->dt;
        double emin = e[0];
        for (int r = 1; r < N; ++r)
            if (e[r] < emin) emin = e[r];
        me = emin < me ? emin : me;
        for (int r = 0; r < N; ++r)
            if (fabs(mu[r]) > h->mu_abort) {
                rc = r;
                if (kind) *kind = 1;
                break;
            }
        if (rc != -1) break;
    }
    if (rc == -1) {
        for (int r = 0; r < N; ++r) sigma_out[r] = mt[r] > 0.0 ? 1 : 0;
        if (mu_out) memcpy(mu_out, mu, sizeof(double) * (size_t)N);
        if (n_out) memcpy(n_out, n, sizeof(double) * (size_t)N);
        if (m_out) memcpy(m_out, m, sizeof(double) * (size_t)N);
        if (e_out) memcpy(e_out, e, sizeof(double) * (size_t)N);
        if (mt_out) memcpy(mt_out, mt, sizeof(double) * (size_t)N);
        if (min_e) *min_e = me;
    }
    free(st);
    free(mt);
    free(noise);
    free(hf);
    return rc;
}

/* Precision-sensitivity knob (tools/precision_study.py only; 0 everywhere
 * else): bit 1 rounds the local field to fp32 every step, bit 2 the state c, e
 * after every step, bit 4 the refit R after every alternation, bits 8 / 16 add a
 * uniform relative error of up to 2^-20 / 2^-16 to the field every step.  It measures
 * which fp32 quantity moves the fp64 answer; the reference has no such knob. */
static int g_perturb = 0;
void orc_set_perturb(int mode) { g_perturb = mode; }

/* run_mfz solver_mfz.cpp:90-124 with init_mfz :24-31 */
int orc_run_mfz(const orc_problem* p, const double* R, const orc_hyper* h, double eta,
                int backend, orc_rng* rng, double* c_out, double* e_out, int32_t* sigma_out,
                double* min_e, int trace_mode, int* trace_count, int32_t* trace_steps,
                double* trace_c, double* trace_e, int trace_cap) {
    if (orc_hyper_validate(h)) return -3;
    const int N = p->N;
    double* c = (double*)malloc(sizeof(double) * (size_t)N);
    double* e = (double*)malloc(sizeof(double) * (size_t)N);
    double* c2 = (double*)malloc(sizeof(double) * (size_t)N);
    double* e2 = (double*)malloc(sizeof(double) * (size_t)N);
    double* hf = (double*)malloc(sizeof(double) * (size_t)N);
    int32_t* sigma = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
    for (int r = 0; r < N; ++r) {
        c[r] = 0.01 * orc_gauss(rng);
        e[r] = 1.0;
    }
    double t = 0.0, me = 1.0;
    const double T = (double)h->n_steps * h->dt;
    const int stride = trace_mode == 2 ? 1 : orc_trace_stride(h->n_steps, 500);
    int ntr = 0;
#define RECORD(step)                                                                   \
    do {                                                                               \
        if (trace_mode && ((step) % stride == 0 || (step) == h->n_steps) && ntr < trace_cap) { \
            trace_steps[ntr] = (step);                                                 \
            memcpy(trace_c + (size_t)ntr * N, c, sizeof(double) * (size_t)N);         \
            memcpy(trace_e + (size_t)ntr * N, e, sizeof(double) * (size_t)N);         \
            ++ntr;                                                                     \
        }                                                                              \
    } while (0)
    RECORD(0);
    int rc = -1;
    for (int step = 0; step < h->n_steps; ++step) {
        const double pp = h->pump_kind == ORC_PUMP_LINEAR ? orc_pump_linear(t, h->pump_end, T)
                                                          : orc_pump_sigmoid(t, h->p_thr, h->d);
        if (backend == ORC_MFZ_BN) {
            for (int r = 0; r < N; ++r) sigma[r] = c[r] > 0.0 ? 1 : 0;
            orc_local_field_bn(p, R, sigma, h->tau, hf);
        } else {
            orc_local_field_cn(p, R, c, h->tau, hf);
        }
        if (g_perturb & 1)
            for (int r = 0; r < N; ++r) hf[r] = (double)(float)hf[r];
        if (g_perturb & (8 | 16)) { /* relative field noise 2^-20 / 2^-16 (xorshift, per spin) */
            const double amp = (g_perturb & 8) ? 0x1p-20 : 0x1p-16;
            uint64_t x = 0x9E3779B97F4A7C15ull ^ (uint64_t)step;
            for (int r = 0; r < N; ++r) {
                x ^= x << 13; x ^= x >> 7; x ^= x << 17;
                const double u = (double)(x >> 11) * 0x1p-53 * 2.0 - 1.0;
                hf[r] = hf[r] * (1.0 + amp * u);
            }
        }
        rc = orc_mfz_step(N, c, e, pp, h, eta, R, hf, c2, e2);
        if (rc != -1) break;
        if (g_perturb & 2)
            for (int r = 0; r < N; ++r) {
                c2[r] = (double)(float)c2[r];
                e2[r] = (double)(float)e2[r];
            }
        double* tmp = c;
        c = c2;
        c2 = tmp;
        tmp = e;
        e = e2;
        e2 = tmp;
        t = t + h->dt;
        double emin = e[0];
        for (int r = 1; r < N; ++r)
            if (e[r] < emin) emin = e[r];
        me = (emin < me) ? emin : me;
        RECORD(step + 1);
    }
#undef RECORD
    if (trace_count) *trace_count = ntr;
    if (rc == -1) {
        for (int r = 0; r < N; ++r) sigma_out[r] = c[r] > 0.0 ? 1 : 0;
        if (c_out) memcpy(c_out, c, sizeof(double) * (size_t)N);
        if (e_out) memcpy(e_out, e, sizeof(double) * (size_t)N);
        if (min_e) *min_e = me;
    }
    free(c);
    free(e);
    free(c2);
    free(e2);
    free(hf);
    free(sigma);
    return rc;
}

/* ===================================================================== cdp */
/* Restricted operator y = G_sub v on the active set. */
typedef struct {
    const orc_problem* p;
    const int* act;
    int k;
    const double* Gs; /* k x k (LITERAL / EXPLICIT) */
    double* full;     /* N scratch (CANON) */
} sub_op;

static void sub_apply(const sub_op* s, const double* v, double* out) {
    const int k = s->k;
    if (s->p->mode == ORC_CANON) {
        const int N = s->p->N;
        for (int j = 0; j < N; ++j) s->full[j] = 0.0;
        for (int c = 0; c < k; ++c) s->full[s->act[c]] = v[c];
        for (int r = 0; r < k; ++r)
            out[r] = orc_canon_dot(s->p->G + (size_t)s->act[r] * N, s->full, N, s->p->nseg,
                                   s->p->gran);
    } else {
        for (int r = 0; r < k; ++r) out[r] = seq_dot(s->Gs + (size_t)r * k, v, k);
    }
}

/* cdp.cpp:17-28 / 30-46 (build_subproblem) + 48-64 (jacobi_solve) +
 * 66-105 (cg) + 109-139 (gather/scatter/cdp_minimize). */
int orc_cdp_minimize(const orc_problem* p, const int32_t* sigma, const double* R_prev,
                     int method, const orc_hyper* h, double* R_out, int* bad_index) {
    const int N = p->N, M = p->M;
    memcpy(R_out, R_prev, sizeof(double) * (size_t)N);
    int* act = (int*)malloc(sizeof(int) * (size_t)N);
    int k = 0;
    for (int r = 0; r < N; ++r) {
        if (sigma[r] != 0 && sigma[r] != 1) {
            free(act);
            return 1;
        }
        if (sigma[r] == 1) act[k++] = r;
    }
    if (k == 0) {
        free(act);
        return 0;
    }
    double* Gs = NULL;
    double* b = (double*)malloc(sizeof(double) * (size_t)k);
    double* D = (double*)malloc(sizeof(double) * (size_t)k);
    if (p->mode == ORC_CANON) {
        for (int c = 0; c < k; ++c) {
            b[c] = p->hz[act[c]];
            D[c] = p->G[(size_t)act[c] * N + act[c]];
        }
    } else if (!p->A) {
        /* gram-given problem (orc_problem_init_gram): G_sub = G[act, act],
         * b = hz[act] (cdp_minimize(G_full, hz, ...) orchestrator.cpp:110-113 /
         * cdp_minimize_operator's restricted apply, cdp.cpp:161-167) */
        Gs = (double*)malloc(sizeof(double) * (size_t)k * k);
        for (int r = 0; r < k; ++r) {
            for (int c = 0; c < k; ++c) Gs[(size_t)r * k + c] = p->G[(size_t)act[r] * N + act[c]];
            b[r] = p->hz[act[r]];
        }
        for (int c = 0; c < k; ++c) D[c] = Gs[(size_t)c * k + c];
    } else {
        /* A_act^T A_act, A_act^T y (sequential) -- identical in LITERAL and
         * EXPLICIT since both build G sequentially without FMA. */
        Gs = (double*)malloc(sizeof(double) * (size_t)k * k);
        for (int r = 0; r < k; ++r) {
            const double* cr = p->A + (size_t)act[r] * M;
            for (int c = r; c < k; ++c) {
                const double v = seq_dot(cr, p->A + (size_t)act[c] * M, M);
                Gs[(size_t)r * k + c] = v;
                Gs[(size_t)c * k + r] = v;
            }
            b[r] = seq_dot(cr, p->y, M);
        }
        for (int c = 0; c < k; ++c) D[c] = Gs[(size_t)c * k + c];
    }
    sub_op so = {p, act, k, Gs, NULL};
    if (p->mode == ORC_CANON) so.full = (double*)malloc(sizeof(double) * (size_t)N);
    double* R = (double*)malloc(sizeof(double) * (size_t)k);
    double* t1 = (double*)malloc(sizeof(double) * (size_t)k);
    for (int c = 0; c < k; ++c) R[c] = R_prev[act[c]];
    int rc = 0;
    if (method == ORC_CDP_JACOBI) {
        for (int r = 0; r < k; ++r)
            if (D[r] == 0.0) {
                if (bad_index) *bad_index = act[r];
                rc = 1;
                break;
            }
        if (!rc) {
            const double dt_c = h->dt_c;
            for (int it = 0; it < h->jacobi_iters; ++it) {
                sub_apply(&so, R, t1);
                for (int r = 0; r < k; ++r) t1[r] = t1[r] - D[r] * R[r]; /* offdiag */
                for (int r = 0; r < k; ++r)
                    R[r] = (1.0 - dt_c) * R[r] + dt_c * ((b[r] - t1[r]) / D[r]);
            }
        }
    } else {
        /* cg_solve_operator cdp.cpp:66-94 */
        double* rr = (double*)malloc(sizeof(double) * (size_t)k);
        double* pp = (double*)malloc(sizeof(double) * (size_t)k);
        double* Gp = (double*)malloc(sizeof(double) * (size_t)k);
        sub_apply(&so, R, t1);
        for (int c = 0; c < k; ++c) rr[c] = b[c] - t1[c];
        memcpy(pp, rr, sizeof(double) * (size_t)k);
        double rs = seq_dot(rr, rr, k);
        const double bnorm = sqrt(seq_dot(b, b, k));
        const double stop = h->cg_tol * (bnorm > 0.0 ? bnorm : 1.0);
        for (int it = 0; it < h->cg_max_iters && sqrt(rs) > stop; ++it) {
            sub_apply(&so, pp, Gp);
            const double curv = seq_dot(pp, Gp, k);
            if (!(curv > 0.0)) break;
            const double alpha = rs / curv;
            for (int c = 0; c < k; ++c) R[c] += alpha * pp[c];
            for (int c = 0; c < k; ++c) rr[c] -= alpha * Gp[c];
            const double rs_new = seq_dot(rr, rr, k);
            for (int c = 0; c < k; ++c) pp[c] = rr[c] + (rs_new / rs) * pp[c];
            rs = rs_new;
        }
        free(rr);
        free(pp);
        free(Gp);
    }
    if (!rc)
        for (int c = 0; c < k; ++c) R_out[act[c]] = R[c];
    free(act);
    free(Gs);
    free(b);
    free(D);
    free(so.full);
    free(R);
    free(t1);
    return rc;
}

/* ================================================================= scoring */
/* SolverProblem::objective_at orchestrator.cpp:57-62 */
double orc_objective_at(const orc_problem* p, const double* R, const int32_t* sigma,
                        double lambda) {
    const int N = p->N;
    double* w = (double*)malloc(sizeof(double) * (size_t)N);
    double* g = (double*)malloc(sizeof(double) * (size_t)N);
    long ssum = 0;
    for (int r = 0; r < N; ++r) {
        w[r] = R[r] * (double)sigma[r];
        ssum += sigma[r];
    }
    orc_gram_apply(p, w, g);
    const double v = 0.5 * seq_dot(w, g, N) - seq_dot(p->hz, w, N) + lambda * (double)ssum;
    free(w);
    free(g);
    return v;
}

/* orchestrator.cpp:64-68 */
double orc_hamiltonian_at(const orc_problem* p, const double* R, const int32_t* sigma,
                          double lambda) {
    const int N = p->N;
    double s = 0.0;
    for (int r = 0; r < N; ++r) {
        const double w = R[r] * (double)sigma[r];
        s = s + p->D[r] * (w * w);
    }
    return orc_objective_at(p, R, sigma, lambda) - 0.5 * s;
}

/* model.cpp:18-38 */
double orc_hamiltonian(int N, int M, const double* A, const double* y, const double* R,
                       const int32_t* sigma, double lambda) {
    double* w = (double*)malloc(sizeof(double) * (size_t)N);
    double* Aw = (double*)calloc((size_t)M, sizeof(double));
    int support = 0;
    for (int r = 0; r < N; ++r) {
        w[r] = sigma[r] ? R[r] : 0.0;
        support += sigma[r];
    }
    for (int r = 0; r < N; ++r)
        for (int k = 0; k < M; ++k) Aw[k] = Aw[k] + A[(size_t)r * M + k] * w[r];
    double diag = 0.0;
    for (int r = 0; r < N; ++r)
        if (sigma[r]) {
            const double* col = A + (size_t)r * M;
            diag += seq_dot(col, col, M) * w[r] * w[r];
        }
    const double pair = 0.5 * (seq_dot(Aw, Aw, M) - diag);
    const double zeeman = seq_dot(y, Aw, M);
    free(w);
    free(Aw);
    return pair - zeeman + lambda * support;
}

/* model.cpp:40-52 */
double orc_objective(int N, int M, const double* A, const double* y, const double* R,
                     const int32_t* sigma, double lambda) {
    double* w = (double*)malloc(sizeof(double) * (size_t)N);
    double* res = (double*)malloc(sizeof(double) * (size_t)M);
    int support = 0;
    for (int r = 0; r < N; ++r) {
        w[r] = sigma[r] ? R[r] : 0.0;
        support += sigma[r];
    }
    for (int k = 0; k < M; ++k) res[k] = 0.0;
    for (int r = 0; r < N; ++r)
        for (int k = 0; k < M; ++k) res[k] = res[k] + A[(size_t)r * M + k] * w[r];
    for (int k = 0; k < M; ++k) res[k] = y[k] - res[k];
    const double fit = 0.5 * seq_dot(res, res, M);
    const double v = fit - 0.5 * seq_dot(y, y, M) + lambda * support;
    free(w);
    free(res);
    return v;
}

/* model.cpp:128-144 */
double orc_rmse(int N, const double* R, const int32_t* sigma, const double* x,
                const int32_t* xi) {
    double s = 0.0;
    for (int r = 0; r < N; ++r) {
        const double d = (sigma[r] ? R[r] : 0.0) - (xi[r] ? x[r] : 0.0);
        s += d * d;
    }
    return sqrt(s / (double)N);
}

/* model.cpp:146-153 */
double orc_hamming(int N, const int32_t* sigma, const int32_t* xi) {
    double s = 0.0;
    for (int r = 0; r < N; ++r) s += fabs((double)(sigma[r] - xi[r]));
    return s / (double)N;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* orchestrator.cpp:163-168 */
double orc_median(int n, const double* v) {
    if (n == 0) return NAN;
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(s, v, sizeof(double) * (size_t)n);
    qsort(s, (size_t)n, sizeof(double), cmp_double);
    const double m = n % 2 == 1 ? s[n / 2] : 0.5 * (s[n / 2 - 1] + s[n / 2]);
    free(s);
    return m;
}

/* ==================================================== alternating_minimize */
static int alternating_impl(const orc_problem* p, int backend, const orc_hyper* h,
                            const double* R_init, orc_rng* rng, int cdp_method, int track_best,
                            int alt_limit, double* R_out, int32_t* sigma_out, orc_record* hist,
                            int* n_hist, double* hist_R, int32_t* hist_sigma, int* fail_alt,
                            int* fail_index) {
    if (orc_hyper_validate(h)) return 2;
    const int N = p->N;
    double* R = (double*)malloc(sizeof(double) * (size_t)N);
    double* Rn = (double*)malloc(sizeof(double) * (size_t)N);
    double* e = (double*)malloc(sizeof(double) * (size_t)N);
    int32_t* sigma = (int32_t*)calloc((size_t)N, sizeof(int32_t));
    int32_t* sig_new = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
    double* bestR = (double*)malloc(sizeof(double) * (size_t)N);
    int32_t* bestS = (int32_t*)calloc((size_t)N, sizeof(int32_t));
    memcpy(R, R_init, sizeof(double) * (size_t)N);
    memcpy(bestR, R_init, sizeof(double) * (size_t)N);
    double best = INFINITY;
    int nh = 0, rc = 0;
    *fail_alt = -1;
    if (fail_index) *fail_index = -1;
    const int last = alt_limit > 0 && alt_limit - 1 < h->velo ? alt_limit - 1 : h->velo;
    for (int i = 0; i <= last; ++i) {
        const double eta = orc_eta_schedule(i, h->eta_init, h->eta_end, h->velo);
        const double lambda = eta * eta / 2.0;
        double min_e;
        const int frc = backend == ORC_PP
                            ? orc_run_pp(p, R, h, eta, rng, NULL, NULL, NULL, e, NULL, sig_new,
                                         &min_e, NULL)
                            : orc_run_mfz(p, R, h, eta, backend, rng, NULL, e, sig_new, &min_e, 0,
                                          NULL, NULL, NULL, NULL, 0);
        if (frc >= 0) {
            *fail_alt = i;
            if (fail_index) *fail_index = frc;
            break;
        }
        if (frc < -1) {
            rc = frc == -3 ? 2 : 1;
            break;
        }
        memcpy(sigma, sig_new, sizeof(int32_t) * (size_t)N);
        int bad = -1;
        if (orc_cdp_minimize(p, sigma, R, cdp_method, h, Rn, &bad)) {
            rc = 1;
            if (fail_index) *fail_index = bad;
            break;
        }
        memcpy(R, Rn, sizeof(double) * (size_t)N);
        if (g_perturb & 4)
            for (int r = 0; r < N; ++r) R[r] = (double)(float)R[r];
        orc_record* rec = &hist[nh];
        rec->i = i;
        rec->eta = eta;
        rec->hamiltonian = orc_objective_at(p, R, sigma, lambda);
        rec->rmse = p->x_true ? orc_rmse(N, R, sigma, p->x_true, p->xi_true) : NAN;
        rec->hamming = p->xi_true ? orc_hamming(N, sigma, p->xi_true) : NAN;
        rec->min_e = min_e;
        rec->median_e = orc_median(N, e);
        int sup = 0;
        for (int r = 0; r < N; ++r) sup += sigma[r];
        rec->support = sup;
        if (hist_R) memcpy(hist_R + (size_t)nh * N, R, sizeof(double) * (size_t)N);
        if (hist_sigma) memcpy(hist_sigma + (size_t)nh * N, sigma, sizeof(int32_t) * (size_t)N);
        if (rec->hamiltonian < best) {
            best = rec->hamiltonian;
            memcpy(bestR, R, sizeof(double) * (size_t)N);
            memcpy(bestS, sigma, sizeof(int32_t) * (size_t)N);
        }
        ++nh;
    }
    if (track_best && isfinite(best)) {
        memcpy(R, bestR, sizeof(double) * (size_t)N);
        memcpy(sigma, bestS, sizeof(int32_t) * (size_t)N);
    }
    memcpy(R_out, R, sizeof(double) * (size_t)N);
    memcpy(sigma_out, sigma, sizeof(int32_t) * (size_t)N);
    *n_hist = nh;
    free(R);
    free(Rn);
    free(e);
    free(sigma);
    free(sig_new);
    free(bestR);
    free(bestS);
    return rc;
}

int orc_alternating_minimize(const orc_problem* p, int backend, const orc_hyper* h,
                             const double* R_init, orc_rng* rng, int cdp_method, int track_best,
                             double* R_out, int32_t* sigma_out, orc_record* hist, int* n_hist,
                             double* hist_R, int32_t* hist_sigma, int* fail_alt,
                             int* fail_index) {
    return alternating_impl(p, backend, h, R_init, rng, cdp_method, track_best, 0, R_out,
                            sigma_out, hist, n_hist, hist_R, hist_sigma, fail_alt, fail_index);
}

int orc_solve_trial(int N, int M, const double* A, const double* y, const double* x,
                    const int32_t* xi, int mode, int nseg, int gran, int backend,
                    const orc_hyper* h, uint64_t seed, int cdp_method, int track_best,
                    double* R_out, int32_t* sigma_out, orc_record* hist, int* n_hist,
                    int* fail_alt, int* fail_index) {
    orc_problem p;
    if (orc_problem_init(&p, N, M, A, y, mode, nseg, gran)) return 1;
    p.x_true = x;
    p.xi_true = xi;
    orc_rng rng;
    orc_rng_init(&rng, seed);
    /* default_r_init = hz (orchestrator.cpp:138) */
    const int rc = orc_alternating_minimize(&p, backend, h, p.hz, &rng, cdp_method, track_best,
                                            R_out, sigma_out, hist, n_hist, NULL, NULL,
                                            fail_alt, fail_index);
    orc_problem_free(&p);
    return rc;
}

/* ====================================================== batch (run_jobs) */
typedef struct {
    int ntrials, N, mode, nseg, gran, backend, cdp_method, alt_limit;
    const int* M;
    const double* const* A;
    const double* const* y;
    const double* const* x;
    const int32_t* const* xi;
    const orc_hyper* h;
    const uint64_t* seeds;
    double* R_out;
    int32_t* sigma_out;
    int* fail_alt;
    int next;
    pthread_mutex_t mu;
} batch_ctx;

static void* batch_worker(void* arg) {
    batch_ctx* b = (batch_ctx*)arg;
    orc_record* hist = (orc_record*)malloc(sizeof(orc_record) * (size_t)(b->h->velo + 1));
    for (;;) {
        pthread_mutex_lock(&b->mu);
        const int t = b->next++;
        pthread_mutex_unlock(&b->mu);
        if (t >= b->ntrials) break;
        orc_problem p;
        orc_problem_init(&p, b->N, b->M[t], b->A[t], b->y[t], b->mode, b->nseg, b->gran);
        p.x_true = b->x ? b->x[t] : NULL;
        p.xi_true = b->xi ? b->xi[t] : NULL;
        orc_rng rng;
        orc_rng_init(&rng, b->seeds[t]);
        int nh, fa, fi;
        alternating_impl(&p, b->backend, b->h, p.hz, &rng, b->cdp_method, 0, b->alt_limit,
                         b->R_out + (size_t)t * b->N, b->sigma_out + (size_t)t * b->N, hist,
                         &nh, NULL, NULL, &fa, &fi);
        if (b->fail_alt) b->fail_alt[t] = fa;
        orc_problem_free(&p);
    }
    free(hist);
    return NULL;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static double batch_run(batch_ctx* b, int nthreads) {
    pthread_mutex_init(&b->mu, NULL);
    b->next = 0;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > b->ntrials) nthreads = b->ntrials;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    const double t0 = now_s();
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, batch_worker, b);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    const double dt = now_s() - t0;
    free(th);
    pthread_mutex_destroy(&b->mu);
    return dt;
}

double orc_solve_batch(int ntrials, int nthreads, int N, const int* M, const double* const* A,
                       const double* const* y, const double* const* x,
                       const int32_t* const* xi, int mode, int nseg, int gran, int backend,
                       const orc_hyper* h, const uint64_t* seeds, int cdp_method,
                       double* R_out, int32_t* sigma_out, int* fail_alt) {
    batch_ctx b;
    memset(&b, 0, sizeof(b));
    b.ntrials = ntrials;
    b.N = N;
    b.M = M;
    b.A = A;
    b.y = y;
    b.x = x;
    b.xi = xi;
    b.mode = mode;
    b.nseg = nseg;
    b.gran = gran;
    b.backend = backend;
    b.h = h;
    b.seeds = seeds;
    b.cdp_method = cdp_method;
    b.R_out = R_out;
    b.sigma_out = sigma_out;
    b.fail_alt = fail_alt;
    b.alt_limit = 0;
    return batch_run(&b, nthreads);
}

/* Bounded CPU-baseline sample: the first `alt_limit` alternations of each
 * trial (1 = one CIM call of n_steps Euler steps + one refit + scoring). */
double orc_solve_batch_limited(int ntrials, int nthreads, int alt_limit, int N, const int* M,
                               const double* const* A, const double* const* y, int mode,
                               int backend, const orc_hyper* h, const uint64_t* seeds,
                               double* R_out, int32_t* sigma_out) {
    batch_ctx b;
    memset(&b, 0, sizeof(b));
    b.ntrials = ntrials;
    b.N = N;
    b.M = M;
    b.A = A;
    b.y = y;
    b.mode = mode;
    b.nseg = 8;
    b.gran = 8;
    b.backend = backend;
    b.h = h;
    b.seeds = seeds;
    b.cdp_method = ORC_CDP_JACOBI;
    b.R_out = R_out;
    b.sigma_out = sigma_out;
    b.alt_limit = alt_limit;
    return batch_run(&b, nthreads);
}
