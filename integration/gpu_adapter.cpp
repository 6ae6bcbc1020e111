// gpu_adapter.cpp -- the reference-side adapter a maintainer would add to
// /root/reference/proj/src: the reference's own alternating_minimize signature
// (orchestrator.hpp:139-141) served by libcimcs_gpu.so through the C ABI
// (include/cimcs_gpu.h).  INTEGRATION.md section 2 documents it; this file is
// the COMPILED version: oracle/Makefile.ref builds it against the reference's
// real headers (and the sequential Eigen shim, Eigen3 being absent here) into
// oracle/_ref/libref_adapter.so, and tests/test_gpu_adapter.py calls it on the
// GPU next to the reference's own CPU solver.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "cimcs/orchestrator.hpp"
#include "cimcs_gpu.h"

namespace cimcs {
namespace {

cimcs_hyper to_c(const HyperParams& p) {  // types.hpp:77-96 -> cimcs_hyper
    cimcs_hyper h;
    cimcs_hyper_default(&h);
    h.g2 = p.g2;
    h.j = p.j;
    h.K = p.K;
    h.beta = p.beta;
    h.tau = p.tau;
    h.dt = p.dt;
    h.n_steps = p.n_steps;
    h.p_thr = p.p_thr;
    h.d = p.d;
    h.eta_init = p.eta_init;
    h.eta_end = p.eta_end;
    h.velo = p.velo;
    h.dt_c = p.dt_c;
    h.jacobi_iters = p.jacobi_iters;
    h.cg_max_iters = p.cg_max_iters;
    h.cg_tol = p.cg_tol;
    h.gamma = p.gamma;
    h.mfz_loss_minus_j = p.mfz_loss_minus_j ? 1 : 0;
    h.mu_abort = p.mu_abort;
    h.pump_kind = CIMCS_PUMP_SIGMOID;  // the reference's pump_schedule (orchestrator.cpp:12-14)
    return h;
}

void check(int rc) {  // status -> the reference's exceptions (types.hpp:16-33)
    if (rc == CIMCS_OK || rc == CIMCS_DIVERGENCE) return;
    if (rc == CIMCS_INPUT_ERROR) throw input_error(cimcs_last_error());
    if (rc == CIMCS_CONFIG_ERROR) throw config_error(cimcs_last_error());
    throw std::runtime_error(cimcs_last_error());
}

int32_t backend_c(Backend b) {
    return b == Backend::MfzBN ? CIMCS_MFZ_BN : (b == Backend::MfzCN ? CIMCS_MFZ_CN : CIMCS_PP);
}

}  // namespace

// Drop-in for alternating_minimize(make_problem(inst), backend, params,
// default_r_init(prob), Rng(seed), opts) (orchestrator.cpp:80-99, 138, 170-235)
// on ONE trial; the GPU draws c0 from the same Rng(seed) stream.  dtype:
// CIMCS_F64 (bitwise-reproducible canonical order) or CIMCS_F32 / CIMCS_F32X.
AlternatingResult alternating_minimize_gpu(const ProblemInstance& inst, Backend backend,
                                           const HyperParams& params, std::uint64_t seed,
                                           const AlternateOptions& opts, int dtype = CIMCS_F64,
                                           int device = 0) {
    params.validate();
    cimcs_ctx* ctx = nullptr;
    check(cimcs_create(device, dtype, &ctx));
    struct Guard {
        cimcs_ctx* c;
        ~Guard() { cimcs_destroy(c); }
    } guard{ctx};
    const int N = inst.N(), M = inst.M();
    const double* A = inst.A.data();  // Eigen column-major M x N == the ABI layout
    const double* y = inst.y.data();
    const double* x = inst.has_truth() ? inst.x_true.data() : nullptr;
    std::vector<int32_t> xi(inst.xi_true.data(), inst.xi_true.data() + inst.xi_true.size());
    const int32_t* xip = inst.has_truth() ? xi.data() : nullptr;
    check(cimcs_set_problems(ctx, 1, N, &M, &A, &y, x ? &x : nullptr, xip ? &xip : nullptr));
    check(cimcs_build_coupling(ctx));
    const cimcs_hyper h = to_c(params);
    AlternatingResult res;
    res.R.resize(N);
    std::vector<int32_t> sigma(N);
    std::vector<cimcs_record> hist(params.velo + 1);
    int32_t nh = 0, fa = -1, fi = -1;
    check(cimcs_solve(ctx, 1, backend_c(backend), &h,
                      opts.method == CdpMethod::Jacobi ? CIMCS_CDP_JACOBI : CIMCS_CDP_CG, &seed,
                      nullptr, opts.track_best ? 1 : 0, res.R.data(), sigma.data(), hist.data(),
                      &nh, &fa, &fi));
    res.sigma.resize(N);
    for (int r = 0; r < N; ++r) res.sigma[r] = sigma[r];
    for (int k = 0; k < nh; ++k) {
        AlternationRecord rec;
        rec.i = hist[k].i;
        rec.eta = hist[k].eta;
        rec.hamiltonian = hist[k].hamiltonian;
        rec.rmse = hist[k].rmse;
        rec.hamming = hist[k].hamming;
        rec.min_e = hist[k].min_e;
        rec.median_e = hist[k].median_e;
        res.history.push_back(std::move(rec));
    }
    res.failed = fa >= 0;
    res.fail_alternation = fa;
    if (res.failed)
        res.fail_reason = (backend == Backend::PositiveP ? "pp: divergence at spin "
                                                         : "mfz_step: non-finite amplitude at spin ") +
                          std::to_string(fi);
    return res;
}

}  // namespace cimcs

// extern "C" test hook (tests/test_gpu_adapter.py): raw arrays in, the
// adapter's AlternatingResult out (hist rows [i, eta, hamiltonian, rmse,
// hamming, min_e, median_e]).  hyper: the oracle's orc_hyper layout.
extern "C" {
struct adapter_hyper {
    double g2, j, K, beta, tau, dt;
    int n_steps;
    double p_thr, d, eta_init, eta_end;
    int velo;
    double dt_c;
    int jacobi_iters, cg_max_iters;
    double cg_tol, gamma;
    int mfz_loss_minus_j;
    double mu_abort;
    int pump_kind;
    double pump_end;
};

int adapter_alternating_minimize_gpu(int N, int M, const double* A, const double* y,
                                     const double* x, const int32_t* xi, int backend,
                                     const adapter_hyper* ah, uint64_t seed, int cdp,
                                     int track_best, int dtype, double* R_out,
                                     int32_t* sigma_out, double* hist, int* n_hist,
                                     int* fail_alt) {
    try {
        cimcs::ProblemInstance inst;
        inst.A.resize(M, N);
        std::memcpy(inst.A.data(), A, sizeof(double) * static_cast<size_t>(M) * N);
        inst.y.resize(M);
        std::memcpy(inst.y.data(), y, sizeof(double) * static_cast<size_t>(M));
        if (x && xi) {
            inst.x_true.resize(N);
            inst.xi_true.resize(N);
            for (int r = 0; r < N; ++r) {
                inst.x_true[r] = x[r];
                inst.xi_true[r] = xi[r];
            }
        }
        cimcs::HyperParams p;
        p.g2 = ah->g2;
        p.j = ah->j;
        p.K = ah->K;
        p.beta = ah->beta;
        p.tau = ah->tau;
        p.dt = ah->dt;
        p.n_steps = ah->n_steps;
        p.p_thr = ah->p_thr;
        p.d = ah->d;
        p.eta_init = ah->eta_init;
        p.eta_end = ah->eta_end;
        p.velo = ah->velo;
        p.dt_c = ah->dt_c;
        p.jacobi_iters = ah->jacobi_iters;
        p.cg_max_iters = ah->cg_max_iters;
        p.cg_tol = ah->cg_tol;
        p.gamma = ah->gamma;
        p.mfz_loss_minus_j = ah->mfz_loss_minus_j != 0;
        p.mu_abort = ah->mu_abort;
        cimcs::AlternateOptions opts;
        opts.method = cdp ? cimcs::CdpMethod::ConjugateGradient : cimcs::CdpMethod::Jacobi;
        opts.track_best = track_best != 0;
        const cimcs::Backend be = backend == 0 ? cimcs::Backend::MfzCN
                                  : backend == 1 ? cimcs::Backend::MfzBN
                                                 : cimcs::Backend::PositiveP;
        const cimcs::AlternatingResult res =
            cimcs::alternating_minimize_gpu(inst, be, p, seed, opts, dtype);
        for (int r = 0; r < N; ++r) {
            R_out[r] = res.R[r];
            sigma_out[r] = res.sigma[r];
        }
        *n_hist = static_cast<int>(res.history.size());
        for (size_t k = 0; k < res.history.size(); ++k) {
            const auto& rec = res.history[k];
            double* o = hist + 7 * k;
            o[0] = rec.i;
            o[1] = rec.eta;
            o[2] = rec.hamiltonian;
            o[3] = rec.rmse;
            o[4] = rec.hamming;
            o[5] = rec.min_e;
            o[6] = rec.median_e;
        }
        *fail_alt = res.failed ? res.fail_alternation : -1;
        return 0;
    } catch (const std::exception& e) {
        return 1;
    }
}
}
