// extern "C" face of the reference's own solver -- alternating_minimize,
// run_cim, cdp_minimize and the scorer (orchestrator.cpp, solver_mfz.cpp,
// solver_pp.cpp, cdp.cpp, model.cpp), compiled UNMODIFIED from
// /root/reference/proj against the sequential Eigen shim (refshim/Eigen/Dense).
// TEST INFRASTRUCTURE ONLY: tests/test_ref_solver.py checks the oracle's
// LITERAL restatement against it bit for bit.  The reference has only its
// sigmoid pump (orchestrator.cpp:12-14), so the builder's linear-pump
// extension is rejected here.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "cimcs/cdp.hpp"
#include "cimcs/model.hpp"
#include "cimcs/orchestrator.hpp"

namespace {

// layout of the oracle's orc_hyper (oracle/oracle.h), so Python passes one struct
struct ref_hyper {
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

thread_local std::string g_msg;

cimcs::HyperParams to_params(const ref_hyper* h) {
    cimcs::HyperParams p;
    p.g2 = h->g2;
    p.j = h->j;
    p.K = h->K;
    p.beta = h->beta;
    p.tau = h->tau;
    p.dt = h->dt;
    p.n_steps = h->n_steps;
    p.p_thr = h->p_thr;
    p.d = h->d;
    p.eta_init = h->eta_init;
    p.eta_end = h->eta_end;
    p.velo = h->velo;
    p.dt_c = h->dt_c;
    p.jacobi_iters = h->jacobi_iters;
    p.cg_max_iters = h->cg_max_iters;
    p.cg_tol = h->cg_tol;
    p.gamma = h->gamma;
    p.mfz_loss_minus_j = h->mfz_loss_minus_j != 0;
    p.mu_abort = h->mu_abort;
    return p;
}

cimcs::ProblemInstance make_inst(int N, int M, const double* A, const double* y,
                                 const double* x, const int32_t* xi) {
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
    return inst;
}

cimcs::Backend backend_of(int b) {
    return b == 0 ? cimcs::Backend::MfzCN
                  : (b == 1 ? cimcs::Backend::MfzBN : cimcs::Backend::PositiveP);
}

// 0 ok, 1 input_error, 2 config_error, 3 divergence, 5 other
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const cimcs::input_error& e) {
        g_msg = e.what();
        return 1;
    } catch (const cimcs::config_error& e) {
        g_msg = e.what();
        return 2;
    } catch (const cimcs::divergence_error& e) {
        g_msg = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 5;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }

// alternating_minimize(make_problem(inst), backend, params, R_init, Rng(seed), opts)
// (orchestrator.cpp:80-99, 170-235).  hist: (velo+1) rows of
// [i, eta, hamiltonian, rmse, hamming, min_e, median_e].
int ref_alternating_minimize(int N, int M, const double* A, const double* y, const double* x,
                             const int32_t* xi, int backend, const ref_hyper* h, uint64_t seed,
                             const double* R_init, int cdp, int track_best, double* R_out,
                             int32_t* sigma_out, double* hist, int* n_hist, int* fail_alt,
                             char* fail_reason, int reason_cap) {
    if (h->pump_kind != 0) {
        g_msg = "the reference has only the sigmoid pump";
        return 2;
    }
    return guarded([&] {
        const cimcs::ProblemInstance inst = make_inst(N, M, A, y, x, xi);
        const cimcs::SolverProblem prob = cimcs::make_problem(inst);
        cimcs::VectorXd r0 = cimcs::default_r_init(prob);
        if (R_init)
            for (int r = 0; r < N; ++r) r0[r] = R_init[r];
        cimcs::Rng rng(seed);
        cimcs::AlternateOptions opts;
        opts.method = cdp ? cimcs::CdpMethod::ConjugateGradient : cimcs::CdpMethod::Jacobi;
        opts.track_best = track_best != 0;
        const cimcs::AlternatingResult res =
            cimcs::alternating_minimize(prob, backend_of(backend), to_params(h), r0, rng, opts);
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
        if (fail_reason && reason_cap > 0) {
            std::strncpy(fail_reason, res.fail_reason.c_str(), reason_cap - 1);
            fail_reason[reason_cap - 1] = 0;
        }
    });
}

// run_cim(prob.coupling(), backend, R, params, eta, Rng(seed)) (orchestrator.cpp:140-161)
int ref_run_cim(int N, int M, const double* A, const double* y, int backend, const ref_hyper* h,
                double eta, uint64_t seed, const double* R, int32_t* sigma_out, double* e_out,
                double* amp_out, double* min_e) {
    return guarded([&] {
        const cimcs::ProblemInstance inst = make_inst(N, M, A, y, nullptr, nullptr);
        const cimcs::SolverProblem prob = cimcs::make_problem(inst);
        cimcs::VectorXd Rv(N);
        for (int r = 0; r < N; ++r) Rv[r] = R[r];
        cimcs::Rng rng(seed);
        const cimcs::CimCallResult c =
            cimcs::run_cim(prob.coupling(), backend_of(backend), Rv, to_params(h), eta, rng);
        for (int r = 0; r < N; ++r) {
            sigma_out[r] = c.sigma[r];
            e_out[r] = c.e_final[r];
            amp_out[r] = c.amplitude[r];
        }
        *min_e = c.min_e;
    });
}

// cdp_minimize(inst, sigma, R_prev, method, params) (cdp.cpp:132-139)
int ref_cdp_minimize(int N, int M, const double* A, const double* y, const int32_t* sigma,
                     const double* R_prev, int cdp, const ref_hyper* h, double* R_out) {
    return guarded([&] {
        const cimcs::ProblemInstance inst = make_inst(N, M, A, y, nullptr, nullptr);
        cimcs::VectorXi s(N);
        cimcs::VectorXd rp(N);
        for (int r = 0; r < N; ++r) {
            s[r] = sigma[r];
            rp[r] = R_prev[r];
        }
        const cimcs::VectorXd out = cimcs::cdp_minimize(
            inst, s, rp, cdp ? cimcs::CdpMethod::ConjugateGradient : cimcs::CdpMethod::Jacobi,
            to_params(h));
        for (int r = 0; r < N; ++r) R_out[r] = out[r];
    });
}

// SolverProblem::objective_at / rmse / hamming_loss (orchestrator.cpp:57-80, model.cpp:128-153)
int ref_score(int N, int M, const double* A, const double* y, const double* x, const int32_t* xi,
              const double* R, const int32_t* sigma, double lambda, double* objective,
              double* rmse, double* hamming) {
    return guarded([&] {
        const cimcs::ProblemInstance inst = make_inst(N, M, A, y, x, xi);
        const cimcs::SolverProblem prob = cimcs::make_problem(inst);
        cimcs::VectorXd Rv(N);
        cimcs::VectorXi s(N);
        for (int r = 0; r < N; ++r) {
            Rv[r] = R[r];
            s[r] = sigma[r];
        }
        *objective = prob.objective_at(Rv, s, lambda);
        *rmse = prob.rmse_at(Rv, s);
        *hamming = prob.hamming_at(s);
    });
}
}
