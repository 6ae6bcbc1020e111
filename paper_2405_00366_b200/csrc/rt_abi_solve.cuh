// rt_abi_solve.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): C ABI: one step, CIM call, Positive-P, refit, score, the alternating
// solve, timing.
#pragma once

extern "C" {

int cimcs_mfz_step(cimcs_ctx* c, int32_t R, int32_t backend, const cimcs_hyper* hp, double eta,
                   double p, const double* Rsig, const double* cin, const double* ein,
                   double* c_out, double* e_out, double* h_out, int32_t* fail_index) {
    NvtxRange nvtx_range_("cimcs_mfz_step");
    NvtxRange nv_solve("cimcs_solve");
    if (int rc = check_ready(c, R)) return rc;
    if (int rc = validate(hp)) return rc;
    if (!std::isfinite(p)) return fail(CIMCS_INPUT_ERROR, "mfz_step: non-finite pump");
    if (backend != CIMCS_MFZ_BN && backend != CIMCS_MFZ_CN)
        return fail(CIMCS_CONFIG_ERROR, "backend must be mfz-bn or mfz-cn");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    const size_t n = (size_t)c->B * R * c->N;
    if (int rc = reset_flags(c, R)) return rc;
    if (int rc = set_alt(c, make_alt(hp, eta, 0))) return rc;
    if (int rc = upload_traj(c, Rsig, c->Rs, R)) return rc;
    // c and e go through a second staging area (the init kernel reads host layout)
    double* dce = nullptr;
    if (int rc = dalloc(c, &dce, 2 * n * 8)) return rc;
    CK(cudaMemcpyAsync(dce, cin, n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dce + n, ein, n * 8, cudaMemcpyHostToDevice, c->stream));
    const StepScalars s = make_scalars(hp);
    int rc = run_init(c, R, backend == CIMCS_MFZ_BN, dce, dce + n, s.rt);
    if (!rc) {
        GemvArgs a = base_args(c, s);
        a.pump = nullptr;
        a.p_scalar = p;
        a.step = 0;
        a.Win = c->W0;
        a.Wout = c->W1;
        a.Hdbg = c->Hdbg;
        rc = launch_gemv(c, backend == CIMCS_MFZ_BN ? EPI_STEP_BN : EPI_STEP_CN, a);
        if (!rc) rc = reconcile_cim(c);
        if (!rc && c->world > 1) {
            rc = allgather_state(c, c->C);
            if (!rc) rc = allgather_state(c, c->E);
            if (!rc) rc = allgather_state(c, c->Hdbg);
        }
    }
    if (!rc && c_out) rc = download_traj(c, c->C, c_out, R);
    if (!rc && e_out) rc = download_traj(c, c->E, e_out, R);
    if (!rc && h_out) rc = download_traj(c, c->Hdbg, h_out, R);
    std::vector<int> fi(c->B * c->NR);
    if (!rc)
        if (cudaMemcpyAsync(fi.data(), c->fail_idx, fi.size() * 4, cudaMemcpyDeviceToHost,
                            c->stream) != cudaSuccess)
            rc = fail(CIMCS_CUDA_ERROR, "copy");
    cudaStreamSynchronize(c->stream);
    cudaFree(dce);
    if (rc) return rc;
    bool div = false;
    for (int b = 0; b < c->B; ++b)
        for (int r = 0; r < R; ++r) {
            const int v = fi[b * c->NR + r];
            if (fail_index) fail_index[b * R + r] = v == INT_MAX ? -1 : v;
            div |= v != INT_MAX;
        }
    return div ? fail(CIMCS_DIVERGENCE, "mfz_step: non-finite amplitude") : 0;
}

int cimcs_run_pp(cimcs_ctx* c, int32_t R, const cimcs_hyper* hp, double eta, const double* Rsig,
                 const uint64_t* seeds, double* mu_out, double* e_out, double* mt_out,
                 int32_t* sigma_out, double* min_e, int32_t* fail_index) {
    if (int rc = check_ready(c, R)) return rc;
    if (int rc = validate(hp)) return rc;
    if (!(hp->j > 0.0)) return fail(CIMCS_CONFIG_ERROR, "measured_amplitude: j must be positive");
    if (!seeds) return fail(CIMCS_INPUT_ERROR, "null seeds");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    if (int rc = ensure_pp(c)) return rc;
    if (int rc = upload_pump(c, hp)) return rc;
    if (int rc = reset_flags(c, R)) return rc;
    if (int rc = set_alt(c, make_alt(hp, eta, 0))) return rc;
    if (int rc = upload_traj(c, Rsig, c->Rs, R)) return rc;
    std::vector<HostRng> rngs;
    for (int t = 0; t < c->B * R; ++t) rngs.emplace_back(seeds[t]);
    const StepScalars s = make_scalars(hp);
    Events ev(2);
    cudaEventRecord(ev.ev[0], c->stream);
    int rc = run_pp_cim(c, R, s, hp, rngs);
    cudaEventRecord(ev.ev[1], c->stream);
    if (!rc && mu_out) rc = download_traj(c, c->C, mu_out, R);
    if (!rc) rc = pp_amplitude_to_c(c);
    if (!rc) rc = run_support(c);  // sigma = mu~ > 0
    if (!rc && mt_out) rc = download_traj(c, c->C, mt_out, R);
    if (!rc && e_out) rc = download_traj(c, c->E, e_out, R);
    if (!rc && sigma_out) rc = download_sig(c, c->sig, sigma_out, R);
    std::vector<int> fi(c->B * c->NR);
    std::vector<unsigned long long> me(c->B * c->NR);
    if (!rc) {
        cudaMemcpyAsync(fi.data(), c->fail_idx, fi.size() * 4, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(me.data(), c->minE, me.size() * 8, cudaMemcpyDeviceToHost, c->stream);
    }
    cudaError_t se = cudaStreamSynchronize(c->stream);
    if (rc) return rc;
    if (se != cudaSuccess) return fail(CIMCS_CUDA_ERROR, cudaGetErrorString(se));
    c->timing.cim_ms = ev.ms(0, 1);
    c->timing.step_launches = hp->n_steps;
    bool div = false;
    int kind = 0;
    for (int b = 0; b < c->B; ++b)
        for (int r = 0; r < R; ++r) {
            const int v = fi[b * c->NR + r];
            const bool f = v != INT_MAX;
            if (fail_index) fail_index[b * R + r] = f ? (v & ((1 << 30) - 1)) : -1;
            if (min_e) min_e[b * R + r] = ord_val(me[b * c->NR + r]);
            if (f && !div) kind = v >> 30;
            div |= f;
        }
    return div ? fail(CIMCS_DIVERGENCE, kind ? "run_pp: |mu| exceeded mu_abort"
                                             : "pp_step: non-finite value")
               : 0;
}

int cimcs_run_cim(cimcs_ctx* c, int32_t R, int32_t backend, const cimcs_hyper* hp, double eta,
                  const double* Rsig, const double* c0, double* c_out, double* e_out,
                  int32_t* sigma_out, double* min_e, int32_t* fail_index) {
    NvtxRange nvtx_range_("cimcs_run_cim");
    if (int rc = check_ready(c, R)) return rc;
    if (int rc = validate(hp)) return rc;
    if (backend != CIMCS_MFZ_BN && backend != CIMCS_MFZ_CN)
        return fail(CIMCS_CONFIG_ERROR, "backend must be mfz-bn or mfz-cn");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    if (int rc = upload_pump(c, hp)) return rc;
    const size_t n = (size_t)c->B * R * c->N;
    if (int rc = reset_flags(c, R)) return rc;
    if (int rc = set_alt(c, make_alt(hp, eta, 0))) return rc;
    if (int rc = upload_traj(c, Rsig, c->Rs, R)) return rc;
    double* dc0 = nullptr;
    if (int rc = dalloc(c, &dc0, n * 8)) return rc;
    CK(cudaMemcpyAsync(dc0, c0, n * 8, cudaMemcpyHostToDevice, c->stream));
    const StepScalars s = make_scalars(hp);
    Events ev(2);
    cudaEventRecord(ev.ev[0], c->stream);
    int rc = run_init(c, R, backend == CIMCS_MFZ_BN, dc0, nullptr, s.rt);
    if (!rc) rc = enqueue_steps(c, backend == CIMCS_MFZ_BN, s, hp->n_steps);
    cudaEventRecord(ev.ev[1], c->stream);
    if (!rc) rc = run_support(c);
    if (!rc && c->world > 1) {
        rc = allgather_state(c, c->C);
        if (!rc) rc = allgather_state(c, c->E);
        if (!rc) rc = allgather_sig(c, c->sig);
    }
    if (!rc && c_out) rc = download_traj(c, c->C, c_out, R);
    if (!rc && e_out) rc = download_traj(c, c->E, e_out, R);
    if (!rc && sigma_out) rc = download_sig(c, c->sig, sigma_out, R);
    std::vector<int> fi(c->B * c->NR);
    std::vector<unsigned long long> me(c->B * c->NR);
    if (!rc) {
        cudaMemcpyAsync(fi.data(), c->fail_idx, fi.size() * 4, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(me.data(), c->minE, me.size() * 8, cudaMemcpyDeviceToHost, c->stream);
    }
    cudaError_t se = cudaStreamSynchronize(c->stream);
    cudaFree(dc0);
    if (rc) return rc;
    if (se != cudaSuccess) return fail(CIMCS_CUDA_ERROR, cudaGetErrorString(se));
    c->timing.cim_ms = ev.ms(0, 1);
    c->timing.step_launches = hp->n_steps;
    bool div = false;
    for (int b = 0; b < c->B; ++b)
        for (int r = 0; r < R; ++r) {
            const int v = fi[b * c->NR + r];
            if (fail_index) fail_index[b * R + r] = v == INT_MAX ? -1 : v;
            if (min_e) min_e[b * R + r] = ord_val(me[b * c->NR + r]);
            div |= v != INT_MAX;
        }
    return div ? fail(CIMCS_DIVERGENCE, "mfz_step: non-finite amplitude") : 0;
}

int cimcs_cdp_minimize(cimcs_ctx* c, int32_t R, const int32_t* sigma, const double* R_prev,
                       int32_t method, const cimcs_hyper* hp, double* R_out,
                       int32_t* iterations) {
    NvtxRange nvtx_range_("cimcs_cdp_minimize");
    if (int rc = check_ready(c, R)) return rc;
    if (!hp) return fail(CIMCS_CONFIG_ERROR, "null hyper-parameters");
    if (method != CIMCS_CDP_JACOBI && method != CIMCS_CDP_CG)
        return fail(CIMCS_CONFIG_ERROR, "cdp method must be jacobi or cg");
    if (method == CIMCS_CDP_CG && c->world > 1)
        return fail(CIMCS_CONFIG_ERROR, "cdp=cg is not supported on row-sharded contexts");
    if (c->mri && c->mri_kind == 0 && method == CIMCS_CDP_JACOBI)  // cdp.cpp:158-159
        return fail(CIMCS_CONFIG_ERROR, "cdp_minimize_operator: damped Jacobi needs an assembled matrix");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    if (method == CIMCS_CDP_CG)
        if (int rc = ensure_cg(c)) return rc;
    if (int rc = reset_flags(c, R)) return rc;
    if (int rc = upload_traj(c, R_prev, c->Rs, R)) return rc;
    if (int rc = upload_sig(c, sigma, c->sig, R)) return rc;
    const StepScalars s = make_scalars(hp);
    int rc = c->st64() ? mask_T<double>(c, c->W0) : mask_T<float>(c, c->W0);
    Events ev(2);
    cudaEventRecord(ev.ev[0], c->stream);
    if (!rc)
        rc = method == CIMCS_CDP_CG  ? enqueue_cg(c, s, hp)
             : cmp64_refit_ok(c)    ? enqueue_refit_compact64(c, s, hp->jacobi_iters, false)
                                    : enqueue_refit(c, s, hp->jacobi_iters, false);
    cudaEventRecord(ev.ev[1], c->stream);
    if (!rc) rc = download_traj(c, c->Rs, R_out, R);
    int err = INT_MAX;
    std::vector<CgTraj> st(method == CIMCS_CDP_CG ? c->B * c->NR : 0);
    cudaMemcpyAsync(&err, c->err, 4, cudaMemcpyDeviceToHost, c->stream);
    if (!rc && !st.empty())
        cudaMemcpyAsync(st.data(), c->cg_st, st.size() * sizeof(CgTraj), cudaMemcpyDeviceToHost,
                        c->stream);
    CK(cudaStreamSynchronize(c->stream));
    if (rc) return rc;
    c->timing.refit_ms = ev.ms(0, 1);
    if (iterations)
        for (int b = 0; b < c->B; ++b)
            for (int q = 0; q < R; ++q)
                iterations[b * R + q] =
                    method == CIMCS_CDP_CG ? st[b * c->NR + q].it : hp->jacobi_iters;
    if (err == -2) return fail(CIMCS_CUDA_ERROR, "update kernel: item flags timed out");
    if (method == CIMCS_CDP_JACOBI && err != 0x7f7f7f7f && err != INT_MAX)
        return fail(CIMCS_INPUT_ERROR,
                    "jacobi_solve: singular diagonal at active index " + std::to_string(err));
    return 0;
}

int cimcs_refit(cimcs_ctx* c, int32_t R, const int32_t* sigma, const double* R_prev,
                double* R_out, const cimcs_hyper* hp) {
    return cimcs_cdp_minimize(c, R, sigma, R_prev, CIMCS_CDP_JACOBI, hp, R_out, nullptr);
}

int cimcs_score(cimcs_ctx* c, int32_t R, const double* Rsig, const int32_t* sigma, double lambda,
                double* objective, double* rmse, double* hamming) {
    if (int rc = check_ready(c, R)) return rc;
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    if (int rc = reset_flags(c, R)) return rc;
    AltParams ap{};
    ap.lambda = lambda;
    if (int rc = set_alt(c, ap)) return rc;
    if (int rc = upload_traj(c, Rsig, c->Rs, R)) return rc;
    if (int rc = upload_sig(c, sigma, c->sig, R)) return rc;
    cimcs_hyper h;
    cimcs_hyper_default(&h);
    const StepScalars s = make_scalars(&h);
    int rc = c->st64() ? mask_T<double>(c, c->W0) : mask_T<float>(c, c->W0);
    if (!rc) rc = enqueue_score(c, s, 0, nullptr, false);
    const int nT = c->B * c->NR;
    std::vector<double> o(nT), r(nT), h_(nT);
    if (!rc) {
        cudaMemcpyAsync(o.data(), c->obj, nT * 8, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(r.data(), c->rmse, nT * 8, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(h_.data(), c->ham, nT * 8, cudaMemcpyDeviceToHost, c->stream);
    }
    CK(cudaStreamSynchronize(c->stream));
    if (rc) return rc;
    for (int b = 0; b < c->B; ++b)
        for (int q = 0; q < R; ++q) {
            if (objective) objective[b * R + q] = o[b * c->NR + q];
            if (rmse) rmse[b * R + q] = r[b * c->NR + q];
            if (hamming) hamming[b * R + q] = h_[b * c->NR + q];
        }
    return 0;
}

int cimcs_solve(cimcs_ctx* c, int32_t R, int32_t backend, const cimcs_hyper* hp, int32_t cdp,
                const uint64_t* seeds, const double* R_init, int32_t track_best, double* R_out,
                int32_t* sigma_out, cimcs_record* hist, int32_t* n_hist, int32_t* fail_alt,
                int32_t* fail_index) {
    if (int rc = check_ready(c, R)) return rc;
    if (int rc = validate(hp)) return rc;
    if (backend != CIMCS_MFZ_BN && backend != CIMCS_MFZ_CN && backend != CIMCS_PP)
        return fail(CIMCS_CONFIG_ERROR, "backend must be mfz-bn, mfz-cn or pp");
    const bool pp = backend == CIMCS_PP;
    if (pp && !(hp->j > 0.0))
        return fail(CIMCS_CONFIG_ERROR, "measured_amplitude: j must be positive");
    if (cdp != CIMCS_CDP_JACOBI && cdp != CIMCS_CDP_CG)
        return fail(CIMCS_CONFIG_ERROR, "cdp must be jacobi or cg");
    if (cdp == CIMCS_CDP_CG && c->world > 1)
        return fail(CIMCS_CONFIG_ERROR, "cdp=cg is not supported on row-sharded contexts");
    // the reference's DFT transform-chain problems always use CG (orchestrator.cpp:128-133);
    // the DCT chain stands in for config 3's dense matrix and keeps the requested refit
    if (c->mri && c->mri_kind == 0) cdp = CIMCS_CDP_CG;
    if (!seeds) return fail(CIMCS_INPUT_ERROR, "null seeds");
    CK(cudaSetDevice(c->device));
    const int NR = slots_for(c, R);
    if (int rc = ensure_state(c, NR)) return rc;
    // fp32 symmetric path: the Jacobi refit runs compacted to the union of supports
    const bool cmp = cdp == CIMCS_CDP_JACOBI && !pp && cmp_refit_ok(c);
    const bool cmp64 = cdp == CIMCS_CDP_JACOBI && !pp && cmp64_refit_ok(c);
    if (cdp == CIMCS_CDP_CG)
        if (int rc = ensure_cg(c)) return rc;
    if (pp)
        if (int rc = ensure_pp(c)) return rc;
    if (int rc = upload_pump(c, hp)) return rc;
    const int nalt = hp->velo + 1;
    const int nT = c->B * NR;
    if (c->hist_cap < nalt * nT) {
        if (c->hist) cudaFree(c->hist);
        c->hist = nullptr;
        if (int rc = dalloc(c, &c->hist, (size_t)nalt * nT * sizeof(DevRecord))) return rc;
        c->hist_cap = nalt * nT;
    }
    const int bn = backend == CIMCS_MFZ_BN;
    const StepScalars s = make_scalars(hp);
    const int ntraj = c->B * R;
    const size_t nc0 = (size_t)ntraj * c->N;

    // host streams + pinned double buffer for c0
    std::vector<HostRng> rngs;
    rngs.reserve(ntraj);
    for (int t = 0; t < ntraj; ++t) rngs.emplace_back(seeds[t]);
    if (c->pin_c0_elems < nc0) {
        if (c->pin_c0) cudaFreeHost(c->pin_c0);
        c->pin_c0 = nullptr;
        CK(cudaMallocHost(&c->pin_c0, 2 * nc0 * 8));
        c->pin_c0_elems = nc0;
    }
    if (c->dc0_elems < nc0) {
        if (c->dc0) cudaFree(c->dc0);
        c->dc0 = nullptr;
        drop_graphs(c);  // the CIM graph reads dc0
        if (int rc = dalloc(c, &c->dc0, nc0 * 8)) return rc;
        c->dc0_elems = nc0;
    }
    double* pinned = c->pin_c0;
    double* dc0 = c->dc0;
    std::vector<AltParams> alts(nalt);
    for (int i = 0; i < nalt; ++i)
        alts[i] = make_alt(hp, eta_schedule(i, hp->eta_init, hp->eta_end, hp->velo), i);
    AltParams* halts = nullptr;
    CK(cudaMallocHost(&halts, nalt * sizeof(AltParams)));
    std::unique_ptr<AltParams, decltype(&cudaFreeHost)> alt_guard(halts, &cudaFreeHost);
    std::copy(alts.begin(), alts.end(), halts);

    Events ev(4 * nalt + 2);
    Events slot_done(2);
    cudaEventRecord(ev.ev[4 * nalt], c->stream);

    // initial state: R_init (default hz), flags, best objective = +inf
    int rc = reset_flags(c, R);
    if (!rc) {
        if (R_init)
            rc = upload_traj(c, R_init, c->Rs, R);
        else
            rc = c->st64() ? rinit_hz_T<double>(c, R) : rinit_hz_T<float>(c, R);
    }
    if (rc) return rc;
    CK(cudaMemsetAsync(c->sig, 0, c->state_elems(), c->stream));
    {
        std::vector<double> inf(nT, INFINITY);
        CK(cudaMemcpyAsync(c->best_obj, inf.data(), nT * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemsetAsync(c->improved, 0, nT * 4, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // `inf` leaves scope
    }
    if (track_best) {
        CK(cudaMemcpyAsync(c->bestR, c->Rs, c->state_elems() * c->elt(), cudaMemcpyDeviceToDevice,
                           c->stream));
        CK(cudaMemsetAsync(c->bestS, 0, c->state_elems(), c->stream));
    }

    // graphs: [init + steps], [support + jacobi], [score + finalize + median (+best)]
    // The history slot differs per alternation, so the score graph is per-alternation
    // cheap; the two heavy graphs are captured once and replayed.
    // the two heavy graphs are cached across solves with the same shape and
    // schedule (the scalars they bake in are part of the key)
    if (c->use_graphs) {
        auto bits = [](double v) {
            long long u;
            std::memcpy(&u, &v, 8);
            return u;
        };
        const std::vector<long long> key = {R, NR, bn, hp->n_steps, hp->jacobi_iters,
                                            (long long)(uintptr_t)dc0, bits(s.dt), bits(s.rt),
                                            bits(s.nbeta), bits(s.Kj), bits(s.minus_j),
                                            bits(s.dt_c), c->B, c->N, cdp, hp->cg_max_iters,
                                            bits(hp->cg_tol), backend};
        if (key != c->graph_key || (!pp && !c->g_cim) || (!cmp && !cmp64 && !c->g_refit)) {
            drop_graphs(c);
            Graph gc, gr;
            if (!pp)  // the Positive-P CIM call is host-driven (chunked noise upload)
                rc = capture(c, gc, [&] {
                    int r2 = run_init(c, R, bn, dc0, nullptr, s.rt);
                    return r2 ? r2 : enqueue_steps(c, bn, s, hp->n_steps);
                });
            if (!rc && !cmp && !cmp64)
                rc = capture(c, gr, [&] {
                    if (cdp == CIMCS_CDP_CG) {
                        int r2 = run_support(c);
                        return r2 ? r2 : enqueue_cg(c, s, hp);
                    }
                    return enqueue_refit(c, s, hp->jacobi_iters, true);
                });
            if (rc) return rc;
            c->g_cim = gc.exec;
            c->g_refit = gr.exec;
            gc.exec = gr.exec = nullptr;
            c->graph_key = key;
        }
    }
    const int v_slot = cdp == CIMCS_CDP_CG ? 0 : hp->jacobi_iters & 1;
    if (!pp) gen_c0(rngs, c->N, pinned, c->host_threads);
    for (int i = 0; i < nalt; ++i) {
        double* slot = pinned + (size_t)(i & 1) * nc0;
        CK(cudaMemcpyAsync(c->alt, &halts[i], sizeof(AltParams), cudaMemcpyHostToDevice,
                           c->stream));
        if (!pp) {
            CK(cudaMemcpyAsync(dc0, slot, nc0 * 8, cudaMemcpyHostToDevice, c->stream));
            CK(cudaEventRecord(slot_done.ev[i & 1], c->stream));
        }
        NvtxRange nv_alt("alternation");
        CK(cudaEventRecord(ev.ev[4 * i + 0], c->stream));
        if (pp) {
            if ((rc = run_pp_cim(c, R, s, hp, rngs)) || (rc = pp_amplitude_to_c(c))) return rc;
        } else if (c->use_graphs) {
            CK(cudaGraphLaunch(c->g_cim, c->stream));
        } else {
            rc = run_init(c, R, bn, dc0, nullptr, s.rt);
            if (!rc) rc = enqueue_steps(c, bn, s, hp->n_steps);
            if (rc) return rc;
        }
        CK(cudaEventRecord(ev.ev[4 * i + 1], c->stream));
        if (i + 1 < nalt && !pp) {
            // draw the next alternation's c0 while the GPU runs this CIM call (its
            // pinned slot was last uploaded before the previous CIM call)
            CK(cudaEventSynchronize(slot_done.ev[(i + 1) & 1]));
            gen_c0(rngs, c->N, pinned + (size_t)((i + 1) & 1) * nc0, c->host_threads);
        }
        if (cmp) {
            if ((rc = enqueue_refit_compact(c, s, hp->jacobi_iters))) return rc;
        } else if (cmp64) {
            if ((rc = enqueue_refit_compact64(c, s, hp->jacobi_iters, true))) return rc;
        } else if (c->use_graphs) {
            CK(cudaGraphLaunch(c->g_refit, c->stream));
        } else if (cdp == CIMCS_CDP_CG) {
            if ((rc = run_support(c)) || (rc = enqueue_cg(c, s, hp))) return rc;
        } else if ((rc = enqueue_refit(c, s, hp->jacobi_iters, true))) {
            return rc;
        }
        CK(cudaEventRecord(ev.ev[4 * i + 2], c->stream));
        if ((rc = enqueue_score(c, s, v_slot, c->hist + (size_t)i * nT, track_best != 0)))
            return rc;
        CK(cudaEventRecord(ev.ev[4 * i + 3], c->stream));

    }
    cudaEventRecord(ev.ev[4 * nalt + 1], c->stream);

    // results
    if (c->world > 1) {  // every rank returns the full vectors
        if ((rc = allgather_sig(c, c->sig))) return rc;
        if (track_best && (rc = allgather_sig(c, c->bestS))) return rc;
    }
    const void* Rsrc = track_best ? c->bestR : c->Rs;
    const int8_t* Ssrc = track_best ? c->bestS : c->sig;
    if (track_best) {
        // best is only used when some alternation was recorded (isfinite(best_energy))
        // -- trajectories with no record keep their current R/sigma.
        std::vector<double> bo(nT);
        CK(cudaMemcpyAsync(bo.data(), c->best_obj, nT * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        bool all = true;
        for (int b = 0; b < c->B; ++b)
            for (int q = 0; q < R; ++q) all &= std::isfinite(bo[b * NR + q]);
        if (!all) {
            // copy current state into best slots of unrecorded trajectories
            std::vector<int> imp(nT, 0);
            for (int b = 0; b < c->B; ++b)
                for (int q = 0; q < R; ++q) imp[b * NR + q] = !std::isfinite(bo[b * NR + q]);
            CK(cudaMemcpyAsync(c->improved, imp.data(), nT * 4, cudaMemcpyHostToDevice,
                               c->stream));
            const int g = grid_for(c->state_elems());
            if (c->st64()) {
                DISPATCH_NR(NR, {
                    best_update_kernel<double, NR_><<<g, 256, 0, c->stream>>>(
                        c->improved, static_cast<const double*>(c->Rs), c->sig,
                        static_cast<double*>(c->bestR), c->bestS, c->ldN, c->B);
                });
            } else {
                DISPATCH_NR(NR, {
                    best_update_kernel<float, NR_><<<g, 256, 0, c->stream>>>(
                        c->improved, static_cast<const float*>(c->Rs), c->sig,
                        static_cast<float*>(c->bestR), c->bestS, c->ldN, c->B);
                });
            }
            CK(cudaStreamSynchronize(c->stream));
        }
    }
    if (R_out && (rc = download_traj(c, Rsrc, R_out, R))) return rc;
    if (sigma_out && (rc = download_sig(c, Ssrc, sigma_out, R))) return rc;
    std::vector<DevRecord> dh((size_t)nalt * nT);
    std::vector<int> nh(nT), fg(nT), fi(nT);
    CK(cudaMemcpyAsync(dh.data(), c->hist, dh.size() * sizeof(DevRecord), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaMemcpyAsync(nh.data(), c->n_hist, nT * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(fg.data(), c->fail_gstep, nT * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(fi.data(), c->fail_idx, nT * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    int err = 0;
    if (int rc_ = copy_sync(c, &err, c->err, 4, cudaMemcpyDeviceToHost)) return rc_;
    if (err == -2) return fail(CIMCS_CUDA_ERROR, "update kernel: item flags timed out");
    if (err != 0x7f7f7f7f && err != INT_MAX)
        return fail(CIMCS_INPUT_ERROR,
                    "jacobi_solve: singular diagonal at active index " + std::to_string(err));

    cimcs_timing& tm = c->timing;
    tm.total_ms = ev.ms(4 * nalt, 4 * nalt + 1);
    tm.cim_ms = tm.refit_ms = tm.score_ms = 0.0;
    for (int i = 0; i < nalt; ++i) {
        tm.cim_ms += ev.ms(4 * i + 0, 4 * i + 1);
        tm.refit_ms += ev.ms(4 * i + 1, 4 * i + 2);
        tm.score_ms += ev.ms(4 * i + 2, 4 * i + 3);
    }
    // kernels of this library per alternation: init + steps | support + sweeps |
    // score contraction, tp, finalize, median (+ best).  The small-N cluster loop
    // runs a whole CIM call / refit in one launch; CG counts its last iteration total.
    const bool cl = cluster_ok(c) && !pp;
    const int per = c->sym || c->sym64 ? 2 : 1;  // symmetric paths: tile kernel + update kernel
    tm.step_launches = (int64_t)nalt * (cl ? 1 : per * hp->n_steps + (pp ? 1 : 0));
    if (cdp == CIMCS_CDP_CG) {
        std::vector<CgTraj> st(nT);
        if (int rc_ = copy_sync(c, st.data(), c->cg_st, nT * sizeof(CgTraj), cudaMemcpyDeviceToHost))
            return rc_;
        int mx = 0;
        for (const CgTraj& t : st) mx = std::max(mx, t.it);
        tm.refit_launches = (int64_t)nalt * (6 + 3 * (int64_t)mx);
    } else {
        tm.refit_launches = (int64_t)nalt * (cl ? 1 : per * hp->jacobi_iters);
    }
    tm.other_launches = (int64_t)nalt * (2 + 4 + (track_best ? 1 : 0));
    tm.step_bytes = (double)c->B * c->N * (double)c->N * c->elt();  // dense G share
    tm.step_flops = 2.0 * c->B * (double)c->N * c->N * R;

    for (int b = 0; b < c->B; ++b)
        for (int q = 0; q < R; ++q) {
            const int dt = b * NR + q, ht = b * R + q;
            if (n_hist) n_hist[ht] = nh[dt];
            const bool failed = fg[dt] != kFreeTraj;
            if (fail_alt) fail_alt[ht] = failed ? fg[dt] / hp->n_steps : -1;
            if (fail_index) fail_index[ht] = failed ? (fi[dt] & ((1 << 30) - 1)) : -1;
            if (hist)
                for (int i = 0; i < nalt; ++i) {
                    cimcs_record& o = hist[(size_t)ht * nalt + i];
                    if (i < nh[dt]) {
                        const DevRecord& d = dh[(size_t)i * nT + dt];
                        o.i = d.i;
                        o.support = d.support;
                        o.eta = d.eta;
                        o.hamiltonian = d.hamiltonian;
                        o.rmse = d.rmse;
                        o.hamming = d.hamming;
                        o.min_e = d.min_e;
                        o.median_e = d.median_e;
                    } else {
                        std::memset(&o, 0, sizeof(o));
                        o.i = -1;
                    }
                }
        }
    return 0;
}

int cimcs_get_timing(const cimcs_ctx* c, cimcs_timing* out) {
    if (!c || !out) return fail(CIMCS_INPUT_ERROR, "null argument");
    *out = c->timing;
    return 0;
}

}  // extern "C"
