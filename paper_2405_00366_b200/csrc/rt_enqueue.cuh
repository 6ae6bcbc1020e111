// rt_enqueue.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): graph bodies: Euler steps, Jacobi / CG refits, scoring, Positive-P
// noise streaming.
#pragma once

namespace {

// n_iters launches of `mode` with W ping-pong (Euler steps or Jacobi sweeps) on
// the symmetric path (pipelining instance groups over two streams was measured
// slower: DESIGN.md section 4).
int enqueue_sym_loop(cimcs_ctx* c, int mode, GemvArgs a, int n_iters, bool steps) {
    for (int k = 0; k < n_iters; ++k) {
        if (steps) a.step = k;
        a.Win = (k & 1) ? c->W1 : c->W0;
        a.Wout = (k & 1) ? c->W0 : c->W1;
        if (int rc = launch_gemv(c, mode, a)) return rc;
    }
    return 0;
}

int enqueue_steps(cimcs_ctx* c, int bn, const StepScalars& s, int n_steps) {
    GemvArgs a = base_args(c, s);
    a.pump = c->pump;
    a.Hdbg = nullptr;
    if (cluster_ok(c)) {  // all n_steps in one launch; final w in W[n_steps & 1]
        a.step = 0;
        a.Win = c->W0;
        a.Wout = (n_steps & 1) ? c->W1 : c->W0;
        return launch_cluster(c, bn ? EPI_STEP_BN : EPI_STEP_CN, a, n_steps);
    }
    if (c->sym || c->sym64)
        return enqueue_sym_loop(c, bn ? EPI_STEP_BN : EPI_STEP_CN, a, n_steps, true);
    for (int k = 0; k < n_steps; ++k) {
        a.step = k;
        a.Win = (k & 1) ? c->W1 : c->W0;
        a.Wout = (k & 1) ? c->W0 : c->W1;
        if (int rc = launch_gemv(c, bn ? EPI_STEP_BN : EPI_STEP_CN, a)) return rc;
        if (int rc = allgather_w(c, a.Wout)) return rc;  // row sharding: exchange w
    }
    return reconcile_cim(c);
}

// support + masked Jacobi sweeps (graph-capturable).  Final V in W[iters&1].
int enqueue_refit(cimcs_ctx* c, const StepScalars& s, int iters, bool do_support) {
    if (do_support) {
        if (int rc = run_support(c)) return rc;
    }
    if (int rc = allgather_w(c, c->W0)) return rc;
    GemvArgs a = base_args(c, s);
    if (cluster_ok(c) && iters > 0) {  // all sweeps in one launch; final V in W[iters & 1]
        a.Win = c->W0;
        a.Wout = (iters & 1) ? c->W1 : c->W0;
        return launch_cluster(c, EPI_JACOBI, a, iters);
    }
    if (c->sym || c->sym64) {
        if (int rc = enqueue_sym_loop(c, EPI_JACOBI, a, iters, false)) return rc;
        return 0;
    }
    for (int it = 0; it < iters; ++it) {
        a.Win = (it & 1) ? c->W1 : c->W0;
        a.Wout = (it & 1) ? c->W0 : c->W1;
        if (int rc = launch_gemv(c, EPI_JACOBI, a)) return rc;
        if (int rc = allgather_w(c, a.Wout)) return rc;
    }
    if (c->world > 1) {
        if (int rc = allgather_state(c, c->Rs)) return rc;
        NK(ncclAllReduce(c->err, c->err, 1, ncclInt32, ncclMin, c->comm, c->stream));
    }
    return 0;
}

// The compacted Jacobi refit of the fp32 symmetric path (cmp_kernels.cuh):
// support -> union of the replicas' supports per instance -> (host reads the
// largest union) -> gathered tiles / state -> the unchanged symmetric sweeps on
// the compacted problem -> R scattered back -> the full W[iters & 1] = R o sigma
// that the scorer reads.  Eager (the compacted size is data-dependent).
bool cmp_refit_ok(const cimcs_ctx* c) {
    return c->sym && !c->tshard && c->cmp_opt && c->cU && !c->mri;
}

int enqueue_refit_compact(cimcs_ctx* c, const StepScalars& s, int iters) {
    if (int rc = run_support(c)) return rc;
    CK(cudaMemsetAsync(c->cMax, 0, 4, c->stream));
    DISPATCH_NR_TC(c->NR, {
        cmp_union_kernel<NR_><<<c->B, 1024, 0, c->stream>>>(c->sig, c->N, c->ldN, c->cU,
                                                            c->cCnt, c->cMax);
    });
    CK(cudaGetLastError());
    int mx = 0;
    if (int rc = copy_sync(c, &mx, c->cMax, 4, cudaMemcpyDeviceToHost)) return rc;
    // Dense unions: the compacted problem is padded to 128-row blocks, which can exceed the
    // state's leading dimension ldN = round_up(N, 32) (N = 577: 5 blocks = 640 > 608; the
    // union index list and the compacted state are [B][ldN]).  Nothing to gain then: the
    // full refit.
    if ((mx + kSyT - 1) / kSyT * kSyT > c->ldN) return enqueue_refit(c, s, iters, false);
    if (mx > 0 && iters > 0) {
        const int nRBc = (mx + kSyT - 1) / kSyT, ntric = nRBc * (nRBc + 1) / 2;
        cmp_gather_tiles_kernel<<<dim3(ntric, c->B), 256, 0, c->stream>>>(
            static_cast<const __half*>(c->dG), c->ntri, c->nRB, c->cU, c->ldN, nRBc, ntric, c->Gc);
        DISPATCH_NR_TC(c->NR, {
            cmp_gather_state_kernel<NR_><<<grid_for((size_t)c->B * c->ldN), 256, 0, c->stream>>>(
                static_cast<const float*>(c->Rs), c->sig, static_cast<const float*>(c->dD),
                static_cast<const float*>(c->dhz), c->cU, c->ldN, c->B, c->Rc, c->sigc, c->Dc,
                c->hzc, static_cast<float*>(c->W0));
        });
        CK(cudaGetLastError());
        // swap the context to the compacted problem (same ldN / layouts, fewer blocks)
        struct Swap {
            cimcs_ctx* c;
            int N, nRB, ntri, nSB, symS;
            void *dG, *Rs, *dD, *dhz;
            int8_t* sig;
            ~Swap() {
                c->N = N;
                c->nRB = nRB;
                c->ntri = ntri;
                c->nSB = nSB;
                c->symS = symS;
                c->dG = dG;
                c->Rs = Rs;
                c->dD = dD;
                c->dhz = dhz;
                c->sig = sig;
                c->cmp_active = false;
            }
        } sw{c, c->N, c->nRB, c->ntri, c->nSB, c->symS, c->dG, c->Rs, c->dD, c->dhz, c->sig};
        c->N = mx;
        c->nRB = nRBc;
        c->ntri = ntric;
        c->symS = 2;  // 2 x 2-tile items: enough of them to balance 148 CTAs
        c->nSB = (nRBc + c->symS - 1) / c->symS;
        c->dG = c->Gc;
        c->Rs = c->Rc;
        c->dD = c->Dc;
        c->dhz = c->hzc;
        c->sig = c->sigc;
        c->cmp_active = true;
        if (int rc = sym_sync_w(c, c->W0)) return rc;
        GemvArgs a = base_args(c, s);
        if (int rc = enqueue_sym_loop(c, EPI_JACOBI, a, iters, false)) return rc;
    }
    if (mx > 0 && iters > 0) {
        DISPATCH_NR_TC(c->NR, {
            cmp_scatter_kernel<NR_><<<grid_for((size_t)c->B * c->ldN), 256, 0, c->stream>>>(
                c->Rc, c->cU, c->ldN, c->B, static_cast<float*>(c->Rs));
        });
        CK(cudaGetLastError());
    }
    return mask_T<float>(c, (iters & 1) ? c->W1 : c->W0);  // what the scorer reads
}

// fp64 path: the segment-preserving compacted refit (cmp_kernels.cuh, cmp64) --
// bitwise the full refit's result
bool cmp64_refit_ok(const cimcs_ctx* c) {
    return c->sym64 && c->cmp_opt && c->cU6 && (c->N + cmp64::kSeg - 1) / cmp64::kSeg <= cmp64::kMaxSeg &&
           c->nSB6 == (c->N + cmp64::kSeg - 1) / cmp64::kSeg;
}

int enqueue_refit_compact64(cimcs_ctx* c, const StepScalars& s, int iters, bool do_support) {
    if (do_support)
        if (int rc = run_support(c)) return rc;
    const int nseg = c->nSB6, B = c->B;
    CK(cudaMemsetAsync(c->cMax, 0, 4, c->stream));
    CK(cudaMemsetAsync(c->cSegc, 0, (size_t)B * nseg * 4, c->stream));
    DISPATCH_NR_TC(c->NR, {
        cmp_union_kernel<NR_><<<B, 1024, 0, c->stream>>>(c->sig, c->N, c->ldN, c->cU, c->cCnt,
                                                         c->cMax);
    });
    cmp64_segcount_kernel<<<grid_for((size_t)B * c->ldN), 256, 0, c->stream>>>(
        c->cU, c->cCnt, c->ldN, nseg, B, c->cSegc);
    CK(cudaGetLastError());
    std::vector<int> segc((size_t)B * nseg), pfx((size_t)B * nseg), off(nseg, -1);
    if (int rc = copy_sync(c, segc.data(), c->cSegc, segc.size() * 4, cudaMemcpyDeviceToHost))
        return rc;
    // compacted segment widths: the batch maximum, rounded up to 64-row blocks
    std::vector<int2> seg;
    int Nc = 0;
    for (int sg = 0; sg < nseg; ++sg) {
        int w = 0;
        for (int b = 0; b < B; ++b) w = std::max(w, segc[(size_t)b * nseg + sg]);
        w = (w + kT6 - 1) / kT6 * kT6;
        if (!w) continue;  // no instance uses it: its partial is an exact +0
        off[sg] = Nc;
        seg.push_back(make_int2(Nc / kT6, w / kT6));
        Nc += w;
    }
    for (int b = 0; b < B; ++b)
        for (int sg = 0, a = 0; sg < nseg; ++sg) {
            pfx[(size_t)b * nseg + sg] = a;
            a += segc[(size_t)b * nseg + sg];
        }
    // Dense unions: every segment's width rounds UP to 64 rows, so the compacted size can
    // exceed the state's leading dimension ldN = round_up(N, 32) (N = 1100: 512 + 512 + 128
    // = 1152 > 1120).  Nothing to gain then: the full refit, bitwise the same result.
    if (Nc > c->ldN) return enqueue_refit(c, s, iters, false);
    if (Nc > 0 && iters > 0) {
        const int nsc = (int)seg.size(), nRBc = Nc / kT6, ntric = nRBc * (nRBc + 1) / 2;
        // the LPT schedule of the variable-width segment items
        std::vector<std::pair<int, int2>> items;
        for (int b = 0; b < B; ++b)
            for (int P = 0; P < nsc; ++P)
                for (int Q = P; Q < nsc; ++Q) {
                    const int nI = seg[P].y, nJ = seg[Q].y;
                    items.push_back({sym_item_cost(P == Q, nI, nJ), make_int2(b, P << 16 | Q)});
                }
        if ((int)items.size() > c->cmp_items_cap) return fail(CIMCS_CUDA_ERROR, "cmp64 schedule capacity");
        std::vector<int2> flat;
        std::vector<int> beg;
        c->cmp_sched.grid = lpt_place(items, c->sched_n(), flat, beg);
        c->cmp_sched.nb = B;
        c->cmp_sched.nRB = nRBc;
        c->cmp_sched.S = kS6;
        int rc;
        if ((rc = copy_sync(c, c->cmp_sched.items, flat.data(), flat.size() * sizeof(int2),
                            cudaMemcpyHostToDevice)) ||
            (rc = copy_sync(c, c->cmp_sched.sched, beg.data(), beg.size() * 4,
                            cudaMemcpyHostToDevice)) ||
            (rc = copy_sync(c, c->cSeg, seg.data(), seg.size() * sizeof(int2),
                            cudaMemcpyHostToDevice)) ||
            (rc = copy_sync(c, c->cSegOff, off.data(), off.size() * 4, cudaMemcpyHostToDevice)) ||
            (rc = copy_sync(c, c->cPfx, pfx.data(), pfx.size() * 4, cudaMemcpyHostToDevice)))
            return rc;
        CK(cudaMemsetAsync(c->cU6, 0xff, (size_t)B * c->ldN * 4, c->stream));  // -1: pad
        cmp64_map_kernel<<<grid_for((size_t)B * c->ldN), 256, 0, c->stream>>>(
            c->cU, c->cCnt, c->cPfx, c->cSegOff, c->ldN, nseg, B, c->cU6);
        cmp64_gather_tiles_kernel<<<dim3(ntric, B), 256, 0, c->stream>>>(
            static_cast<const double*>(c->dG6), c->ntri6, c->nRB6, c->cU6, c->ldN, nRBc, ntric,
            static_cast<double*>(c->Gc6));
        DISPATCH_NR_TC(c->NR, {
            cmp64_gather_state_kernel<NR_><<<grid_for((size_t)B * c->ldN), 256, 0, c->stream>>>(
                static_cast<const double*>(c->Rs), c->sig, static_cast<const double*>(c->dD),
                static_cast<const double*>(c->dhz), c->cU6, c->ldN, B, c->Rc6, c->sigc, c->Dc6,
                c->hzc6, static_cast<double*>(c->W0));
        });
        CK(cudaGetLastError());
        struct Swap {  // the context runs the compacted problem until this goes out of scope
            cimcs_ctx* c;
            int N, nRB6, ntri6, nSB6;
            void *dG6, *Rs, *dD, *dhz;
            int8_t* sig;
            ~Swap() {
                c->N = N;
                c->nRB6 = nRB6;
                c->ntri6 = ntri6;
                c->nSB6 = nSB6;
                c->dG6 = dG6;
                c->Rs = Rs;
                c->dD = dD;
                c->dhz = dhz;
                c->sig = sig;
                c->cmp_active = false;
            }
        } sw{c, c->N, c->nRB6, c->ntri6, c->nSB6, c->dG6, c->Rs, c->dD, c->dhz, c->sig};
        c->N = Nc;
        c->nRB6 = nRBc;
        c->ntri6 = ntric;
        c->nSB6 = nsc;
        c->dG6 = c->Gc6;
        c->Rs = c->Rc6;
        c->dD = c->Dc6;
        c->dhz = c->hzc6;
        c->sig = c->sigc;
        c->cmp_active = true;
        if ((rc = sym_sync_w(c, c->W0))) return rc;
        GemvArgs a = base_args(c, s);
        if ((rc = enqueue_sym_loop(c, EPI_JACOBI, a, iters, false))) return rc;
    }
    if (Nc > 0 && iters > 0) {
        DISPATCH_NR_TC(c->NR, {
            cmp64_scatter_kernel<NR_><<<grid_for((size_t)B * c->ldN), 256, 0, c->stream>>>(
                c->Rc6, c->cU6, c->ldN, B, static_cast<double*>(c->Rs));
        });
        CK(cudaGetLastError());
    }
    return mask_T<double>(c, (iters & 1) ? c->W1 : c->W0);
}

// ---------------------------------------------------- CG refit (cdp="cg")
int ensure_cg(cimcs_ctx* c) {  // outside any capture: allocates
    if (c->cgX) return 0;
    const size_t n = c->state_elems();
    for (double** p : {&c->cgX, &c->cgR, &c->cgP, &c->cgGp})
        if (int rc = dalloc(c, p, n * 8)) return rc;
    if (int rc = dalloc(c, &c->cg_act, n * 4)) return rc;
    if (int rc = dalloc(c, &c->cg_st, (size_t)c->B * c->NR * sizeof(CgTraj))) return rc;
    if (int rc = dalloc(c, &c->cg_live, 2 * 4)) return rc;
    if (!c->side) CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    return 0;
}

CgArgs cg_args(cimcs_ctx* c, const cimcs_hyper* hp) {
    CgArgs a{};
    a.Rs = c->Rs;
    a.sig = c->sig;
    a.hz = c->dhz;
    a.X = c->cgX;
    a.Rr = c->cgR;
    a.P = c->cgP;
    a.Gp = c->cgGp;
    a.act = c->cg_act;
    a.st = static_cast<CgTraj*>(c->cg_st);
    a.fail_gstep = c->fail_gstep;
    a.W = c->W0;
    a.n_live = c->cg_live;
    a.tc = wcanon(c);
    a.ldJ = c->ldJ;
    a.N = c->N;
    a.ldN = c->ldN;
    a.max_iters = hp->cg_max_iters;
    a.tol = hp->cg_tol;
    return a;
}

template <typename T>
int cg_launch(cimcs_ctx* c, int which, const CgArgs& a) {
    const int nT = c->B * c->NR;
    DISPATCH_NR(c->NR, {
        if (which == 0) cg_init_kernel<T, NR_><<<nT, kCgThreads, 0, c->stream>>>(a);
        else if (which == 1) cg_iter_kernel<T, NR_><<<nT, kCgThreads, 0, c->stream>>>(a);
        else cg_final_kernel<T, NR_><<<nT, kCgThreads, 0, c->stream>>>(a);
    });
    CK(cudaGetLastError());
    return 0;
}

int cg_kernel(cimcs_ctx* c, int which, const CgArgs& a) {
    return c->st64() ? cg_launch<double>(c, which, a) : cg_launch<float>(c, which, a);
}

// G p for every trajectory (the EPI_MATVEC contraction of W0 into cgGp)
int cg_matvec(cimcs_ctx* c, const StepScalars& s) {
    GemvArgs g = base_args(c, s);
    g.Win = c->W0;
    g.Wout = nullptr;
    g.Mv = c->cgGp;
    return launch_gemv(c, EPI_MATVEC, g);
}

int cg_cond(cimcs_ctx* c, cudaGraphConditionalHandle h, int use) {
    cg_cond_kernel<<<1, 1, 0, c->stream>>>(c->cg_live, c->cg_live + 1, h, use);
    CK(cudaGetLastError());
    return 0;
}

// The whole masked CG refit of every trajectory on its current support
// (sig), Rs in/out; afterwards W0 = Rs∘sig for the scorer.  Inside a stream
// capture the data-dependent loop is a conditional WHILE node (the body is
// captured on the side stream), so the refit stays one graph launch; outside
// a capture the host polls the live count after every iteration.
int enqueue_cg(cimcs_ctx* c, const StepScalars& s, const cimcs_hyper* hp) {
    if (c->world > 1) return fail(CIMCS_CONFIG_ERROR, "cdp=cg is not supported on row-sharded contexts");
    if (int rc = ensure_cg(c)) return rc;
    cudaStreamCaptureStatus cs;
    cudaGraph_t cgraph = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CK(cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &cgraph, &deps, &ndeps));
    const bool in_graph = cs == cudaStreamCaptureStatusActive;
    cudaGraphConditionalHandle h{};
    if (in_graph) CK(cudaGraphConditionalHandleCreate(&h, cgraph, 0, 0));
    const CgArgs a = cg_args(c, hp);
    int rc = c->st64() ? mask_T<double>(c, c->W0) : mask_T<float>(c, c->W0);
    if (!rc) rc = cg_matvec(c, s);  // G x0
    if (!rc) rc = cg_kernel(c, 0, a);
    if (!rc) rc = sym_sync_w(c, c->W0);
    if (!rc) rc = cg_cond(c, h, in_graph ? 1 : 0);
    if (rc) return rc;
    if (in_graph) {
        CK(cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &cgraph, &deps, &ndeps));
        cudaGraphNodeParams np{};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, cgraph, deps, ndeps, &np));
        cudaGraph_t body = np.conditional.phGraph_out[0];
        CK(cudaStreamUpdateCaptureDependencies(c->stream, &node, 1,
                                               cudaStreamSetCaptureDependencies));
        cudaStream_t main = c->stream;
        c->stream = c->side;
        cudaError_t e = cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0,
                                                      cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            rc = cg_matvec(c, s);
            if (!rc) rc = cg_kernel(c, 1, a);
            if (!rc) rc = sym_sync_w(c, c->W0);
            if (!rc) rc = cg_cond(c, h, 1);
            cudaGraph_t out;
            e = cudaStreamEndCapture(c->stream, &out);
        }
        c->stream = main;
        if (rc) return rc;
        CK(e);
    } else {
        int live = 0;
        CK(cudaMemcpyAsync(&live, c->cg_live + 1, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        while (live > 0) {
            if ((rc = cg_matvec(c, s)) || (rc = cg_kernel(c, 1, a)) ||
                (rc = sym_sync_w(c, c->W0)) || (rc = cg_cond(c, h, 0)))
                return rc;
            CK(cudaMemcpyAsync(&live, c->cg_live + 1, 4, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
    }
    rc = cg_kernel(c, 2, a);
    if (!rc) rc = c->st64() ? mask_T<double>(c, c->W0) : mask_T<float>(c, c->W0);
    return rc;
}

template <typename T>
int enqueue_median_T(cimcs_ctx* c, DevRecord* hist_alt) {
    int P = 1;
    while (P < c->N) P <<= 1;
    const size_t smem = (size_t)P * sizeof(T);
    if (smem > 200 * 1024) return 0;  // median left as NaN beyond 25k/51k spins
    DISPATCH_NR(c->NR, {
        auto k = median_kernel<T, NR_>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<c->B * c->NR, 1024, smem, c->stream>>>(static_cast<const T*>(c->E), c->fail_gstep,
                                                  c->N, c->ldN, P, hist_alt);
    });
    CK(cudaGetLastError());
    return 0;
}

// scorer on V = W[v_slot]: score GEMV + finalize (+ history, + best tracking)
int enqueue_score(cimcs_ctx* c, const StepScalars& s, int v_slot, DevRecord* hist_alt,
                  bool track_best) {
    GemvArgs a = base_args(c, s);
    a.Win = v_slot ? c->W1 : c->W0;
    a.Wout = nullptr;
    if (int rc = launch_gemv(c, EPI_SCORE, a)) return rc;
    const int nT = c->B * c->NR;
    DISPATCH_NR(c->NR, {
        tp_kernel<NR_><<<nT, 256, 0, c->stream>>>(c->part, nRB_of(c), c->sig, c->dxi, c->row0,
                                                  c->row1, c->ldN, c->has_truth ? 1 : 0, c->tp);
    });
    CK(cudaGetLastError());
    if (c->world > 1)
        NK(ncclAllReduce(c->tp, c->tp, (size_t)nT * 5, ncclFloat64, ncclSum, c->comm, c->stream));
    finalize_kernel<<<(nT + 127) / 128, 128, 0, c->stream>>>(
        c->tp, nT, c->minE, c->fail_gstep, c->alt, c->N, c->has_truth ? 1 : 0, hist_alt,
        c->n_hist, track_best ? c->best_obj : nullptr, c->improved, c->obj, c->rmse, c->ham);
    CK(cudaGetLastError());
    if (hist_alt && c->world > 1) {
        if (int rc = allgather_state(c, c->E)) return rc;
    }
    if (hist_alt) {
        if (int rc = c->st64() ? enqueue_median_T<double>(c, hist_alt)
                                           : enqueue_median_T<float>(c, hist_alt))
            return rc;
    }
    if (track_best) {
        const int g = grid_for(c->state_elems());
        if (c->st64()) {
            DISPATCH_NR(c->NR, {
                best_update_kernel<double, NR_><<<g, 256, 0, c->stream>>>(
                    c->improved, static_cast<const double*>(c->Rs), c->sig,
                    static_cast<double*>(c->bestR), c->bestS, c->ldN, c->B);
            });
        } else {
            DISPATCH_NR(c->NR, {
                best_update_kernel<float, NR_><<<g, 256, 0, c->stream>>>(
                    c->improved, static_cast<const float*>(c->Rs), c->sig,
                    static_cast<float*>(c->bestR), c->bestS, c->ldN, c->B);
            });
        }
        CK(cudaGetLastError());
    }
    return 0;
}

int check_ready(cimcs_ctx* c, int R) {
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    if (!c->built) return fail(CIMCS_INPUT_ERROR, "coupling not built (cimcs_build_coupling)");
    if (R < 1 || R > 16) return fail(CIMCS_INPUT_ERROR, "R must be in [1, 16]");
    return 0;
}

int validate(const cimcs_hyper* h) {
    if (!h) return fail(CIMCS_CONFIG_ERROR, "null hyper-parameters");
    if (!(h->dt > 0)) return fail(CIMCS_CONFIG_ERROR, "dt must be > 0");
    if (h->n_steps < 1) return fail(CIMCS_CONFIG_ERROR, "n_steps must be >= 1");
    if (!(h->tau > 0)) return fail(CIMCS_CONFIG_ERROR, "tau must be > 0");
    if (h->g2 < 0) return fail(CIMCS_CONFIG_ERROR, "g2 must be >= 0");
    if (h->eta_init < h->eta_end || h->eta_end < 0)
        return fail(CIMCS_CONFIG_ERROR, "need eta_init >= eta_end >= 0");
    if (h->velo < 1) return fail(CIMCS_CONFIG_ERROR, "velo must be >= 1");
    if (h->pump_kind != CIMCS_PUMP_SIGMOID && h->pump_kind != CIMCS_PUMP_LINEAR)
        return fail(CIMCS_CONFIG_ERROR, "pump_kind must be sigmoid or linear");
    return 0;
}

int upload_pump(cimcs_ctx* c, const cimcs_hyper* hp) {
    const std::vector<double> p = pump_table(hp);
    for (double v : p)
        if (!std::isfinite(v)) return fail(CIMCS_INPUT_ERROR, "mfz_step: non-finite pump");
    if (c->pump_cap < hp->n_steps) {
        // cached graphs bake the pump pointer: drop them with the old buffer
        drop_graphs(c);
        if (c->pump) cudaFree(c->pump);
        c->pump = nullptr;
        if (int rc = dalloc(c, &c->pump, (size_t)hp->n_steps * 8)) return rc;
        c->pump_cap = hp->n_steps;
    }
    if (int rc_ = copy_sync(c, c->pump, p.data(), (size_t)hp->n_steps * 8, cudaMemcpyHostToDevice)) return rc_;
    return 0;
}

int set_alt(cimcs_ctx* c, const AltParams& ap) {
    CK(cudaMemcpyAsync(c->alt, &ap, sizeof(AltParams), cudaMemcpyHostToDevice, c->stream));
    return 0;
}

// Host c0 generator pool: trajectory streams split contiguously over threads.
void gen_c0(std::vector<HostRng>& rngs, int N, double* out, int threads) {
    const int nt = (int)rngs.size();
    threads = std::max(1, std::min(threads, nt));
    auto work = [&](int t0, int t1) {
        for (int t = t0; t < t1; ++t) {
            double* o = out + (size_t)t * N;
            for (int i = 0; i < N; ++i) o[i] = 0.01 * rngs[t].gauss();  // init_mfz :27
        }
    };
    if (threads == 1) {
        work(0, nt);
        return;
    }
    std::vector<std::thread> pool;
    const int per = (nt + threads - 1) / threads;
    for (int k = 0; k < threads; ++k) {
        const int t0 = k * per, t1 = std::min(nt, t0 + per);
        if (t0 < t1) pool.emplace_back(work, t0, t1);
    }
    for (auto& th : pool) th.join();
}

// Host -> device upload of B variable-size pieces through two pinned slots:
// host threads pack a slot while the DMA engine drains the other.
template <class SizeF, class SrcF, class DstF>
int staged_upload(cimcs_ctx* c, int B, SizeF size_of, SrcF src_of, DstF dst_of) {
    const size_t slot = (size_t)64 << 20;
    if (c->pin_bytes < slot) {
        if (c->pin) cudaFreeHost(c->pin);
        c->pin = nullptr;
        CK(cudaMallocHost(&c->pin, 2 * slot));
        c->pin_bytes = slot;
    }
    cudaEvent_t done[2];
    CK(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    std::unique_ptr<cudaEvent_t[], void (*)(cudaEvent_t*)> guard(done, [](cudaEvent_t* e) {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
    });
    const int threads = std::max(1, std::min(c->host_threads, 16));
    int k = 0;
    char* base = reinterpret_cast<char*>(c->pin);
    for (int b = 0; b < B; ++b) {
        const size_t n = size_of(b);
        const char* src = src_of(b);
        char* dst = dst_of(b);
        for (size_t off = 0; off < n; off += slot, ++k) {
            const size_t len = std::min(slot, n - off);
            char* buf = base + (size_t)(k & 1) * slot;
            if (k >= 2) CK(cudaEventSynchronize(done[k & 1]));
            const int nt = len >= ((size_t)8 << 20) ? threads : 1;
            if (nt == 1) {
                std::memcpy(buf, src + off, len);
            } else {
                std::vector<std::thread> pool;
                const size_t per = (len + nt - 1) / nt;
                for (int t = 0; t < nt; ++t) {
                    const size_t o = (size_t)t * per;
                    if (o >= len) break;
                    pool.emplace_back([=] { std::memcpy(buf + o, src + off + o, std::min(per, len - o)); });
                }
                for (auto& th : pool) th.join();
            }
            CK(cudaMemcpyAsync(dst + off, buf, len, cudaMemcpyHostToDevice, c->stream));
            CK(cudaEventRecord(done[k & 1], c->stream));
        }
    }
    // the slots are reused by the next upload: drain them before returning
    if (k >= 1) CK(cudaEventSynchronize(done[(k - 1) & 1]));
    if (k >= 2) CK(cudaEventSynchronize(done[k & 1]));
    return 0;
}

struct Graph {
    cudaGraphExec_t exec = nullptr;
    ~Graph() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

template <typename F>
int capture(cimcs_ctx* c, Graph& g, F&& body) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = body();
    cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
    if (rc) {
        if (e == cudaSuccess) cudaGraphDestroy(graph);
        return rc;
    }
    CK(e);
    CK(cudaGraphInstantiate(&g.exec, graph, 0));
    cudaGraphDestroy(graph);
    return 0;
}

struct Events {
    std::vector<cudaEvent_t> ev;
    explicit Events(size_t n) : ev(n, nullptr) {
        for (auto& e : ev) cudaEventCreate(&e);
    }
    ~Events() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
    float ms(size_t a, size_t b) const {
        float t = 0.f;
        cudaEventElapsedTime(&t, ev[a], ev[b]);
        return t;
    }
};

// ------------------------------------------------------ Positive-P backend
constexpr int kPpChunk = 64;  // steps of unit normals per host -> device chunk

int ensure_pp(cimcs_ctx* c) {  // outside any capture
    if (c->mri)
        return fail(CIMCS_CONFIG_ERROR, "pp backend: not on matrix-free MRI problems (fp32 MFZ only)");
    if (c->tshard)
        return fail(CIMCS_CONFIG_ERROR, "pp backend is not supported on tile-sharded contexts");
    if (c->world > 1)
        return fail(CIMCS_CONFIG_ERROR, "pp backend is not supported on row-sharded contexts");
    const size_t n = c->state_elems();
    if (!c->Pn) {
        int rc;
        if ((rc = dalloc(c, &c->Pn, n * c->elt())) || (rc = dalloc(c, &c->Pm, n * c->elt())) ||
            (rc = dalloc(c, &c->MT, n * c->elt())))
            return rc;
    }
    const size_t nz = (size_t)kPpChunk * n;
    if (c->nz_elems < nz) {
        for (int k = 0; k < 2; ++k) {
            if (c->nzd[k]) cudaFree(c->nzd[k]);
            if (c->nzh[k]) cudaFreeHost(c->nzh[k]);
            c->nzd[k] = c->nzh[k] = nullptr;
        }
        for (int k = 0; k < 2; ++k) {
            if (int rc = dalloc(c, &c->nzd[k], nz * 8)) return rc;
            CK(cudaMallocHost(&c->nzh[k], nz * 8));
            std::memset(c->nzh[k], 0, nz * 8);  // padded slots stay zero
        }
        c->nz_elems = nz;
    }
    return 0;
}

// kc steps of unit normals per trajectory (make_noise_draw, solver_pp.cpp:9: N
// deviates per step from the trial stream), device layout [kc][B][ldN][NR]
void gen_noise(cimcs_ctx* c, std::vector<HostRng>& rngs, int Rreal, int kc, double* out) {
    const int nt = (int)rngs.size();
    const size_t S = c->state_elems();
    auto work = [&](int t0, int t1) {
        for (int t = t0; t < t1; ++t) {
            const int b = t / Rreal, r = t % Rreal;
            for (int k = 0; k < kc; ++k) {
                double* o = out + (size_t)k * S + ((size_t)b * c->ldN) * c->NR + r;
                for (int i = 0; i < c->N; ++i) o[(size_t)i * c->NR] = rngs[t].gauss();
            }
        }
    };
    const int threads = std::max(1, std::min(c->host_threads, nt));
    if (threads == 1) {
        work(0, nt);
        return;
    }
    std::vector<std::thread> pool;
    const int per = (nt + threads - 1) / threads;
    for (int k = 0; k < threads; ++k) {
        const int t0 = k * per, t1 = std::min(nt, t0 + per);
        if (t0 < t1) pool.emplace_back(work, t0, t1);
    }
    for (auto& th : pool) th.join();
}

template <typename T>
int pp_init_T(cimcs_ctx* c, int Rreal, const double* nz0, const StepScalars& s) {
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        init_pp_kernel<T, NR_><<<g, 256, 0, c->stream>>>(
            Rreal, c->N, c->ldN, c->B, static_cast<const T*>(c->Rs), static_cast<T*>(c->C),
            static_cast<T*>(c->E), static_cast<T*>(c->Pn), static_cast<T*>(c->Pm),
            static_cast<T*>(c->MT), static_cast<T*>(c->W0), c->fail_gstep, c->minE, nz0,
            s.pp_scale, s.rt);
    });
    CK(cudaGetLastError());
    return 0;
}

// One Positive-P CIM call (run_pp, solver_pp.cpp:100-132) for all trajectories.
// The unit normals are drawn on the host from each trajectory's reference
// stream (bit-exact) and uploaded in chunks of kPpChunk steps while the GPU
// integrates the previous chunk.  Host-driven (not captured).  Afterwards C
// holds mu and MT the last measured amplitude (the sigma source, run_pp :126-129).
int run_pp_cim(cimcs_ctx* c, int Rreal, const StepScalars& s, const cimcs_hyper* hp,
               std::vector<HostRng>& rngs) {
    const int n_steps = hp->n_steps, K = std::min(kPpChunk, n_steps);
    const int nch = (n_steps + K - 1) / K;
    const size_t S = c->state_elems();
    Events cp(2);
    auto stage = [&](int ch) -> int {
        const int sl = ch & 1, kc = std::min(K, n_steps - ch * K);
        gen_noise(c, rngs, Rreal, kc, c->nzh[sl]);
        CK(cudaMemcpyAsync(c->nzd[sl], c->nzh[sl], (size_t)kc * S * 8, cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaEventRecord(cp.ev[sl], c->stream));
        return 0;
    };
    int rc = stage(0);
    if (!rc && nch > 1) rc = stage(1);
    if (!rc)
        rc = c->st64() ? pp_init_T<double>(c, Rreal, c->nzd[0], s)
                                   : pp_init_T<float>(c, Rreal, c->nzd[0], s);
    if (!rc) rc = sym_sync_w(c, c->W0);  // symmetric-tile paths: the tiles of the first w
    GemvArgs a = base_args(c, s);
    a.pump = c->pump;
    a.Hdbg = nullptr;
    a.Pn = c->Pn;
    a.Pm = c->Pm;
    a.MT = c->MT;
    for (int ch = 0; ch < nch && !rc; ++ch) {
        const int k0 = ch * K, kc = std::min(K, n_steps - k0);
        for (int k = k0; k < k0 + kc && !rc; ++k) {
            a.step = k;
            a.Win = (k & 1) ? c->W1 : c->W0;
            a.Wout = (k & 1) ? c->W0 : c->W1;
            a.nz = c->nzd[ch & 1] + (size_t)(k - k0) * S;
            a.nz_next = k + 1 >= n_steps ? a.nz
                        : k + 1 < k0 + kc ? a.nz + S
                                          : c->nzd[(ch + 1) & 1];
            rc = launch_gemv(c, EPI_STEP_PP, a);
        }
        if (!rc && ch + 2 < nch) {
            CK(cudaEventSynchronize(cp.ev[ch & 1]));  // its pinned slot has been copied
            rc = stage(ch + 2);
        }
    }
    // the next call refills both pinned slots at once: the copies still queued
    // behind this call's kernels must have read them first
    CK(cudaEventSynchronize(cp.ev[0]));
    CK(cudaEventSynchronize(cp.ev[1]));
    return rc;
}

// C = the measured amplitude (CimCallResult::amplitude of the PP backend), so the
// support / refit path (support_kernel: sigma = C > 0) serves both backends
int pp_amplitude_to_c(cimcs_ctx* c) {
    CK(cudaMemcpyAsync(c->C, c->MT, c->state_elems() * c->elt(), cudaMemcpyDeviceToDevice,
                       c->stream));
    return 0;
}

}  // namespace
