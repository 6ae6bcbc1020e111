// rt_memory.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): allocation, stream-ordered copies, item schedules, state buffers,
// per-call scalars.
#pragma once

namespace {

// contraction-input layout: the streaming tcgen05 kernel reads W
// as the canonical [W | W_lo] operand (tc_wofs); the symmetric-tile path and
// the CUDA-core paths use [b][i][r] (coalesced float4 rows in the update)
inline int wcanon(const cimcs_ctx*) { return 0; }  // plain [b][i][r] on every path

void drop_graphs(cimcs_ctx* c) {
    if (c->g_cim) cudaGraphExecDestroy(c->g_cim);
    if (c->g_refit) cudaGraphExecDestroy(c->g_refit);
    c->g_cim = c->g_refit = nullptr;
    c->graph_key.clear();
}

void free_state(cimcs_ctx* c) {
    drop_graphs(c);
    void* ptrs[] = {c->Rs,  c->C,        c->E,          c->W0,  c->W1,       c->Hdbg,
                    c->bestR, c->sig,    c->bestS,      c->fail_gstep, c->fail_idx, c->n_hist,
                    c->improved, c->minE, c->part,      c->best_obj, c->obj, c->rmse, c->ham,
                    c->tp, c->fail_tmp, c->cgX, c->cgR, c->cgP, c->cgGp, c->cg_act,
                    c->cg_st, c->cg_live, c->WB0, c->WB1, c->WS0, c->WS1, c->WT0, c->WT1, c->Pn, c->Pm,
                    c->MT, c->nzd[0], c->nzd[1], c->dPart6};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    c->cgX = c->cgR = c->cgP = c->cgGp = nullptr;
    c->WB0 = c->WB1 = nullptr;
    c->WS0 = c->WS1 = nullptr;
    c->WT0 = c->WT1 = c->dPart6 = nullptr;
    if (c->dDone) cudaFree(c->dDone);
    c->dDone = nullptr;
    for (void* q : {(void*)c->cU, (void*)c->cCnt, (void*)c->cMax, (void*)c->Rc, (void*)c->Dc,
                    (void*)c->hzc, (void*)c->sigc, (void*)c->cU6, (void*)c->cSegc,
                    (void*)c->cPfx, (void*)c->cSegOff, (void*)c->cSeg, (void*)c->Rc6,
                    (void*)c->Dc6, (void*)c->hzc6, (void*)c->cmp_sched.items,
                    (void*)c->cmp_sched.sched})
        if (q) cudaFree(q);
    c->cU6 = c->cSegc = c->cPfx = c->cSegOff = nullptr;
    c->cSeg = nullptr;
    c->Rc6 = c->Dc6 = c->hzc6 = nullptr;
    c->cmp_sched = cimcs_ctx::SymSched{};
    c->cmp_items_cap = 0;
    c->cU = c->cCnt = c->cMax = nullptr;
    c->Rc = c->Dc = c->hzc = nullptr;
    c->sigc = nullptr;
    c->Pn = c->Pm = c->MT = nullptr;
    c->nzd[0] = c->nzd[1] = nullptr;
    for (double*& h : c->nzh)
        if (h) {
            cudaFreeHost(h);
            h = nullptr;
        }
    c->nz_elems = 0;
    c->cg_act = c->cg_live = nullptr;
    c->cg_st = nullptr;
    c->Rs = c->C = c->E = c->W0 = c->W1 = c->Hdbg = c->bestR = nullptr;
    c->sig = c->bestS = nullptr;
    c->fail_gstep = c->fail_idx = c->n_hist = c->improved = nullptr;
    c->minE = nullptr;
    c->part = c->best_obj = c->obj = c->rmse = c->ham = nullptr;
    c->tp = nullptr;
    c->fail_tmp = nullptr;
    c->NR = 0;
}

void free_problems(cimcs_ctx* c) {
    free_state(c);
    void* ptrs[] = {c->dA, c->dy, c->dM, c->dG, c->dG6, c->dD, c->dhz, c->dx, c->dxi,
                    c->dSg, c->dSpart, c->dMaskBr, c->dTw, c->dTarget,
                    c->dH, c->Gc, c->Gc6, c->dDctC, c->dDctMask, c->dDctY};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (auto& q : c->ssched) {
        cudaFree(q.items);
        cudaFree(q.sched);
    }
    c->ssched.clear();
    c->Gc = nullptr;
    c->Gc6 = nullptr;
    c->dSg = nullptr;
    c->dSpart = nullptr;
    c->dMaskBr = nullptr;
    c->dH = nullptr;
    c->dTw = nullptr;
    c->dTarget = nullptr;
    c->mri = false;
    c->mri_kind = 0;
    c->dDctC = nullptr;
    c->dDctMask = nullptr;
    c->dDctY = nullptr;
    c->spart_elems = 0;
    c->dA = c->dy = nullptr;
    c->dM = nullptr;
    c->dG = c->dG6 = nullptr;
    c->dD = c->dhz = nullptr;
    c->dx = nullptr;
    c->dxi = nullptr;
    c->B = c->N = c->ldN = 0;
    c->built = false;
}

// Device allocation, zero-filled ON THE CONTEXT STREAM: every later upload,
// kernel and download of the context is ordered after the fill by the stream
// itself (no device-wide sync; round 1 filled on the legacy stream, which does
// not order against the non-blocking context stream, and a second context's
// fill overwrote freshly uploaded instances).
template <typename P>
int dalloc(cimcs_ctx* c, P** p, size_t bytes) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 16));
    if (e != cudaSuccess)
        return fail(CIMCS_CUDA_ERROR, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    e = cudaMemsetAsync(*p, 0, std::max<size_t>(bytes, 16), c->stream);
    if (e != cudaSuccess)
        return fail(CIMCS_CUDA_ERROR, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
    return 0;
}

// Synchronous copy ordered on the context stream (all host <-> device traffic
// of a context goes through its stream; the host buffer may be reused on return).
int copy_sync(cimcs_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess)
        return fail(CIMCS_CUDA_ERROR, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
    return 0;
}

#define NK(x)                                                                           \
    do {                                                                                \
        ncclResult_t r_ = (x);                                                          \
        if (r_ != ncclSuccess)                                                          \
            return fail(CIMCS_CUDA_ERROR, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

// Super-rows [P0, P1) of rank `rank` of `world`: contiguous, balanced by the
// number of upper-triangle tiles (super-row P holds the items (P, Q >= P)).
void tile_shard(int nRB, int world, int rank, int* P0, int* P1) {
    const int nSB = (nRB + kSyS - 1) / kSyS;
    std::vector<long long> w(nSB, 0);
    for (int P = 0; P < nSB; ++P)
        for (int Q = P; Q < nSB; ++Q) {
            const int nI = std::min(kSyS, nRB - P * kSyS), nJ = std::min(kSyS, nRB - Q * kSyS);
            w[P] += P == Q ? nI * (nI + 1) / 2 : nI * nJ;
        }
    long long total = 0;
    for (long long x : w) total += x;
    std::vector<int> cut(world + 1, nSB);
    cut[0] = 0;
    long long acc = 0;
    int P = 0;
    for (int r = 1; r < world; ++r) {
        const long long target = total * r / world;
        while (P < nSB && acc + w[P] / 2 < target) acc += w[P++];
        cut[r] = P;
    }
    *P0 = cut[rank];
    *P1 = cut[rank + 1];
}

// Super-block items of nb instances placed on the persistent CTAs, largest
// first onto the least-loaded CTA (LPT); built once per nb and cached.
// LPT placement of weighted items on min(items, SMs) CTAs: flat item list + CTA ranges
int lpt_place(std::vector<std::pair<int, int2>>& items, int nsm, std::vector<int2>& flat,
              std::vector<int>& beg) {
    std::stable_sort(items.begin(), items.end(),
                     [](const auto& x, const auto& y) { return x.first > y.first; });
    const int grid = (int)std::max<size_t>(1, std::min<size_t>(items.size(), (size_t)nsm));
    std::vector<std::vector<int2>> per(grid);
    using L = std::pair<long long, int>;  // (load, cta)
    std::priority_queue<L, std::vector<L>, std::greater<L>> pq;
    for (int g = 0; g < grid; ++g) pq.push({0, g});
    for (const auto& it : items) {
        L l = pq.top();
        pq.pop();
        per[l.second].push_back(it.second);
        pq.push({l.first + it.first, l.second});
    }
    flat.clear();
    beg.assign(grid + 1, 0);
    for (int g = 0; g < grid; ++g) {
        // a CTA walks its items in instance order, so instance b's last item (and with the
        // fp64 path's item flags its update) finishes about b / B into the launch
        std::stable_sort(per[g].begin(), per[g].end(),
                         [](const int2& x, const int2& y) { return x.x < y.x; });
        beg[g] = (int)flat.size();
        flat.insert(flat.end(), per[g].begin(), per[g].end());
    }
    beg[grid] = (int)flat.size();
    return grid;
}

// LPT weight of an item in half-tiles: a tile on the diagonal (I == J) feeds one product
// instead of two and costs about half a tile (measured per CTA: 1.47 us per off-diagonal
// tile, 0.75 per I == J tile on the fp32 path, tools/sm_speed.py; half the DMMAs on the
// fp64 path), so a diagonal item of n x n blocks weighs n (n + 1) - n = n^2.
inline int sym_item_cost(bool diag, int nI, int nJ) { return diag ? nI * nI : 2 * nI * nJ; }

int sym_schedule(cimcs_ctx* c, int nb, const cimcs_ctx::SymSched** out, bool s64 = false) {
    if (s64 && c->cmp_active) {  // built per alternation by enqueue_refit_compact64
        *out = &c->cmp_sched;
        return 0;
    }
    const int kS = s64 ? kS6 : c->symS;  // item edge in tiles
    const int nRB = s64 ? c->nRB6 : c->nRB, nSB = s64 ? c->nSB6 : c->nSB;
    for (auto& q : c->ssched)
        if (q.nb == nb && q.nRB == nRB && q.S == kS) {
            *out = &q;
            return 0;
        }
    std::vector<std::pair<int, int2>> items;  // (tiles, item)
    const int P0 = c->tshard && !s64 ? c->sP0 : 0, P1 = c->tshard && !s64 ? c->sP1 : nSB;
    for (int b = 0; b < nb; ++b)
        for (int P = P0; P < P1; ++P)
            for (int Q = P; Q < nSB; ++Q) {
                const int nI = std::min(kS, nRB - P * kS), nJ = std::min(kS, nRB - Q * kS);
                items.push_back({sym_item_cost(P == Q, nI, nJ), make_int2(b, P << 16 | Q)});
            }
    std::vector<int2> flat;
    std::vector<int> beg;
    const int grid = lpt_place(items, c->sched_n(), flat, beg);
    cimcs_ctx::SymSched q;
    q.nb = nb;
    q.nRB = nRB;
    q.S = kS;
    q.grid = grid;
    int rc;
    if ((rc = dalloc(c, &q.items, flat.size() * sizeof(int2))) ||
        (rc = dalloc(c, &q.sched, beg.size() * sizeof(int))))
        return rc;
    if (int rc_ = copy_sync(c, q.items, flat.data(), flat.size() * sizeof(int2), cudaMemcpyHostToDevice)) return rc_;
    if (int rc_ = copy_sync(c, q.sched, beg.data(), beg.size() * sizeof(int), cudaMemcpyHostToDevice)) return rc_;
    c->ssched.push_back(q);
    *out = &c->ssched.back();
    return 0;
}


int ensure_stage(cimcs_ctx* c, size_t elems) {
    if (c->stage_elems >= elems) return 0;
    if (c->stage) cudaFree(c->stage);
    if (c->stage_i) cudaFree(c->stage_i);
    c->stage = nullptr;
    c->stage_i = nullptr;
    c->stage_elems = 0;
    if (int rc = dalloc(c, &c->stage, elems * 8)) return rc;
    if (int rc = dalloc(c, &c->stage_i, elems * 4)) return rc;
    c->stage_elems = elems;
    return 0;
}

int ensure_state(cimcs_ctx* c, int NR) {
    if (c->NR == NR && c->Rs) return 0;
    free_state(c);
    c->NR = NR;
    const size_t n = c->state_elems(), es = c->elt();
    const int nT = c->B * NR;
    const int nRB = std::max(std::max(c->nRB, c->nRB6), 1);
    int rc = 0;
    const size_t nw = c->w_elems();
    if ((rc = dalloc(c, &c->Rs, n * es)) || (rc = dalloc(c, &c->C, n * es)) ||
        (rc = dalloc(c, &c->E, n * es)) || (rc = dalloc(c, &c->W0, nw * es)) ||
        (rc = dalloc(c, &c->W1, nw * es)) || (rc = dalloc(c, &c->Hdbg, n * es)) ||
        (rc = dalloc(c, &c->bestR, n * es)) || (rc = dalloc(c, &c->sig, n)) ||
        (rc = dalloc(c, &c->bestS, n)) || (rc = dalloc(c, &c->fail_gstep, nT * 4)) ||
        (rc = dalloc(c, &c->fail_idx, nT * 4)) || (rc = dalloc(c, &c->n_hist, nT * 4)) ||
        (rc = dalloc(c, &c->improved, nT * 4)) || (rc = dalloc(c, &c->minE, nT * 8)) ||
        (rc = dalloc(c, &c->part, (size_t)c->B * nRB * NR * 4 * 8)) ||
        (rc = dalloc(c, &c->best_obj, nT * 8)) || (rc = dalloc(c, &c->obj, nT * 8)) ||
        (rc = dalloc(c, &c->rmse, nT * 8)) || (rc = dalloc(c, &c->ham, nT * 8)) ||
        (rc = dalloc(c, &c->tp, (size_t)nT * 5 * 8)) || (rc = dalloc(c, &c->fail_tmp, nT * 4)))
        return rc;
    if (c->sym64 && (rc = dalloc(c, &c->dDone, (size_t)2 * c->B * 4))) return rc;
    if (c->mri) {  // G w of the transform chain, one slot: [N][NR]
        const size_t ne = (size_t)c->nRB * kSyT * NR;
        if (c->spart_elems < ne) {
            if (c->dSpart) cudaFree(c->dSpart);
            c->dSpart = nullptr;
            c->spart_elems = 0;
            if ((rc = dalloc(c, &c->dSpart, ne * 4))) return rc;
            c->spart_elems = ne;
        }
    }
    if (c->sym64) {  // fp64 w tiles of W0/W1, the slot partials and the item schedule
        const size_t nw = (size_t)c->B * c->nRB6 * kT6 * NR;
        if ((rc = dalloc(c, &c->WT0, nw * 8)) || (rc = dalloc(c, &c->WT1, nw * 8)) ||
            (rc = dalloc(c, &c->dPart6, nw * c->nSB6 * 8)))
            return rc;
        const cimcs_ctx::SymSched* ss;
        if ((rc = sym_schedule(c, c->B, &ss, true))) return rc;
    }
    if (c->sym64 && c->cmp_opt) {  // the fp64 compacted refit's buffers
        const size_t nv = (size_t)c->B * c->ldN, ns = (size_t)c->B * cmp64::kMaxSeg;
        const int cap = c->B * c->nSB6 * (c->nSB6 + 1) / 2;
        if ((rc = dalloc(c, &c->cU, nv * 4)) || (rc = dalloc(c, &c->cCnt, (size_t)c->B * 4)) ||
            (rc = dalloc(c, &c->cMax, 16)) || (rc = dalloc(c, &c->cU6, nv * 4)) ||
            (rc = dalloc(c, &c->cSegc, ns * 4)) || (rc = dalloc(c, &c->cPfx, ns * 4)) ||
            (rc = dalloc(c, &c->cSegOff, cmp64::kMaxSeg * 4)) ||
            (rc = dalloc(c, &c->cSeg, cmp64::kMaxSeg * sizeof(int2))) ||
            (rc = dalloc(c, &c->Rc6, n * 8)) || (rc = dalloc(c, &c->sigc, n)) ||
            (rc = dalloc(c, &c->Dc6, nv * 8)) || (rc = dalloc(c, &c->hzc6, nv * 8)) ||
            (rc = dalloc(c, &c->cmp_sched.items, (size_t)cap * sizeof(int2))) ||
            (rc = dalloc(c, &c->cmp_sched.sched, (size_t)(c->num_sms + 1) * 4)))
            return rc;
        c->cmp_items_cap = cap;
        if (!c->Gc6 && (rc = dalloc(c, &c->Gc6, (size_t)c->B * c->ntri6 * kT6 * kT6 * 8)))
            return rc;
    }
    if (c->sym && !c->tshard && c->cmp_opt) {  // compacted refit buffers
        const size_t nv = (size_t)c->B * c->ldN;
        if ((rc = dalloc(c, &c->cU, nv * 4)) || (rc = dalloc(c, &c->cCnt, (size_t)c->B * 4)) ||
            (rc = dalloc(c, &c->cMax, 16)) || (rc = dalloc(c, &c->Rc, n * 4)) ||
            (rc = dalloc(c, &c->sigc, n)) || (rc = dalloc(c, &c->Dc, nv * 4)) ||
            (rc = dalloc(c, &c->hzc, nv * 4)))
            return rc;
        if (!c->Gc && (rc = dalloc(c, &c->Gc, (size_t)c->B * c->ntri * 2 * kSyPlaneBytes)))
            return rc;
    }
    if (c->sym) {  // fp16 B tiles of W0/W1 and the partial products of the symmetric kernel
        const size_t nb = (size_t)c->B * c->nRB * 2 * NR * kSyT, ns = (size_t)c->B * c->nRB * NR;
        if ((rc = dalloc(c, &c->WB0, nb * 2)) || (rc = dalloc(c, &c->WB1, nb * 2)) ||
            (rc = dalloc(c, &c->WS0, ns * 4)) || (rc = dalloc(c, &c->WS1, ns * 4)))
            return rc;
        // slots: nSB = ceil(nRB / 4); the compacted refit's 2 x 2 items need up to ceil(nRB / 2)
        const size_t nslot = c->cmp_opt && !c->tshard ? std::max(c->nSB, (c->nRB + 1) / 2) : c->nSB;
        const size_t ne = (size_t)c->B * c->nRB * nslot * kSyT * NR;
        // the item schedule (built outside graph capture)
        const cimcs_ctx::SymSched* ss;
        if ((rc = sym_schedule(c, c->B, &ss))) return rc;
        if (ne && c->spart_elems < ne) {
            if (c->dSpart) cudaFree(c->dSpart);
            c->dSpart = nullptr;
            c->spart_elems = 0;
            if ((rc = dalloc(c, &c->dSpart, ne * 4))) return rc;
            c->spart_elems = ne;
        }
        if (c->tshard) {  // slots of other ranks' items stay zero for good
            CK(cudaMemsetAsync(c->dSpart, 0, ne * 4, c->stream));
            if (c->dH) cudaFree(c->dH);
            c->dH = nullptr;
            if ((rc = dalloc(c, &c->dH, (size_t)c->B * c->nRB * kSyT * NR * 4))) return rc;
        }
    }
    return 0;
}

StepScalars make_scalars(const cimcs_hyper* hp) {
    StepScalars s{};
    s.dt = hp->dt;
    s.rt = std::sqrt(hp->tau);
    s.half_rt = s.rt / 2.0;
    s.tau = hp->tau;
    s.nbeta = -hp->beta;
    s.Kj = hp->K * hp->j;
    s.minus_j = hp->mfz_loss_minus_j ? hp->j : 0.0;
    s.one_minus_dtc = 1.0 - hp->dt_c;
    s.dt_c = hp->dt_c;
    s.g2 = hp->g2;
    s.j = hp->j;
    s.pp_scale = std::sqrt(hp->g2 / (4.0 * hp->j * hp->dt));  // solver_pp.cpp:27
    s.pp_sdt = std::sqrt(hp->dt);
    s.pp_sjg = std::sqrt(hp->j * hp->g2);
    s.pp_m2j = -2.0 * (1.0 + hp->j);
    s.mu_abort = hp->mu_abort;
    s.n_steps = hp->n_steps;
    return s;
}

AltParams make_alt(const cimcs_hyper* hp, double eta, int alt) {
    AltParams a{};
    const double rt = std::sqrt(hp->tau);
    a.thresh = eta * eta / 4.0 * rt;  // solver_mfz.cpp:69
    a.thresh_pp = rt * eta * eta / 4.0;  // solver_pp.cpp:59
    a.lambda = eta * eta / 2.0;       // orchestrator.cpp:189
    a.eta = eta;
    a.alt = alt;
    a.gstep_base = alt * hp->n_steps;
    return a;
}

double eta_schedule(int i, double eta_init, double eta_end, int velo) {
    const double linear = eta_init * (1.0 - static_cast<double>(i) / velo);
    return std::max(linear, eta_end);
}

std::vector<double> pump_table(const cimcs_hyper* hp) {
    std::vector<double> p(hp->n_steps);
    double t = 0.0;
    const double T = static_cast<double>(hp->n_steps) * hp->dt;
    for (int k = 0; k < hp->n_steps; ++k) {
        p[k] = hp->pump_kind == CIMCS_PUMP_LINEAR
                   ? hp->pump_end * t / T
                   : (hp->p_thr - hp->d) + 2.0 * hp->d / (1.0 + std::exp(-(t - 4.0) / 2.0));
        t = t + hp->dt;
    }
    return p;
}

}  // namespace
