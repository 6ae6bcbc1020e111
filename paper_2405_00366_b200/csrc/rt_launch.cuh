// rt_launch.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): kernel launchers: CUDA-core, tcgen05 symmetric (fp32), DMMA symmetric
// (fp64), matrix-free MRI, cluster loop; state uploads; NCCL exchanges.
#pragma once

namespace {

// ----------------------------------------------------- typed dispatch
template <typename T, int NR, int MODE>
int launch_gemv_t(cimcs_ctx* c, const GemvArgs& a) {
    auto kern = gemv_fused_kernel<T, NR, MODE>;
    constexpr size_t smem = gemv_smem_bytes<T, NR>();
    static std::atomic<unsigned long long> attr{0};  // per device: the attribute is per context
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr.fetch_or(1ull << c->device);
    }
    if (c->nRB == 0) return 0;  // this rank holds no rows
    dim3 grid(c->nRB, c->B);
    kern<<<grid, kThreads, smem, c->stream>>>(a);
    CK(cudaGetLastError());
    return 0;
}

template <typename T, int NR>
int launch_gemv_nr(cimcs_ctx* c, int mode, const GemvArgs& a) {
    switch (mode) {
        case EPI_STEP_BN: return launch_gemv_t<T, NR, EPI_STEP_BN>(c, a);
        case EPI_STEP_CN: return launch_gemv_t<T, NR, EPI_STEP_CN>(c, a);
        case EPI_JACOBI: return launch_gemv_t<T, NR, EPI_JACOBI>(c, a);
        case EPI_MATVEC: return launch_gemv_t<T, NR, EPI_MATVEC>(c, a);
        case EPI_STEP_PP: return launch_gemv_t<T, NR, EPI_STEP_PP>(c, a);
        default: return launch_gemv_t<T, NR, EPI_SCORE>(c, a);
    }
}

template <typename T>
int launch_gemv_T(cimcs_ctx* c, int mode, const GemvArgs& a) {
    switch (c->NR) {
        case 1: return launch_gemv_nr<T, 1>(c, mode, a);
        case 2: return launch_gemv_nr<T, 2>(c, mode, a);
        case 4: return launch_gemv_nr<T, 4>(c, mode, a);
        case 8: return launch_gemv_nr<T, 8>(c, mode, a);
        default: return launch_gemv_nr<T, 16>(c, mode, a);
    }
}

TcArgs tc_args(const cimcs_ctx* c, const GemvArgs& g) {
    TcArgs a{};
    a.D = g.D;
    a.hz = g.hz;
    a.Win = g.Win;
    a.Wout = g.Wout;
    a.Rs = g.Rs;
    a.C = g.C;
    a.E = g.E;
    a.Hdbg = g.Hdbg;
    a.Mv = g.Mv;
    a.Pn = g.Pn;
    a.Pm = g.Pm;
    a.MT = g.MT;
    a.nz = g.nz;
    a.nz_next = g.nz_next;
    a.sigma = g.sigma;
    a.fail_gstep = g.fail_gstep;
    a.fail_idx = g.fail_idx;
    a.minE = g.minE;
    a.part = g.part;
    a.pump = g.pump;
    a.alt = g.alt;
    a.xtrue = g.xtrue;
    a.xitrue = g.xitrue;
    a.err = g.err;
    a.p_scalar = g.p_scalar;
    a.step = g.step;
    a.N = c->N;
    a.ldN = c->ldN;
    a.ldJ = c->ldJ;
    a.B = c->B;
    a.nRB = c->nRB;
    a.nch = c->nch;
    a.ntiles = c->B * c->nRB;
    a.rb0 = c->rb0;
    a.s = g.s;
    return a;
}




// symmetric-tile variant (sym_kernels.cuh): half the gram bytes per step.
// The tile kernel, then the slot reduction and the fused update, on the
// context stream (instances [b0, b0 + nb)).
template <int NR, int MODE>
int launch_sym_t(cimcs_ctx* c, const GemvArgs& g, int b0, int nb) {
    cudaStream_t sA = c->stream, sF = c->stream;
    SymArgs sa{};
    sa.t = tc_args(c, g);
    sa.Gs = static_cast<const __half*>(c->dG);
    sa.sg = c->dSg;
    sa.WBin = g.Win == c->W0 ? c->WB0 : c->WB1;
    sa.WSin = g.Win == c->W0 ? c->WS0 : c->WS1;
    sa.WBout = g.Wout == c->W0 ? c->WB0 : c->WB1;
    sa.WSout = g.Wout == c->W0 ? c->WS0 : c->WS1;
    sa.spart = c->dSpart;
    sa.ntri = c->ntri;
    sa.nSB = c->nSB;
    sa.b0 = b0;
    sa.gram_keep = c->gram_l2;
    sa.S = c->symS;
    sa.rowmap = c->cmp_active ? c->cU : nullptr;
    sa.tlog = c->dTl && (size_t)c->B * c->nRB <= (size_t)(kTlTile - kTlUpd) ? c->dTl : nullptr;
    if (nb == 0 || c->ntri == 0) return 0;
    const cimcs_ctx::SymSched* ss = nullptr;
    if (int rc = sym_schedule(c, nb, &ss)) return rc;
    sa.items = ss->items;
    sa.sched = ss->sched;
    auto kern = sym_step_kernel<NR, MODE>;
    constexpr size_t smem = sy_smem_bytes<NR>();
    static std::atomic<unsigned long long> attr{0};  // per device: the attribute is per context
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr.fetch_or(1ull << c->device);
    }
    // same stream: both kernels use programmatic dependent launch (the next
    // kernel's prologue overlaps this one's tail; griddepcontrol.wait orders data)
    const bool pdl = sF == sA && c->use_pdl && !c->tshard;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ss->grid);
    cfg.blockDim = dim3(kSyThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = sA;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    const bool timed = c->kernel_timing && (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) &&
                       cudaStreamIsCapturing(sA, &cap) == cudaSuccess &&
                       cap == cudaStreamCaptureStatusNone;
    if (timed) {
        if (!c->kt_ev[0]) {
            CK(cudaEventCreate(&c->kt_ev[0]));
            CK(cudaEventCreate(&c->kt_ev[1]));
        }
        CK(cudaEventRecord(c->kt_ev[0], sA));
    }
    CK(cudaLaunchKernelEx(&cfg, kern, sa));
    if (timed) {  // the kernel alone, on its own stream (serialises the step: a measurement mode)
        CK(cudaEventRecord(c->kt_ev[1], sA));
        CK(cudaEventSynchronize(c->kt_ev[1]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->kt_ev[0], c->kt_ev[1]));
        c->timing.tile_kernel_ms += ms;
        c->timing.tile_kernel_launches += 1;
    }
    if (c->tshard) {  // own items' slot sums, then the cross-rank sum (one collective)
        sym_slotsum_kernel<NR><<<dim3(c->nRB, nb), kSyT * NR / 4, 0, sF>>>(c->dSpart, c->dH, c->nRB,
                                                                         c->nSB, b0);
        CK(cudaGetLastError());
        if (c->tworld > 1) {
            const size_t per = (size_t)c->nRB * kSyT * NR;
            NK(ncclAllReduce(c->dH + (size_t)b0 * per, c->dH + (size_t)b0 * per, (size_t)nb * per,
                             ncclFloat32, ncclSum, c->comm, sF));
        }
        sa.spart = c->dH;
        sa.nSB = 1;
    }
    cfg.gridDim = dim3(c->nRB, nb);
    cfg.blockDim = dim3(kSyT * NR / 4);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = sF;
    CK(cudaLaunchKernelEx(&cfg, sym_update_kernel<NR, MODE, float>, sa));
    return 0;
}

template <int NR>
int launch_sym_grp(cimcs_ctx* c, int mode, const GemvArgs& a, int b0, int nb) {
    switch (mode) {
        case EPI_STEP_BN: return launch_sym_t<NR, EPI_STEP_BN>(c, a, b0, nb);
        case EPI_STEP_CN: return launch_sym_t<NR, EPI_STEP_CN>(c, a, b0, nb);
        case EPI_JACOBI: return launch_sym_t<NR, EPI_JACOBI>(c, a, b0, nb);
        case EPI_MATVEC: return launch_sym_t<NR, EPI_MATVEC>(c, a, b0, nb);
        case EPI_STEP_PP: return launch_sym_t<NR, EPI_STEP_PP>(c, a, b0, nb);
        default: return launch_sym_t<NR, EPI_SCORE>(c, a, b0, nb);
    }
}


template <int NR>
int launch_sym_nr(cimcs_ctx* c, int mode, const GemvArgs& a) {
    return launch_sym_grp<NR>(c, mode, a, 0, c->B);
}


// fp64 symmetric-tile path (sym64_kernels.cuh): the DMMA tile kernel, then the
// fused fp64 update, both on the context stream with PDL between them.
template <int NR, int MODE, int NC>
int launch_sym64_t(cimcs_ctx* c, const GemvArgs& g) {
    Sym64Args sa{};
    sa.t = tc_args(c, g);
    sa.t.nRB = c->nRB6;
    sa.Gt = static_cast<const double*>(c->dG6);
    sa.WTin = g.Win == c->W0 ? c->WT0 : c->WT1;
    sa.WTout = g.Wout == c->W0 ? c->WT0 : (g.Wout == c->W1 ? c->WT1 : nullptr);
    sa.part = c->dPart6;
    sa.ntri = c->ntri6;
    sa.nSB = c->nSB6;
    sa.seg = c->cmp_active ? c->cSeg : nullptr;  // compacted refit: variable segments
    sa.rowmap = c->cmp_active ? c->cU6 : nullptr;
    sa.tlog = c->dTl && (size_t)2 * c->B * c->nRB6 <= (size_t)(kTlTile - kTlUpd) ? c->dTl : nullptr;
    if (c->overlap_upd && c->dDone) {  // item flags (sym64_kernels.cuh)
        sa.done = c->dDone;
        sa.taken = c->dDone + c->B;
        sa.ipi = (unsigned)(c->nSB6 * (c->nSB6 + 1) / 2);
    }
    const cimcs_ctx::SymSched* ss = nullptr;
    if (int rc = sym_schedule(c, c->B, &ss, true)) return rc;
    sa.items = ss->items;
    sa.sched = ss->sched;
    auto kern = sym64_step_kernel<NR, MODE, NC>;
    constexpr size_t smem = s6_smem_bytes<NR>();
    static std::atomic<unsigned long long> attr{0};
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // Both kernels ask for the largest shared-memory carveout (228 KB), not the smallest
        // that fits (an SM runs CTAs of one L1 / shared split at a time): with the defaults no
        // update CTA became resident before its SM's tile CTA had exited (timeline, DESIGN 4).
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared));
        constexpr int kRowsU = (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) && NR == 16 ? kT6 / 2 : kT6;
        CK(cudaFuncSetAttribute((sym64_update_kernel<NR, MODE, kRowsU>),
                                cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared));
        attr.fetch_or(1ull << c->device);
    }
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ss->grid);
    cfg.blockDim = dim3((NC + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cfg.attrs = at;
    cfg.numAttrs = c->use_pdl ? 1 : 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    const bool timed = c->kernel_timing && (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) &&
                       cudaStreamIsCapturing(c->stream, &cap) == cudaSuccess &&
                       cap == cudaStreamCaptureStatusNone;
    if (timed) {
        if (!c->kt_ev[0]) {
            CK(cudaEventCreate(&c->kt_ev[0]));
            CK(cudaEventCreate(&c->kt_ev[1]));
        }
        CK(cudaEventRecord(c->kt_ev[0], c->stream));
    }
    CK(cudaLaunchKernelEx(&cfg, kern, sa));
    if (timed) {
        CK(cudaEventRecord(c->kt_ev[1], c->stream));
        CK(cudaEventSynchronize(c->kt_ev[1]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->kt_ev[0], c->kt_ev[1]));
        c->timing.tile_kernel_ms += ms;
        c->timing.tile_kernel_launches += 1;
    }
    // step modes: 32-row CTAs (4 warps), the size that fits beside a resident tile CTA
    constexpr int kRows = (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) && NR == 16 ? kT6 / 2 : kT6;
    cfg.gridDim = dim3(c->nRB6 * (kT6 / kRows), c->B);
    cfg.blockDim = dim3(kRows * NR / 4);
    cfg.dynamicSmemBytes = 0;
    CK(cudaLaunchKernelEx(&cfg, (sym64_update_kernel<NR, MODE, kRows>), sa));
    return 0;
}

template <int NR, int NC>
int launch_sym64_nc(cimcs_ctx* c, int mode, const GemvArgs& a) {
    switch (mode) {
        case EPI_STEP_BN: return launch_sym64_t<NR, EPI_STEP_BN, NC>(c, a);
        case EPI_STEP_CN: return launch_sym64_t<NR, EPI_STEP_CN, NC>(c, a);
        case EPI_JACOBI: return launch_sym64_t<NR, EPI_JACOBI, NC>(c, a);
        case EPI_MATVEC: return launch_sym64_t<NR, EPI_MATVEC, NC>(c, a);
        case EPI_STEP_PP: return launch_sym64_t<NR, EPI_STEP_PP, NC>(c, a);
        default: return launch_sym64_t<NR, EPI_SCORE, NC>(c, a);
    }
}

// 8 DMMA warps (4 per use): 16 warps measured slower (297 vs 291 us at config 1,
// bitwise-equal results)
template <int NR>
int launch_sym64_nr(cimcs_ctx* c, int mode, const GemvArgs& a) {
    return launch_sym64_nc<NR, 8>(c, mode, a);
}

// one mri_kernel launch of `grid` CTAs (basis vectors r0.. for DIAG / COLS)
int mri_launch(cimcs_ctx* c, int mode, int grid, int r0, const float* in, float* out) {
    MriArgs ma{};
    ma.H = c->mH;
    ma.W = c->mW;
    ma.N = c->N;
    ma.NR = 1;
    ma.mask_br = c->dMaskBr;
    ma.tw = c->dTw;
    ma.L = c->mL;
    ma.gamma = c->mgamma;
    ma.scale = 1.f / (float)c->N;
    ma.in = in;
    ma.out = out;
    ma.r0 = r0;
    mri_kernel<<<grid, kMriThreads, mri_smem_bytes(c->mH, c->mW, c->mL), c->stream>>>(ma, mode);
    CK(cudaGetLastError());
    return 0;
}

// one dct_cluster_kernel launch: `count` vectors (replica slots for APPLY,
// basis vectors r0.. for DIAG / COLS, 1 for HZ), a cluster of 8 CTAs each
int dct_launch(cimcs_ctx* c, int mode, int count, int r0, const float* in, float* out, int NR) {
    DctArgs da{};
    da.NR = NR;
    da.C = c->dDctC;
    da.mask = c->dDctMask;
    da.in = in;
    da.out = out;
    da.r0 = r0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(count * kDctCS);
    cfg.blockDim = dim3(kDctThreads);
    cfg.dynamicSmemBytes = dct_smem_bytes();
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kDctCS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = mode == DCT_APPLY && c->use_pdl ? 2 : 1;
    switch (c->dct_L) {
        case 1: CK(cudaLaunchKernelEx(&cfg, dct_cluster_kernel<1>, da, mode)); break;
        case 2: CK(cudaLaunchKernelEx(&cfg, dct_cluster_kernel<2>, da, mode)); break;
        default: CK(cudaLaunchKernelEx(&cfg, dct_cluster_kernel<3>, da, mode)); break;
    }
    CK(cudaGetLastError());
    return 0;
}

// transform-chain problems: G w by the matrix-free MRI kernel (one CTA per
// replica slot) into the one-slot partial buffer, then the symmetric path's
// update kernel for the fused epilogue of `mode`
template <int NR, int MODE>
int launch_mri_t(cimcs_ctx* c, const GemvArgs& g) {
    MriArgs ma{};
    ma.H = c->mH;
    ma.W = c->mW;
    ma.N = c->N;
    ma.NR = NR;
    ma.mask_br = c->dMaskBr;
    ma.tw = c->dTw;
    ma.L = c->mL;
    ma.gamma = c->mgamma;
    ma.scale = 1.f / (float)c->N;
    ma.in = static_cast<const float*>(g.Win);
    ma.out = c->dSpart;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    const bool timed = c->kernel_timing && (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) &&
                       cudaStreamIsCapturing(c->stream, &cap) == cudaSuccess &&
                       cap == cudaStreamCaptureStatusNone;
    if (timed) {  // eager mode: CUDA events around the chain kernel
        if (!c->kt_ev[0]) {
            CK(cudaEventCreate(&c->kt_ev[0]));
            CK(cudaEventCreate(&c->kt_ev[1]));
        }
        CK(cudaEventRecord(c->kt_ev[0], c->stream));
    }
    if (c->mri_kind == 1) {
        if (int rc = dct_launch(c, DCT_APPLY, NR, 0, ma.in, ma.out, NR)) return rc;
    } else if (c->mri_cluster && std::min(c->mH, c->mW) >= 2 * kMriCluster) {
        // one thread-block cluster per replica (mri_cluster_kernel)
        const int CS = mri_cluster_size(c->mH, c->mW);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(NR * CS);
        cfg.blockDim = dim3(kMriCThreads);
        cfg.dynamicSmemBytes = mri_cluster_smem_bytes(c->mH, c->mW);
        cfg.stream = c->stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = c->use_pdl ? 2 : 1;
        CK(cudaLaunchKernelEx(&cfg, mri_cluster_kernel, ma));
    } else {
        const size_t smem = mri_smem_bytes(c->mH, c->mW, c->mL);
        mri_kernel<<<NR, kMriThreads, smem, c->stream>>>(ma, MRI_APPLY);
    }
    CK(cudaGetLastError());
    if (timed) {
        CK(cudaEventRecord(c->kt_ev[1], c->stream));
        CK(cudaEventSynchronize(c->kt_ev[1]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->kt_ev[0], c->kt_ev[1]));
        c->timing.tile_kernel_ms += ms;
        c->timing.tile_kernel_launches += 1;
    }
    SymArgs sa{};
    sa.t = tc_args(c, g);
    sa.spart = c->dSpart;
    sa.nSB = 1;
    sa.b0 = 0;
    sa.keep_w = 1;  // the next apply reads the fp32 w
    sa.S = kSyS;
    {
        cudaLaunchConfig_t ucfg{};
        ucfg.gridDim = dim3(c->nRB, 1);
        ucfg.blockDim = dim3(kSyT * NR / 4);
        ucfg.stream = c->stream;
        cudaLaunchAttribute ua[1];
        ua[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        ua[0].val.programmaticStreamSerializationAllowed = 1;
        ucfg.attrs = ua;
        ucfg.numAttrs = c->use_pdl ? 1 : 0;
        CK(cudaLaunchKernelEx(&ucfg, sym_update_kernel<NR, MODE>, sa));
    }
    CK(cudaGetLastError());
    return 0;
}

template <int NR>
int launch_mri_nr(cimcs_ctx* c, int mode, const GemvArgs& a) {
    switch (mode) {
        case EPI_STEP_BN: return launch_mri_t<NR, EPI_STEP_BN>(c, a);
        case EPI_STEP_CN: return launch_mri_t<NR, EPI_STEP_CN>(c, a);
        case EPI_MATVEC: return launch_mri_t<NR, EPI_MATVEC>(c, a);
        case EPI_SCORE: return launch_mri_t<NR, EPI_SCORE>(c, a);
        case EPI_JACOBI:
            if (c->mri_kind == 1) return launch_mri_t<NR, EPI_JACOBI>(c, a);
            [[fallthrough]];
        default: return fail(CIMCS_CONFIG_ERROR, "cdp_minimize_operator: damped Jacobi needs an assembled matrix");
    }
}

int launch_gemv(cimcs_ctx* c, int mode, const GemvArgs& a) {
    if (c->mri) return c->NR == 8 ? launch_mri_nr<8>(c, mode, a) : launch_mri_nr<16>(c, mode, a);
    if (c->sym64)
        return c->NR == 8 ? launch_sym64_nr<8>(c, mode, a) : launch_sym64_nr<16>(c, mode, a);
    if (c->sym) return c->NR == 8 ? launch_sym_nr<8>(c, mode, a) : launch_sym_nr<16>(c, mode, a);
    return c->st64() ? launch_gemv_T<double>(c, mode, a)
                                 : launch_gemv_T<float>(c, mode, a);
}

#define DISPATCH_NR_TC(NRV, ...)                                            \
    if ((NRV) == 8) { constexpr int NR_ = 8; __VA_ARGS__; }                 \
    else { constexpr int NR_ = 16; __VA_ARGS__; }

// symmetric path: refresh the fp16 B tiles of W (W0 or W1) after a writer
// other than the symmetric kernel itself
int sym_sync_w(cimcs_ctx* c, const void* W) {
    const bool w0 = W == c->W0;
    const dim3 g(c->nRB, c->B);
    if (c->sym64) {
        DISPATCH_NR_TC(c->NR, {
            sym64_wconvert_kernel<NR_><<<dim3(c->nRB6, c->B), 256, 0, c->stream>>>(
                static_cast<const double*>(W), c->N, c->ldN, c->nRB6, w0 ? c->WT0 : c->WT1);
        });
        CK(cudaGetLastError());
    }
    if (!c->sym) return 0;
    DISPATCH_NR_TC(c->NR, {
        sym_wconvert_kernel<NR_, float><<<g, 128, 0, c->stream>>>(
            static_cast<const float*>(W), c->N, c->ldN, c->nRB, w0 ? c->WB0 : c->WB1,
            w0 ? c->WS0 : c->WS1);
    });
    CK(cudaGetLastError());
    return 0;
}

// replica slots: a power of two; the tensor-core path needs MMA N in {8, 16}
int slots_for(const cimcs_ctx* c, int R) {
    const int p = pow2_slots(R);
    return c->tc || c->mri || c->sym64 ? std::max(8, p) : p;
}

// Generic NR/T dispatch for the small state kernels.
#define DISPATCH_NR(NRV, ...)                                               \
    switch (NRV) {                                                          \
        case 1: { constexpr int NR_ = 1; __VA_ARGS__; } break;              \
        case 2: { constexpr int NR_ = 2; __VA_ARGS__; } break;              \
        case 4: { constexpr int NR_ = 4; __VA_ARGS__; } break;              \
        case 8: { constexpr int NR_ = 8; __VA_ARGS__; } break;              \
        default: { constexpr int NR_ = 16; __VA_ARGS__; } break;            \
    }

template <typename T>
int run_init_T(cimcs_ctx* c, int Rreal, int bn, const double* dc0, const double* de0, double rt) {
    const int g = grid_for(c->state_elems());
    T* W = static_cast<T*>(c->W0);
    DISPATCH_NR(c->NR, {
        if (bn)
            init_state_kernel<T, NR_, 1><<<g, 256, 0, c->stream>>>(
                dc0, Rreal, c->N, c->ldN, c->B, static_cast<const T*>(c->Rs),
                static_cast<T*>(c->C), static_cast<T*>(c->E), W, c->fail_gstep, c->minE, rt,
                de0, wcanon(c), c->ldJ);
        else
            init_state_kernel<T, NR_, 0><<<g, 256, 0, c->stream>>>(
                dc0, Rreal, c->N, c->ldN, c->B, static_cast<const T*>(c->Rs),
                static_cast<T*>(c->C), static_cast<T*>(c->E), W, c->fail_gstep, c->minE, rt,
                de0, wcanon(c), c->ldJ);
    });
    CK(cudaGetLastError());
    return sym_sync_w(c, c->W0);
}

int run_init(cimcs_ctx* c, int Rreal, int bn, const double* dc0, const double* de0, double rt) {
    return c->st64() ? run_init_T<double>(c, Rreal, bn, dc0, de0, rt)
                                 : run_init_T<float>(c, Rreal, bn, dc0, de0, rt);
}

template <typename T>
int run_support_T(cimcs_ctx* c) {
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        support_kernel<T, NR_><<<g, 256, 0, c->stream>>>(
            static_cast<const T*>(c->C), static_cast<const T*>(c->Rs), c->sig,
            static_cast<T*>(c->W0), c->fail_gstep, c->N, c->ldN, c->B, wcanon(c), c->ldJ);
    });
    CK(cudaGetLastError());
    return sym_sync_w(c, c->W0);
}

int run_support(cimcs_ctx* c) {
    return c->st64() ? run_support_T<double>(c) : run_support_T<float>(c);
}

template <typename T>
int upload_traj_T(cimcs_ctx* c, const double* h, void* d, int Rreal, T pad) {
    const size_t n = (size_t)c->B * Rreal * c->N;
    if (int rc = ensure_stage(c, std::max(n, c->state_elems()))) return rc;
    CK(cudaMemcpyAsync(c->stage, h, n * 8, cudaMemcpyHostToDevice, c->stream));
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        traj_to_dev<T, NR_><<<g, 256, 0, c->stream>>>(c->stage, static_cast<T*>(d), Rreal, c->N,
                                                      c->ldN, c->B, pad);
    });
    CK(cudaGetLastError());
    return 0;
}

int upload_traj(cimcs_ctx* c, const double* h, void* d, int Rreal, double pad = 0.0) {
    return c->st64() ? upload_traj_T<double>(c, h, d, Rreal, pad)
                                 : upload_traj_T<float>(c, h, d, Rreal, (float)pad);
}

template <typename T>
int download_traj_T(cimcs_ctx* c, const void* d, double* h, int Rreal) {
    const size_t n = (size_t)c->B * Rreal * c->N;
    if (int rc = ensure_stage(c, std::max(n, c->state_elems()))) return rc;
    const int g = grid_for(n);
    DISPATCH_NR(c->NR, {
        dev_to_traj<T, NR_><<<g, 256, 0, c->stream>>>(static_cast<const T*>(d), c->stage, Rreal,
                                                      c->N, c->ldN, c->B);
    });
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, c->stage, n * 8, cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

int download_traj(cimcs_ctx* c, const void* d, double* h, int Rreal) {
    return c->st64() ? download_traj_T<double>(c, d, h, Rreal)
                                 : download_traj_T<float>(c, d, h, Rreal);
}

int upload_sig(cimcs_ctx* c, const int32_t* h, int8_t* d, int Rreal) {
    const size_t n = (size_t)c->B * Rreal * c->N;
    if (int rc = ensure_stage(c, std::max(n, c->state_elems()))) return rc;
    for (size_t k = 0; k < n; ++k)
        if (h[k] != 0 && h[k] != 1) return fail(CIMCS_INPUT_ERROR, "sigma must be 0/1");
    CK(cudaMemcpyAsync(c->stage_i, h, n * 4, cudaMemcpyHostToDevice, c->stream));
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        sig_to_dev<NR_><<<g, 256, 0, c->stream>>>(c->stage_i, d, Rreal, c->N, c->ldN, c->B);
    });
    CK(cudaGetLastError());
    return 0;
}

int download_sig(cimcs_ctx* c, const int8_t* d, int32_t* h, int Rreal) {
    const size_t n = (size_t)c->B * Rreal * c->N;
    if (int rc = ensure_stage(c, std::max(n, c->state_elems()))) return rc;
    const int g = grid_for(n);
    DISPATCH_NR(c->NR, {
        sig_to_traj<NR_><<<g, 256, 0, c->stream>>>(d, c->stage_i, Rreal, c->N, c->ldN, c->B);
    });
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, c->stage_i, n * 4, cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

template <typename T>
int rinit_hz_T(cimcs_ctx* c, int Rreal) {
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        rinit_hz_kernel<T, NR_><<<g, 256, 0, c->stream>>>(static_cast<const T*>(c->dhz),
                                                          static_cast<T*>(c->Rs), Rreal, c->N,
                                                          c->ldN, c->B);
    });
    CK(cudaGetLastError());
    return 0;
}

template <typename T>
int mask_T(cimcs_ctx* c, void* V) {
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        mask_kernel<T, NR_><<<g, 256, 0, c->stream>>>(static_cast<const T*>(c->Rs), c->sig,
                                                      static_cast<T*>(V), c->state_elems(), c->N,
                                                      c->ldN, c->ldJ, wcanon(c));
    });
    CK(cudaGetLastError());
    return sym_sync_w(c, V);
}

int reset_flags(cimcs_ctx* c, int Rreal) {
    const int nT = c->B * c->NR;
    traj_flags_kernel<<<(nT + 255) / 256, 256, 0, c->stream>>>(c->fail_gstep, c->fail_idx, Rreal,
                                                              c->NR, c->B);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(c->n_hist, 0, nT * 4, c->stream));
    CK(cudaMemsetAsync(c->err, 0x7f, 4, c->stream));
    return 0;
}

GemvArgs base_args(cimcs_ctx* c, const StepScalars& s) {
    GemvArgs a{};
    a.G = c->G();
    a.D = c->dD;
    a.hz = c->dhz;
    a.Rs = c->Rs;
    a.C = c->C;
    a.E = c->E;
    a.sigma = c->sig;
    a.fail_gstep = c->fail_gstep;
    a.fail_idx = c->fail_idx;
    a.minE = c->minE;
    a.part = c->part;
    a.alt = c->alt;
    a.xtrue = c->has_truth ? c->dx : nullptr;
    a.xitrue = c->dxi;
    a.err = c->err;
    a.N = c->N;
    a.ldN = c->ldN;
    a.ldJ = c->ldJ;
    a.B = c->B;
    a.rb0 = c->rb0;
    a.s = s;
    return a;
}

// row blocks of the score partials: the contraction that scores (sym64 if present)
int nRB_of(const cimcs_ctx* c) { return c->sym64 ? c->nRB6 : c->nRB; }

// ------------------------------------------------ row-sharding collectives

ncclDataType_t nccl_t(const cimcs_ctx* c) {
    return c->st64() ? ncclFloat64 : ncclFloat32;
}

// All-gather this rank's rows of a per-instance array X[b][rows][row_elems]
// (rows padded to world * per): in place, one call per instance, grouped.
int allgather_rows(cimcs_ctx* c, void* X, size_t row_elems, size_t inst_elems,
                   ncclDataType_t t, size_t esize) {
    if (c->world == 1) return 0;
    const size_t per = (size_t)(c->ldN / c->world);
    NK(ncclGroupStart());
    for (int b = 0; b < c->B; ++b) {
        char* base = static_cast<char*>(X) + (size_t)b * inst_elems * esize;
        NK(ncclAllGather(base + (size_t)c->rank * per * row_elems * esize, base, per * row_elems, t,
                         c->comm, c->stream));
    }
    NK(ncclGroupEnd());
    return 0;
}

// contraction input (w or the refit's V)
int allgather_w(cimcs_ctx* c, void* W) {
    return allgather_rows(c, W, c->NR, (size_t)c->ldN * c->NR, nccl_t(c), c->elt());
}
int allgather_state(cimcs_ctx* c, void* X) {
    return allgather_rows(c, X, c->NR, (size_t)c->ldN * c->NR, nccl_t(c), c->elt());
}
int allgather_sig(cimcs_ctx* c, int8_t* S) {
    return allgather_rows(c, S, c->NR, (size_t)c->ldN * c->NR, ncclInt8, 1);
}

// After a CIM call: agree on divergence (first step, then first spin of that
// step) and on min_e across ranks.
int reconcile_cim(cimcs_ctx* c) {
    if (c->world == 1) return 0;
    const int nT = c->B * c->NR;
    CK(cudaMemcpyAsync(c->fail_tmp, c->fail_gstep, nT * 4, cudaMemcpyDeviceToDevice, c->stream));
    NK(ncclAllReduce(c->fail_gstep, c->fail_gstep, nT, ncclInt32, ncclMin, c->comm, c->stream));
    fail_fix_kernel<<<(nT + 255) / 256, 256, 0, c->stream>>>(c->fail_tmp, c->fail_gstep,
                                                             c->fail_idx, nT);
    CK(cudaGetLastError());
    NK(ncclAllReduce(c->fail_idx, c->fail_idx, nT, ncclInt32, ncclMin, c->comm, c->stream));
    NK(ncclAllReduce(c->minE, c->minE, nT, ncclUint64, ncclMin, c->comm, c->stream));
    return 0;
}

// Enqueue the n_steps fused Euler steps of one CIM call (graph-capturable).
// ------------------------------------------ small-N cluster loop (N <= 512)
// Replica slots the register-resident G slice leaves room for.
int cluster_max_nr(const cimcs_ctx* c) { return c->st64() ? 4 : 8; }

bool cluster_ok(const cimcs_ctx* c) {
    return c->use_cluster && !c->mri && c->world == 1 && !c->sharded && c->N <= kClMaxN &&
           c->NR <= cluster_max_nr(c);
}

template <typename T, int NR, int MODE>
int launch_cluster_t(cimcs_ctx* c, GemvArgs a, int n_iters) {
    auto kern = cluster_loop_kernel<T, NR, MODE>;
    constexpr size_t smem = cluster_smem_bytes<T, NR>();
    static std::atomic<unsigned long long> attr{0};  // per device: the attribute is per context
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr.fetch_or(1ull << c->device);
    }
    const unsigned cs = (unsigned)((c->N + kClRows - 1) / kClRows);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c->B * cs);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, a, c->nRB, c->nch, n_iters));
    return 0;
}

template <typename T, int NR>
int launch_cluster_nr(cimcs_ctx* c, int mode, const GemvArgs& a, int n_iters) {
    switch (mode) {
        case EPI_STEP_BN: return launch_cluster_t<T, NR, EPI_STEP_BN>(c, a, n_iters);
        case EPI_STEP_CN: return launch_cluster_t<T, NR, EPI_STEP_CN>(c, a, n_iters);
        default: return launch_cluster_t<T, NR, EPI_JACOBI>(c, a, n_iters);
    }
}

template <typename T>
int launch_cluster_T(cimcs_ctx* c, int mode, const GemvArgs& a, int n_iters) {
    switch (c->NR) {
        case 1: return launch_cluster_nr<T, 1>(c, mode, a, n_iters);
        case 2: return launch_cluster_nr<T, 2>(c, mode, a, n_iters);
        case 4: return launch_cluster_nr<T, 4>(c, mode, a, n_iters);
        default:
            if constexpr (sizeof(T) == 4) return launch_cluster_nr<T, 8>(c, mode, a, n_iters);
            return fail(CIMCS_CONFIG_ERROR, "cluster loop: too many replica slots");
    }
}

int launch_cluster(cimcs_ctx* c, int mode, const GemvArgs& a, int n_iters) {
    return c->st64() ? launch_cluster_T<double>(c, mode, a, n_iters)
                                 : launch_cluster_T<float>(c, mode, a, n_iters);
}

}  // namespace
