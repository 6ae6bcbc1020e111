// rt_context.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): struct cimcs_ctx: the device context (problems, state, paths, graphs).
#pragma once

// NVTX ranges around the host-side phases of the ABI calls (header-only NVTX v3:
// no-ops unless a tool such as Nsight Systems injects itself)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ======================================================================= ctx
struct cimcs_ctx {
    int device = 0, dtype = CIMCS_F32;
    cudaStream_t stream = nullptr;
    int host_threads = 0;
    bool use_graphs = true;
    bool use_cluster = true;  // small N: whole CIM call / refit in one cluster launch
    bool want_tc = true;  // fp32 contraction on tcgen05 (3xTF32)
    bool tc_requested = true;  // want_tc when the resident problems were set
    // row sharding (one rank per GPU): this rank owns spin rows [row0, row1)
    int world = 1, rank = 0;
    bool sharded = false;  // created by cimcs_create_sharded (padded row layout)
    ncclComm_t comm = nullptr;
    int row0 = 0, row1 = 0, rb0 = 0;
    double* tp = nullptr;        // per-trajectory score partials [B*NR][5]
    int* fail_tmp = nullptr;     // local fail_gstep before the cross-rank MIN
    bool tc = false;      // active for the current problem set
    bool sym = false;      // active for the current problem set
    // fp64 symmetric-tile path on the DMMA tensor cores (sym64_kernels.cuh):
    // unsharded fp64 contexts with N > kClMaxN (option "sym64", default on)
    // compacted Jacobi refit of the fp32 symmetric path (cmp_kernels.cuh; option
    // "refit_compact", default on): the union of the replicas' supports per instance
    int cmp_opt = 1;
    bool cmp_active = false;     // the context's fields are swapped to the compacted problem
    int symS = 4;                // item edge of the symmetric schedules (kSyS; 2 when compacted)
    int* cU = nullptr;           // [B][ldN] union spins (ascending), -1 padded
    int* cCnt = nullptr;         // [B] union sizes
    int* cMax = nullptr;         // [1] max union size
    float *Rc = nullptr, *Dc = nullptr, *hzc = nullptr;
    int8_t* sigc = nullptr;
    __half* Gc = nullptr;        // compacted tiles (capacity: the full triangle)
    // the fp64 path's segment-preserving compacted refit (cmp_kernels.cuh, cmp64):
    // 512-column segments compacted one by one so the canonical fma order is kept
    int* cU6 = nullptr;          // [B][ldN] compacted index -> spin (-1: pad)
    int* cSegc = nullptr;        // [B][nseg] union spins per original segment
    int* cPfx = nullptr;         // [B][nseg] their exclusive prefix per instance
    int* cSegOff = nullptr;      // [nseg] compacted offset of segment s (-1: dropped)
    int2* cSeg = nullptr;        // [nseg] compacted segments: (first block, blocks)
    double *Rc6 = nullptr, *Dc6 = nullptr, *hzc6 = nullptr;
    void* Gc6 = nullptr;         // compacted fp64 tiles (capacity: the full triangle)
    bool want_sym64 = true;
    bool sym64 = false;
    int nRB6 = 0, ntri6 = 0, nSB6 = 0;      // its geometry: 64-row blocks, 512 x 512 items
    void* dG6 = nullptr;                    // its gram tiles [B][ntri6][64 x 64] fp64
    double *WT0 = nullptr, *WT1 = nullptr;  // fp64 w tiles of W0 / W1 [B][nRB][64][NR]
    double* dPart6 = nullptr;               // partials [B][nRB][nSB][64][NR]
    int ntri = 0;          // upper-triangle tiles per instance
    int nSB = 0;           // super-block items per row of the tile triangle (kSyS tiles)
    struct SymSched {      // LPT placement of the items of nb instances on the CTAs
        int nb = 0, nRB = 0, S = 0, grid = 0;
        int2* items = nullptr;
        int* sched = nullptr;
    };
    std::vector<SymSched> ssched;
    SymSched cmp_sched;    // the compacted fp64 refit's schedule (rebuilt per alternation)
    int cmp_items_cap = 0;
    int* dSg = nullptr;    // per-instance gram scale exponent
    float* dSpart = nullptr;  // partial products [B][nRB][nSB][128][NR]
    bool use_pdl = true;      // programmatic dependent launch between the step kernels
    bool overlap_upd = true;  // fp64 DMMA path: item flags, an instance's update runs under the tile kernel
    unsigned* dDone = nullptr;  // [2][B] item / update-CTA counters of the flags
    unsigned long long* dTl = nullptr;  // option "timeline": per-CTA %globaltimer stamps
    int gram_l2 = 0;          // per instance, the first gram_l2 tiles of the triangle are copied
                              // with evict_last (an L2-resident subset), the rest evict_first
    bool kernel_timing = false;  // eager mode: CUDA events around each step-mode tile kernel
    cudaEvent_t kt_ev[2] = {nullptr, nullptr};
    // tile sharding of the symmetric path (cimcs_create_sharded contexts, option
    // "tile_shard", default on): every rank keeps the full state and streams only
    // the gram tiles of its super-rows [sP0, sP1); the per-rank slot sums are
    // all-reduced (NCCL) before the replicated update -- one collective per step
    int sh_world = 1, sh_rank = 0;  // geometry given at creation
    bool sh_rows = false;           // created sharded
    int tshard_opt = 1;
    bool tshard = false;            // active for the current problem set
    int tworld = 1, trank = 0, sP0 = 0, sP1 = 0;
    float* dH = nullptr;            // [B][nRB][128][NR] summed partial products
    int gram_tc = 0;          // large-N fp32 gram on tcgen05 (gram_tc_kernels.cuh): 0 auto (N >= 8192), 1, -1
    // matrix-free MRI transform-chain problem (mri_kernels.cuh; mri.hpp:46-99)
    bool mri = false;
    int mH = 0, mW = 0, mL = 0;
    float mgamma = 0.f;
    unsigned char* dMaskBr = nullptr;  // [H*W] sampled, bit-reversed coordinates
    float2* dTw = nullptr;             // [L/2] exp(-2 pi i k / L)
    float* dTarget = nullptr;          // [H*W] target image (row-major)
    bool mri_cluster = true;           // per-step apply on one cluster per replica
    // chain kind: 0 the reference's DFT chain, 1 config 3's DCT o Haar^-1 chain
    // (dct_kernels.cuh; A = S C2 Psi_L^-1, damped Jacobi allowed: its G is the
    // dense config-3 problem's)
    int mri_kind = 0;
    int dct_L = 0;                     // Haar levels
    float* dDctC = nullptr;            // [128][128] DCT-II matrix
    unsigned char* dDctMask = nullptr; // [128 * 128] sampled frequencies
    float* dDctY = nullptr;            // [128 * 128] observations on the frequency grid
    __half *WB0 = nullptr, *WB1 = nullptr;  // fp16 B tiles of W0 / W1 [B][nRB][2NR x 128]
    int *WS0 = nullptr, *WS1 = nullptr;     // their scale exponents [B][nRB][NR]
    size_t spart_elems = 0;
    int nch = 0;
    int num_sms = 148;
    int sched_ctas = 0;   // option: CTAs of the symmetric item schedules (0: one per SM)
    int sched_n() const { return sched_ctas > 0 ? std::min(sched_ctas, num_sms) : num_sms; }
    // problems
    int B = 0, N = 0, ldN = 0, Mmax = 0;
    std::vector<int> M;
    bool has_truth = false, built = false;
    double *dA = nullptr, *dy = nullptr;
    int* dM = nullptr;
    void* dG = nullptr;      // gram panels [B][nRB][ldJ][RB] in the path's dtype
    int ldJ = 0, nRB = 0, RB = 0;  // nRB: row blocks held by this rank
    void *dD = nullptr, *dhz = nullptr;
    double* dx = nullptr;
    int8_t* dxi = nullptr;
    // trajectory state (NR slots)
    int NR = 0;
    void *Rs = nullptr, *C = nullptr, *E = nullptr, *W0 = nullptr, *W1 = nullptr,
         *Hdbg = nullptr, *bestR = nullptr;
    int8_t *sig = nullptr, *bestS = nullptr;
    int *fail_gstep = nullptr, *fail_idx = nullptr, *n_hist = nullptr, *improved = nullptr,
        *err = nullptr;
    unsigned long long* minE = nullptr;
    double *part = nullptr, *best_obj = nullptr, *stage = nullptr, *obj = nullptr,
           *rmse = nullptr, *ham = nullptr;
    int32_t* stage_i = nullptr;
    size_t stage_elems = 0;
    AltParams* alt = nullptr;
    // reusable host/device buffers and the instantiated solve graphs
    double* pin = nullptr;        // pinned staging for uploads (2 slots)
    size_t pin_bytes = 0;         // per slot
    double* pin_c0 = nullptr;     // pinned c0 double buffer
    size_t pin_c0_elems = 0;
    double* dc0 = nullptr;        // device c0 of the current alternation
    size_t dc0_elems = 0;
    cudaGraphExec_t g_cim = nullptr, g_refit = nullptr;
    std::vector<long long> graph_key;
    double* pump = nullptr;
    int pump_cap = 0;
    DevRecord* hist = nullptr;
    int hist_cap = 0;
    // Positive-P state (allocated on first use): moments n, m, measured amplitude,
    // unit normals in chunks of kPpChunk steps (device and pinned, double buffered)
    void *Pn = nullptr, *Pm = nullptr, *MT = nullptr;
    double *nzd[2] = {nullptr, nullptr}, *nzh[2] = {nullptr, nullptr};
    size_t nz_elems = 0;
    // conjugate-gradient refit state (allocated on first use)
    double *cgX = nullptr, *cgR = nullptr, *cgP = nullptr, *cgGp = nullptr;
    int* cg_act = nullptr;
    void* cg_st = nullptr;        // CgTraj[B*NR]
    int* cg_live = nullptr;       // [0] live counter, [1] last value
    cudaStream_t side = nullptr;  // captures the CG loop body
    cimcs_timing timing{};

    // fp64 state arrays (c, e, R, w, D, hz)
    bool st64() const { return dtype == CIMCS_F64; }
    size_t elt() const { return st64() ? 8 : 4; }
    const void* G() const { return dG; }
    size_t state_elems() const { return (size_t)B * ldN * NR; }
    // contraction-input arrays: [b][i][r], or (tc) [W | W_lo] canonical, 2*NR rows
    size_t w_elems() const { return (size_t)B * (ldJ > ldN ? ldJ : ldN) * NR * (tc ? 2 : 1); }
};
