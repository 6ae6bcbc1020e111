// rt_abi_problems.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): C ABI: problem sets (host, device-generated, MRI), K1 coupling build,
// coupling read-back.
#pragma once

extern "C" {

// Problem-set layout decisions and device allocations shared by set_problems
// (host instances) and set_generated_problems (instances generated on the GPU).
int prepare_problems(cimcs_ctx* c, int32_t B, int32_t N, const int32_t* M, bool truth) {
    CK(cudaSetDevice(c->device));
    // same shapes as the resident problem set: keep every device allocation
    const bool reuse = c->dA && c->B == B && c->N == N && c->has_truth == truth &&
                       std::equal(c->M.begin(), c->M.end(), M) && (int)c->M.size() == B &&
                       c->want_tc == c->tc_requested && !c->sh_rows;
    if (!reuse) free_problems(c);
    c->built = false;
    c->tc_requested = c->want_tc;
    c->B = B;
    c->N = N;
    c->ldN = (N + 31) / 32 * 32;
    c->ldJ = (N + kChunk - 1) / kChunk * kChunk;
    // fp32 tensor cores = the symmetric-tile path, for N above the cluster-loop
    // range, unsharded or tile-sharded; everything else runs on CUDA cores
    c->tc = c->dtype == CIMCS_F32 && c->want_tc && N > kClMaxN && (!c->sh_rows || c->tshard_opt);
    c->RB = c->tc ? kTcRows : (c->st64() ? row_block<double>() : row_block<float>());
    c->row0 = 0;
    c->row1 = N;
    c->rb0 = 0;
    c->nRB = (N + c->RB - 1) / c->RB;
    // sharded contexts on the symmetric path split gram TILES (replicated
    // state, one all-reduce per step); otherwise gram ROWS (all-gather of w)
    c->world = c->sh_rows ? c->sh_world : 1;
    c->rank = c->sh_rows ? c->sh_rank : 0;
    c->sharded = c->sh_rows;
    c->tshard = c->sh_rows && c->tc;
    c->tworld = c->tshard ? c->world : 1;
    c->trank = c->tshard ? c->rank : 0;
    if (c->tshard) {
        c->world = 1;
        c->rank = 0;
        c->sharded = false;
    }
    if (c->sharded) {
        // row sharding: equal slices of whole 128-row tiles (sharding.row_shard)
        const int per = (N + c->world * 128 - 1) / (c->world * 128) * 128;
        c->ldN = c->ldJ = per * c->world;
        c->row0 = std::min(N, c->rank * per);
        c->row1 = std::min(N, c->row0 + per);
        c->rb0 = c->row0 / c->RB;
        c->nRB = c->row1 > c->row0 ? (c->row1 - c->row0 + c->RB - 1) / c->RB : 0;
    }
    c->nch = c->ldJ / kTcChunk;
    c->sym = c->tc;
    // fp64: DMMA symmetric tiles for unsharded contexts above the cluster range
    // (64-row blocks = row_block<double>(), 512 x 512 items)
    c->sym64 = c->dtype == CIMCS_F64 && c->want_sym64 && !c->sh_rows && N > kClMaxN;
    c->nRB6 = c->sym64 ? (N + kT6 - 1) / kT6 : 0;
    c->ntri6 = c->nRB6 * (c->nRB6 + 1) / 2;
    c->nSB6 = (c->nRB6 + kS6 - 1) / kS6;
    c->ntri = c->sym ? c->nRB * (c->nRB + 1) / 2 : 0;
    c->nSB = (c->nRB + kSyS - 1) / kSyS;
    if (c->tshard) tile_shard(c->nRB, c->tworld, c->trank, &c->sP0, &c->sP1);
    c->M.assign(M, M + B);
    c->Mmax = *std::max_element(c->M.begin(), c->M.end());
    c->has_truth = truth;
    const size_t astride = (size_t)c->Mmax * N;
    int rc;
    if (!reuse && ((rc = dalloc(c, &c->dA, (size_t)B * astride * 8)) ||
                   (rc = dalloc(c, &c->dy, (size_t)B * c->Mmax * 8)) ||
                   (rc = dalloc(c, &c->dM, (size_t)B * 4))))
        return rc;
    if (truth && !c->dx) {
        if ((rc = dalloc(c, &c->dx, (size_t)B * c->ldN * 8)) ||
            (rc = dalloc(c, &c->dxi, (size_t)B * c->ldN)))
            return rc;
    }
    return 0;
}

// ---------------------------------------- counter-based device generator
// SURVEY 8f row 4, the documented deviation: config-4-scale instances (A alone
// is 5e9 normals) drawn on the GPU from Philox4x32-10 streams instead of the
// reference's single sequential mt19937_64 stream (datagen.cpp:15-55), whose
// bit-exact reproduction needs that stream's order and glibc's log/cos.  Same
// recipe and shapes: A_kr = N(0,1)/sqrt(M) (draw index k N + r, stream 0),
// x_r = N(0,1) (stream 1), support = the K positions with the smallest
// Philox keys (stream 2, a uniform K-subset), y = A (xi . x) + nu N(0,1)
// (stream 3) summed over the support in ascending order as gen_instance does.
// Different numbers from the reference's instances -- never used for parity.
__host__ __device__ inline void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
        const uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
        const uint32_t n0 = h1 ^ c[1] ^ k0, n2 = h0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = l1;
        c[2] = n2;
        c[3] = l0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}
__host__ __device__ inline void philox_u64x2(uint64_t seed, uint32_t stream, uint64_t idx,
                                             uint64_t* a, uint64_t* b) {
    uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), stream, 0x5eedu};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    *a = (uint64_t)c[0] | ((uint64_t)c[1] << 32);
    *b = (uint64_t)c[2] | ((uint64_t)c[3] << 32);
}
__device__ inline double philox_normal(uint64_t seed, uint32_t stream, uint64_t idx) {
    uint64_t a, b;
    philox_u64x2(seed, stream, idx, &a, &b);
    const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53, u2 = (double)(b >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);  // rng.hpp's Box-Muller form
}
__global__ void devgen_a_kernel(double* A, int M, int N, uint64_t seed, double col_std) {
    const size_t total = (size_t)M * N;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t r = t / M, k = t % M;  // column-major storage, row-major draw index
        A[t] = col_std * philox_normal(seed, 0, (uint64_t)k * N + r);
    }
}
__global__ void devgen_x_kernel(double* x, int N, uint64_t seed) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x)
        x[r] = philox_normal(seed, 1, r);
}
__global__ void devgen_y_kernel(const double* __restrict__ A, int M, const int* __restrict__ supp,
                                int K, const double* __restrict__ x, double nu, uint64_t seed,
                                double* y) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < M; k += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < K; ++s) acc = acc + A[(size_t)supp[s] * M + k] * x[supp[s]];
        y[k] = acc + nu * philox_normal(seed, 3, k);
    }
}

int cimcs_set_generated_problems(cimcs_ctx* c, int32_t B, int32_t N, const double* alpha,
                                 const double* a, const double* nu, const uint64_t* seeds) {
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    if (B < 1 || N < 1 || !alpha || !a || !nu || !seeds)
        return fail(CIMCS_INPUT_ERROR, "set_generated_problems: bad arguments");
    std::vector<int32_t> M(B), K(B);
    for (int b = 0; b < B; ++b)
        if (gen_dims(N, alpha[b], a[b], &M[b], &K[b]) || nu[b] < 0.0)
            return fail(CIMCS_INPUT_ERROR, "gen_instance: bad arguments");
    if (int rc = prepare_problems(c, B, N, M.data(), true)) return rc;
    const size_t astride = (size_t)c->Mmax * N;
    int* dsupp = nullptr;
    if (int rc = dalloc(c, &dsupp, (size_t)N * 4)) return rc;
    std::unique_ptr<int, decltype(&cudaFree)> g(dsupp, &cudaFree);
    CK(cudaMemsetAsync(c->dx, 0, (size_t)B * c->ldN * 8, c->stream));
    CK(cudaMemsetAsync(c->dxi, 0, (size_t)B * c->ldN, c->stream));
    CK(cudaMemcpyAsync(c->dM, M.data(), (size_t)B * 4, cudaMemcpyHostToDevice, c->stream));
    for (int b = 0; b < B; ++b) {
        // support: the K smallest stream-2 keys (host, O(N log N))
        std::vector<std::pair<uint64_t, int>> key(N);
        for (int r = 0; r < N; ++r) {
            uint64_t k0, k1;
            philox_u64x2(seeds[b], 2, (uint64_t)r, &k0, &k1);
            key[r] = {k0, r};
        }
        std::partial_sort(key.begin(), key.begin() + K[b], key.end());
        std::vector<int> supp(K[b]);
        for (int s = 0; s < K[b]; ++s) supp[s] = key[s].second;
        std::sort(supp.begin(), supp.end());
        std::vector<int8_t> xi8((size_t)c->ldN, 0);
        for (int r : supp) xi8[r] = 1;
        double* Ab = c->dA + (size_t)b * astride;
        double* xb = c->dx + (size_t)b * c->ldN;
        devgen_a_kernel<<<8 * c->num_sms, 256, 0, c->stream>>>(Ab, M[b], N, seeds[b],
                                                              1.0 / std::sqrt((double)M[b]));
        devgen_x_kernel<<<(N + 255) / 256, 256, 0, c->stream>>>(xb, N, seeds[b]);
        CK(cudaMemcpyAsync(c->dxi + (size_t)b * c->ldN, xi8.data(), xi8.size(),
                           cudaMemcpyHostToDevice, c->stream));
        if (K[b] > 0)
            CK(cudaMemcpyAsync(dsupp, supp.data(), (size_t)K[b] * 4, cudaMemcpyHostToDevice,
                               c->stream));
        devgen_y_kernel<<<(M[b] + 255) / 256, 256, 0, c->stream>>>(
            Ab, M[b], dsupp, K[b], xb, nu[b], seeds[b], c->dy + (size_t)b * c->Mmax);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));  // xi8 / supp are reused next instance
    }
    return 0;
}

// the resident instance b back on the host (A column-major M x N; truth when set)
int cimcs_get_instance(cimcs_ctx* c, int32_t b, double* A, double* y, double* x_true,
                       int32_t* xi_true) {
    if (!c || b < 0 || b >= c->B || c->mri || !c->dA) return fail(CIMCS_INPUT_ERROR, "bad instance");
    CK(cudaStreamSynchronize(c->stream));  // cudaMemcpy does not order against c->stream
    const int N = c->N, M = c->M[b];
    const size_t astride = (size_t)c->Mmax * N;
    if (A) {
        if (int rc_ = copy_sync(c, A, c->dA + (size_t)b * astride, (size_t)M * N * 8,
                                cudaMemcpyDeviceToHost))
            return rc_;
    }
    if (y) {
        if (int rc_ = copy_sync(c, y, c->dy + (size_t)b * c->Mmax, (size_t)M * 8,
                                cudaMemcpyDeviceToHost))
            return rc_;
    }
    if (c->has_truth && x_true)
        if (int rc_ = copy_sync(c, x_true, c->dx + (size_t)b * c->ldN, (size_t)N * 8, cudaMemcpyDeviceToHost)) return rc_;
    if (c->has_truth && xi_true) {
        std::vector<int8_t> t((size_t)N);
        if (int rc_ = copy_sync(c, t.data(), c->dxi + (size_t)b * c->ldN, (size_t)N, cudaMemcpyDeviceToHost)) return rc_;
        for (int i = 0; i < N; ++i) xi_true[i] = t[i];
    }
    return 0;
}

int cimcs_set_problems(cimcs_ctx* c, int32_t B, int32_t N, const int32_t* M,
                       const double* const* A, const double* const* y,
                       const double* const* x_true, const int32_t* const* xi_true) {
    NvtxRange nvtx_range_("cimcs_set_problems");
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    if (B < 1 || N < 1) return fail(CIMCS_INPUT_ERROR, "need B >= 1 and N >= 1");
    for (int b = 0; b < B; ++b)
        if (M[b] < 1 || !A[b] || !y[b]) return fail(CIMCS_INPUT_ERROR, "empty A");
    const bool truth = x_true != nullptr && xi_true != nullptr;
    if (int rc = prepare_problems(c, B, N, M, truth)) return rc;
    const size_t astride = (size_t)c->Mmax * N;
    // A and y go through a pinned double buffer filled by host threads
    // (pageable cudaMemcpy runs at a fraction of the link rate)
    if (int rc2 = staged_upload(c, B, [&](int b) { return (size_t)M[b] * N * 8; },
                                [&](int b) { return reinterpret_cast<const char*>(A[b]); },
                                [&](int b) { return reinterpret_cast<char*>(c->dA + (size_t)b * astride); }))
        return rc2;
    if (int rc2 = staged_upload(c, B, [&](int b) { return (size_t)M[b] * 8; },
                                [&](int b) { return reinterpret_cast<const char*>(y[b]); },
                                [&](int b) { return reinterpret_cast<char*>(c->dy + (size_t)b * c->Mmax); }))
        return rc2;
    CK(cudaMemcpyAsync(c->dM, M, (size_t)B * 4, cudaMemcpyHostToDevice, c->stream));
    if (c->has_truth) {
        std::vector<int8_t> xi8((size_t)B * c->ldN, 0);
        for (int b = 0; b < B; ++b) {
            CK(cudaMemcpyAsync(c->dx + (size_t)b * c->ldN, x_true[b], (size_t)N * 8,
                               cudaMemcpyHostToDevice, c->stream));
            for (int i = 0; i < N; ++i) {
                if (xi_true[b][i] != 0 && xi_true[b][i] != 1)
                    return fail(CIMCS_INPUT_ERROR, "xi_true must be 0/1");
                xi8[(size_t)b * c->ldN + i] = (int8_t)xi_true[b][i];
            }
        }
        CK(cudaMemcpyAsync(c->dxi, xi8.data(), xi8.size(), cudaMemcpyHostToDevice, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int cimcs_mri_lasso(cimcs_ctx* c, double lambda, int32_t max_iters, double tol, double step,
                    double* x_out, int32_t* iterations, double* objective) {
    if (!c || !c->mri || !c->built) return fail(CIMCS_INPUT_ERROR, "mri_lasso: no built MRI problem");
    if (c->mri_kind != 0) return fail(CIMCS_CONFIG_ERROR, "mri_lasso: DFT transform-chain problems only");
    if (lambda < 0.0) return fail(CIMCS_INPUT_ERROR, "lasso: lambda_l1 must be >= 0");
    if (!(step > 0.0)) return fail(CIMCS_INPUT_ERROR, "lasso: step must be > 0");
    if (max_iters < 0 || !x_out) return fail(CIMCS_INPUT_ERROR, "mri_lasso: bad arguments");
    CK(cudaSetDevice(c->device));
    const int N = c->N;
    float *zx = nullptr, *gzx = nullptr;
    LassoState* st = nullptr;
    int rc;
    if ((rc = dalloc(c, &zx, (size_t)N * 2 * 4)) || (rc = dalloc(c, &gzx, (size_t)N * 2 * 4)) ||
        (rc = dalloc(c, &st, sizeof(LassoState))))
        return rc;
    std::unique_ptr<float, decltype(&cudaFree)> g1(zx, &cudaFree), g2(gzx, &cudaFree);
    std::unique_ptr<LassoState, decltype(&cudaFree)> g3(st, &cudaFree);
    LassoState s0{1.0, 0.0, 0.0, 0, max_iters == 0 ? 1 : 0};
    CK(cudaMemsetAsync(zx, 0, (size_t)N * 2 * 4, c->stream));
    CK(cudaMemcpyAsync(st, &s0, sizeof s0, cudaMemcpyHostToDevice, c->stream));
    MriArgs ma{};
    ma.H = c->mH;
    ma.W = c->mW;
    ma.N = N;
    ma.NR = 2;
    ma.mask_br = c->dMaskBr;
    ma.tw = c->dTw;
    ma.L = c->mL;
    ma.gamma = 0.f;  // apply_fit: Re(A^H A), no smoothness (mri.cpp:299-301)
    ma.scale = 1.f / (float)N;
    ma.in = zx;
    ma.out = gzx;
    const size_t smem = mri_smem_bytes(c->mH, c->mW, c->mL);
    LassoState hs = s0;
    while (!hs.done) {
        for (int k = 0; k < 64; ++k) {  // device-side stop: launches after it return at once
            mri_kernel<<<2, kMriThreads, smem, c->stream>>>(ma, MRI_APPLY);
            lasso_kernel<<<1, kLassoThreads, 0, c->stream>>>(gzx, zx, static_cast<const float*>(c->dhz),
                                                             N, lambda, step, tol, max_iters, st);
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    std::vector<float> h((size_t)N * 2);
    if (int rc_ = copy_sync(c, h.data(), zx, h.size() * 4, cudaMemcpyDeviceToHost)) return rc_;
    for (int i = 0; i < N; ++i) x_out[i] = h[2 * i + 1];
    if (iterations) *iterations = hs.it;
    if (objective) *objective = hs.f;
    return 0;
}

int cimcs_tile_shard(int32_t nRB, int32_t world, int32_t rank, int32_t* P0, int32_t* P1) {
    if (nRB < 1 || world < 1 || rank < 0 || rank >= world || !P0 || !P1)
        return fail(CIMCS_INPUT_ERROR, "tile_shard: bad arguments");
    int a = 0, b = 0;
    tile_shard(nRB, world, rank, &a, &b);
    *P0 = a;
    *P1 = b;
    return 0;
}

int cimcs_make_mask(int32_t H, int32_t W, int32_t M, uint64_t seed, int32_t* out) {
    const long long N = (long long)H * W;
    if (H < 1 || W < 1) return fail(CIMCS_INPUT_ERROR, "make_mask: dims must be >= 1");
    if (M < 1 || M > N) return fail(CIMCS_INPUT_ERROR, "make_mask: M out of range");
    std::vector<int> pool((size_t)N);
    for (long long k = 0; k < N; ++k) pool[k] = (int)k;
    HostRng rng(seed);  // partial Fisher-Yates, mri.cpp:185-207
    for (int i = 0; i < M; ++i) {
        const long long pick = i + (long long)rng.uniform_below((uint64_t)(N - i));
        std::swap(pool[i], pool[pick]);
    }
    std::sort(pool.begin(), pool.begin() + M);
    std::copy(pool.begin(), pool.begin() + M, out);
    return 0;
}

int cimcs_set_mri_problem(cimcs_ctx* c, int32_t H, int32_t W, const double* target,
                          int32_t M, const int32_t* mask, double gamma, const double* x_true) {
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    auto pow2 = [](int v) { return v >= 1 && (v & (v - 1)) == 0; };
    if (!pow2(H) || !pow2(W)) return fail(CIMCS_INPUT_ERROR, "MriTransform: dimensions must be powers of two");
    if (H < 2 || W < 2 || H > kMriMaxLine || W > kMriMaxLine)
        return fail(CIMCS_INPUT_ERROR,
                    "MriTransform: need 2 <= H, W <= 128 (an FFT line lives in one warp's registers)");
    if (!(gamma >= 0.0)) return fail(CIMCS_INPUT_ERROR, "MriTransform: gamma must be >= 0");
    if (!target || !mask || M < 1) return fail(CIMCS_INPUT_ERROR, "MriTransform: mask indices must be unique and in range");
    std::vector<int> idx(mask, mask + M);
    std::sort(idx.begin(), idx.end());
    if (idx.front() < 0 || idx.back() >= H * W || std::adjacent_find(idx.begin(), idx.end()) != idx.end())
        return fail(CIMCS_INPUT_ERROR, "MriTransform: mask indices must be unique and in range");
    if (c->dtype != CIMCS_F32) return fail(CIMCS_CONFIG_ERROR, "matrix-free MRI problems run in fp32 contexts");
    if (c->world > 1 || c->sharded) return fail(CIMCS_CONFIG_ERROR, "matrix-free MRI problems are single-GPU");
    CK(cudaSetDevice(c->device));
    free_problems(c);
    const int N = H * W;
    c->built = false;
    c->mri = true;
    c->mH = H;
    c->mW = W;
    c->mL = std::max(H, W);
    c->mgamma = (float)gamma;
    c->B = 1;
    c->N = N;
    c->ldN = c->ldJ = (N + 31) / 32 * 32;
    c->tc = c->sym = c->sym64 = false;
    c->RB = kSyT;
    c->row0 = 0;
    c->row1 = N;
    c->rb0 = 0;
    c->nRB = (N + kSyT - 1) / kSyT;
    c->nSB = 1;
    c->ntri = 0;
    c->nch = 0;
    c->M.assign(1, M);
    c->Mmax = M;
    c->has_truth = x_true != nullptr;
    // mask in the bit-reversed coordinates of the DIF spectrum, twiddles, target
    auto rev = [](int v, int n) {
        int r = 0;
        for (int b = 1; b < n; b <<= 1, v >>= 1) r = (r << 1) | (v & 1);
        return r;
    };
    std::vector<unsigned char> full((size_t)N, 0), br((size_t)N, 0);
    for (int k : idx) full[k] = 1;
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) br[(size_t)i * W + j] = full[(size_t)rev(i, H) * W + rev(j, W)];
    std::vector<float2> tw(64);  // exp(-2 pi i k / 128): every line length divides 128
    for (int k = 0; k < 64; ++k) {
        const double a = -2.0 * M_PI * k / 128.0;
        tw[k] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    std::vector<float> tgt((size_t)N);
    for (int k = 0; k < N; ++k) tgt[k] = (float)target[k];
    int rc;
    if ((rc = dalloc(c, &c->dMaskBr, (size_t)N)) || (rc = dalloc(c, &c->dTw, tw.size() * sizeof(float2))) ||
        (rc = dalloc(c, &c->dTarget, (size_t)N * 4)))
        return rc;
    if (int rc_ = copy_sync(c, c->dMaskBr, br.data(), br.size(), cudaMemcpyHostToDevice)) return rc_;
    if (int rc_ = copy_sync(c, c->dTw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice)) return rc_;
    if (int rc_ = copy_sync(c, c->dTarget, tgt.data(), tgt.size() * 4, cudaMemcpyHostToDevice)) return rc_;
    static std::atomic<unsigned long long> attr{0};
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(mri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)mri_smem_bytes(128, 128, 128)));
        CK(cudaFuncSetAttribute(mri_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)mri_cluster_smem_bytes(128, 128)));
        attr.fetch_or(1ull << c->device);
    }
    if (c->has_truth) {  // make_problem(t, &truth): xi = (x != 0) (mri.cpp:398-405)
        if ((rc = dalloc(c, &c->dx, (size_t)c->ldN * 8)) || (rc = dalloc(c, &c->dxi, (size_t)c->ldN)))
            return rc;
        std::vector<int8_t> xi8((size_t)c->ldN, 0);
        for (int i = 0; i < N; ++i) xi8[i] = x_true[i] != 0.0 ? 1 : 0;
        if (int rc_ = copy_sync(c, c->dx, x_true, (size_t)N * 8, cudaMemcpyHostToDevice)) return rc_;
        if (int rc_ = copy_sync(c, c->dxi, xi8.data(), xi8.size(), cudaMemcpyHostToDevice)) return rc_;
    }
    return 0;
}

int cimcs_set_dct_problem(cimcs_ctx* c, int32_t n, int32_t levels, int32_t M,
                          const int32_t* freqs, const double* y, const double* x_true) {
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    if (n != kDctN) return fail(CIMCS_INPUT_ERROR, "dct problem: the image edge must be 128");
    if (levels < 1 || levels > kDctMaxLevels)
        return fail(CIMCS_INPUT_ERROR, "dct problem: Haar levels must be in [1, 3]");
    const int N = n * n;
    if (M < 1 || M > N || !freqs || !y)
        return fail(CIMCS_INPUT_ERROR, "dct problem: need 1 <= M <= N frequencies and observations");
    std::vector<int> idx(freqs, freqs + M);
    std::sort(idx.begin(), idx.end());
    if (idx.front() < 0 || idx.back() >= N || std::adjacent_find(idx.begin(), idx.end()) != idx.end())
        return fail(CIMCS_INPUT_ERROR, "dct problem: frequencies must be unique and in range");
    if (c->dtype != CIMCS_F32) return fail(CIMCS_CONFIG_ERROR, "matrix-free chain problems run in fp32 contexts");
    if (c->world > 1 || c->sharded) return fail(CIMCS_CONFIG_ERROR, "matrix-free chain problems are single-GPU");
    CK(cudaSetDevice(c->device));
    free_problems(c);
    c->built = false;
    c->mri = true;
    c->mri_kind = 1;
    c->dct_L = levels;
    c->mH = c->mW = c->mL = n;
    c->mgamma = 0.f;
    c->B = 1;
    c->N = N;
    c->ldN = c->ldJ = N;
    c->tc = c->sym = c->sym64 = false;
    c->RB = kSyT;
    c->row0 = 0;
    c->row1 = N;
    c->rb0 = 0;
    c->nRB = (N + kSyT - 1) / kSyT;
    c->nSB = 1;
    c->ntri = 0;
    c->nch = 0;
    c->M.assign(1, M);
    c->Mmax = M;
    c->has_truth = x_true != nullptr;
    // orthonormal DCT-II rows, stored in the kernel's swizzled shared-memory layout
    std::vector<float> C((size_t)N), Y((size_t)N, 0.f);
    for (int u = 0; u < n; ++u)
        for (int x = 0; x < n; ++x)
            C[(size_t)dofs(u, x)] = (float)(std::cos(M_PI * (2 * x + 1) * u / (2.0 * n)) *
                                           std::sqrt((u ? 2.0 : 1.0) / n));
    std::vector<unsigned char> mask((size_t)N, 0);
    for (int m = 0; m < M; ++m) {
        mask[freqs[m]] = 1;
        Y[freqs[m]] = (float)y[m];
    }
    int rc;
    if ((rc = dalloc(c, &c->dDctC, (size_t)N * 4)) || (rc = dalloc(c, &c->dDctMask, (size_t)N)) ||
        (rc = dalloc(c, &c->dDctY, (size_t)N * 4)))
        return rc;
    if ((rc = copy_sync(c, c->dDctC, C.data(), C.size() * 4, cudaMemcpyHostToDevice)) ||
        (rc = copy_sync(c, c->dDctMask, mask.data(), mask.size(), cudaMemcpyHostToDevice)) ||
        (rc = copy_sync(c, c->dDctY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice)))
        return rc;
    static std::atomic<unsigned long long> attr{0};
    if (!(attr.load() >> c->device & 1ull)) {
        for (auto k : {dct_cluster_kernel<1>, dct_cluster_kernel<2>, dct_cluster_kernel<3>})
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)dct_smem_bytes()));
        attr.fetch_or(1ull << c->device);
    }
    if (c->has_truth) {
        if ((rc = dalloc(c, &c->dx, (size_t)c->ldN * 8)) || (rc = dalloc(c, &c->dxi, (size_t)c->ldN)))
            return rc;
        std::vector<int8_t> xi8((size_t)c->ldN, 0);
        for (int i = 0; i < N; ++i) xi8[i] = x_true[i] != 0.0 ? 1 : 0;
        if ((rc = copy_sync(c, c->dx, x_true, (size_t)N * 8, cudaMemcpyHostToDevice)) ||
            (rc = copy_sync(c, c->dxi, xi8.data(), xi8.size(), cudaMemcpyHostToDevice)))
            return rc;
    }
    return 0;
}

int cimcs_build_coupling(cimcs_ctx* c) {
    NvtxRange nvtx_range_("cimcs_build_coupling");
    if (!c || c->B < 1) return fail(CIMCS_INPUT_ERROR, "no problems set");
    CK(cudaSetDevice(c->device));
    if (c->mri) {  // hz = Re(A^H y) and diag(G) of the transform chain (mri.cpp:236-254)
        int rc;
        const size_t nv = (size_t)c->ldN;
        if (!c->dhz && (rc = dalloc(c, &c->dhz, nv * 4))) return rc;
        if (!c->dD && (rc = dalloc(c, &c->dD, nv * 4))) return rc;
        Events ev(2);
        cudaEventRecord(ev.ev[0], c->stream);
        CK(cudaMemsetAsync(c->dhz, 0, nv * 4, c->stream));
        CK(cudaMemsetAsync(c->dD, 0, nv * 4, c->stream));
        if (c->mri_kind == 1) {  // hz = A^T y = Psi C^T Y C, D = diag of the chain
            if ((rc = dct_launch(c, DCT_HZ, 1, 0, c->dDctY, static_cast<float*>(c->dhz), 1)) ||
                (rc = dct_launch(c, DCT_DIAG, c->N, 0, nullptr, static_cast<float*>(c->dD), 1)))
                return rc;
        } else if ((rc = mri_launch(c, MRI_HZ, 1, 0, c->dTarget, static_cast<float*>(c->dhz))) ||
                   (rc = mri_launch(c, MRI_DIAG, c->N, 0, nullptr, static_cast<float*>(c->dD)))) {
            return rc;
        }
        cudaEventRecord(ev.ev[1], c->stream);
        CK(cudaStreamSynchronize(c->stream));
        c->timing.gram_ms = ev.ms(0, 1);
        c->timing.other_launches += 2;
        c->built = true;
        return 0;
    }
    const size_t es = c->elt();
    // gram bytes: symmetric fp16 hi/lo tiles, symmetric fp64 tiles, or CUDA-core panels
    const size_t gbytes = c->sym     ? (size_t)c->B * c->ntri * 2 * kSyPlaneBytes
                          : c->sym64 ? 16
                                     : (size_t)c->B * c->nRB * c->ldJ * c->RB * es;
    if (c->sym64 && !c->dG6) {
        if (int rc = dalloc(c, &c->dG6, (size_t)c->B * c->ntri6 * kT6TileBytes)) return rc;
    }
    const size_t nv = (size_t)c->B * c->ldN;
    int rc;
    if (!c->dG && (rc = dalloc(c, &c->dG, gbytes))) return rc;
    if (!c->dhz && (rc = dalloc(c, &c->dhz, nv * es))) return rc;
    if (!c->dD && (rc = dalloc(c, &c->dD, nv * es))) return rc;
    if (c->sym && !c->dSg && (rc = dalloc(c, &c->dSg, c->B * 4))) return rc;
    Events ev(2);
    cudaEventRecord(ev.ev[0], c->stream);
    CK(cudaMemsetAsync(c->dG, 0, gbytes, c->stream));
    const int nt = (c->N + kG2T - 1) / kG2T;
    const int bi0 = c->row0 / kG2T;
    const int nti = c->world == 1 ? nt : (c->row1 - c->row0 + kG2T - 1) / kG2T;
    const int mirror = c->world == 1 ? 1 : 0;
    const size_t astride = (size_t)c->Mmax * c->N;
    // hz = A^T y, D = diag(G) first: the symmetric tiles are scaled by max D
    const dim3 g2((c->N + 127) / 128, c->B);
    if (c->st64())
        hz_diag_kernel<double><<<g2, 128, 0, c->stream>>>(
            c->dA, c->dy, c->dM, c->N, c->ldN, astride, c->Mmax, static_cast<double*>(c->dhz),
            static_cast<double*>(c->dD), c->B);
    else
        hz_diag_kernel<float><<<g2, 128, 0, c->stream>>>(
            c->dA, c->dy, c->dM, c->N, c->ldN, astride, c->Mmax, static_cast<float*>(c->dhz),
            static_cast<float*>(c->dD), c->B);
    CK(cudaGetLastError());
    if (c->sym) {
        sym_scale_kernel<float><<<c->B, 256, 0, c->stream>>>(
            static_cast<const float*>(c->dD), c->N, c->ldN, c->dSg);
        CK(cudaGetLastError());
    }
    // large instances on the symmetric path (N >= 8192: configs 3 and 4): G = A^T A
    // on the tcgen05 tensor cores from fp16 hi/lo splits of A, written straight into
    // the fp16 hi/lo tiles (gram_tc_kernels.cuh); option "gram_tc": 0 auto, 1 on, -1 off
    const bool blas = c->sym && (c->gram_tc > 0 || (c->gram_tc == 0 && c->N >= 8192));
    if (blas) {
        const int Np = c->nRB * kSyT;
        const int nchx = (c->Mmax + kGtK - 1) / kGtK;
        __half* Pv = nullptr;
        unsigned long long* amax = nullptr;
        unsigned* rounds = nullptr;  // per instance: the tile kernel's round gate (zeroed)
        if ((rc = dalloc(c, &Pv, (size_t)nchx * 2 * Np * kGtK * 2)) ||
            (rc = dalloc(c, &amax, (size_t)c->B * 8)) || (rc = dalloc(c, &rounds, (size_t)c->B * 4)))
            return rc;
        std::unique_ptr<unsigned, decltype(&cudaFree)> rguard(rounds, &cudaFree);
        std::unique_ptr<__half, decltype(&cudaFree)> pguard(Pv, &cudaFree);
        std::unique_ptr<unsigned long long, decltype(&cudaFree)> aguard(amax, &cudaFree);
        static std::atomic<unsigned long long> attr{0};
        if (!(attr.load() >> c->device & 1ull)) {
            CK(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kGtSmem));
            attr.fetch_or(1ull << c->device);
        }
        // tile-sharded: only the row blocks of this rank's super-rows
        const int Ib = c->tshard ? c->sP0 * kSyS : 0;
        const int Ie = c->tshard ? std::min(c->nRB, c->sP1 * kSyS) : c->nRB;
        long long ntile = 0;
        for (int I = Ib; I < Ie; ++I) ntile += c->nRB - I;
        for (int b = 0; b < c->B && ntile > 0; ++b) {
            const int M = c->M[b], nch = (M + kGtK - 1) / kGtK;
            const double* Ab = c->dA + (size_t)b * astride;
            gt_absmax_kernel<<<8 * c->num_sms, 256, 0, c->stream>>>(Ab, (size_t)M * c->N, amax + b);
            gt_split_kernel<<<8 * c->num_sms, 256, 0, c->stream>>>(Ab, M, c->N, Np, nch, amax + b, Pv);
            CK(cudaGetLastError());
            GtArgs ga{};
            ga.P = Pv;
            ga.amax = amax + b;
            ga.out = SymOut{static_cast<__half*>(c->dG), c->dSg, c->nRB, c->ntri};
            ga.b = b;
            ga.N = c->N;
            ga.Np = Np;
            ga.nch = nch;
            ga.I0 = Ib;
            ga.I1 = Ie;
            ga.nRB = c->nRB;
            ga.ntile = ntile;
            ga.round = rounds + b;
            ga.tlog = c->dTl;
            const int grid = (int)std::min<long long>(ntile, c->sched_n());
            gram_tc_kernel<<<grid, kGtThreads, kGtSmem, c->stream>>>(ga);
            CK(cudaGetLastError());
            c->timing.other_launches += 3;
        }
        CK(cudaStreamSynchronize(c->stream));  // P is freed on return
    }
    // one launch per run of equal M (instances of a phase grid differ in M)
    for (int b = 0; b < c->B && !blas;) {
        int e = b;
        while (e < c->B && c->M[e] == c->M[b]) ++e;
        const dim3 grid(nt, nti, e - b);
        const double* Ab = c->dA + (size_t)b * astride;
        if (nti == 0) {
            b = e;
            continue;
        }
        const Sym64Out o64{c->sym64 ? static_cast<double*>(c->dG6) + (size_t)b * c->ntri6 * (kT6 * kT6)
                                    : nullptr,
                           c->nRB6, c->ntri6};
        if (c->sym64) {
            gram128_kernel<<<grid, 256, 0, c->stream>>>(Ab, c->M[b], c->N, astride, o64, bi0, mirror);
        } else if (c->sym) {
            SymOut o{static_cast<__half*>(c->dG) + (size_t)b * c->ntri * 2 * kSyPlaneHalfs,
                     c->dSg + b, c->nRB, c->ntri};
            gram128_kernel<<<grid, 256, 0, c->stream>>>(Ab, c->M[b], c->N, astride, o, bi0, mirror);
        } else if (c->st64()) {
            PanelOut<double, row_block<double>()> o{
                static_cast<double*>(c->dG) + (size_t)b * c->nRB * c->ldJ * c->RB, c->ldJ, c->nRB,
                c->row0};
            gram128_kernel<<<grid, 256, 0, c->stream>>>(Ab, c->M[b], c->N, astride, o, bi0, mirror);
        } else {
            PanelOut<float, row_block<float>()> o{
                static_cast<float*>(c->dG) + (size_t)b * c->nRB * c->ldJ * c->RB, c->ldJ, c->nRB,
                c->row0};
            gram128_kernel<<<grid, 256, 0, c->stream>>>(Ab, c->M[b], c->N, astride, o, bi0, mirror);
        }
        CK(cudaGetLastError());
        b = e;
    }
    cudaEventRecord(ev.ev[1], c->stream);
    CK(cudaStreamSynchronize(c->stream));
    c->timing.gram_ms = ev.ms(0, 1);
    c->timing.other_launches += 2;
    c->built = true;
    return 0;
}

int cimcs_get_coupling(cimcs_ctx* c, int32_t b, double* G, double* hz, double* D) {
    if (!c || !c->built || b < 0 || b >= c->B) return fail(CIMCS_INPUT_ERROR, "bad instance");
    if (c->world > 1 || c->tworld > 1)
        return fail(CIMCS_CONFIG_ERROR, "get_coupling: not on a sharded context");
    const int N = c->N, ld = c->ldN, RB = c->RB, ldJ = c->ldJ;
    const size_t gstride = (size_t)c->nRB * ldJ * RB;
    auto fetch = [&](const void* d, size_t off, size_t n, std::vector<double>& h) -> int {
        h.resize(n);
        if (c->st64()) {
            if (int rc_ = copy_sync(c, h.data(), static_cast<const double*>(d) + off, n * 8,
                                    cudaMemcpyDeviceToHost))
                return rc_;
        } else {
            std::vector<float> f(n);
            if (int rc_ = copy_sync(c, f.data(), static_cast<const float*>(d) + off, n * 4,
                                    cudaMemcpyDeviceToHost))
                return rc_;
            for (size_t k = 0; k < n; ++k) h[k] = f[k];
        }
        return 0;
    };
    std::vector<double> h;
    if (G && c->mri) {  // never stored: the columns G e_r of the transform chain
        float* P = nullptr;
        if (int rc = dalloc(c, &P, (size_t)N * N * 4)) return rc;
        std::unique_ptr<float, decltype(&cudaFree)> pguard(P, &cudaFree);
        if (int rc = c->mri_kind == 1 ? dct_launch(c, DCT_COLS, N, 0, nullptr, P, 1)
                                      : mri_launch(c, MRI_COLS, N, 0, nullptr, P))
            return rc;
        std::vector<float> f((size_t)N * N);
        if (int rc_ = copy_sync(c, f.data(), P, f.size() * 4, cudaMemcpyDeviceToHost)) return rc_;
        for (size_t k = 0; k < f.size(); ++k) G[k] = f[k];
    } else if (G && c->sym64) {
        const size_t nt = (size_t)c->ntri6 * kT6 * kT6;
        std::vector<double> t(nt);
        if (int rc_ = copy_sync(c, t.data(), static_cast<const double*>(c->dG6) + (size_t)b * nt,
                                nt * 8, cudaMemcpyDeviceToHost))
            return rc_;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                int r = i, q = j;  // stored upper triangle: G[i][j] = G[j][i]
                if (r / kT6 > q / kT6) std::swap(r, q);
                G[(size_t)i * N + j] = t[(size_t)sy_tri(r / kT6, q / kT6, c->nRB6) * kT6 * kT6 +
                                         s6_gofs(r % kT6, q % kT6)];
            }
    } else if (G && c->sym) {
        const size_t nh = (size_t)c->ntri * 2 * kSyPlaneHalfs;
        std::vector<__half> t(nh);
        int sg = 0;
        if (int rc_ = copy_sync(c, t.data(), static_cast<const __half*>(c->dG) + (size_t)b * nh,
                                nh * 2, cudaMemcpyDeviceToHost))
            return rc_;
        if (int rc_ = copy_sync(c, &sg, c->dSg + b, 4, cudaMemcpyDeviceToHost)) return rc_;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                int r = i, q = j;  // stored upper triangle: G[i][j] = G[j][i]
                if (r / kSyT > q / kSyT) std::swap(r, q);
                const size_t o = (size_t)sy_tri(r / kSyT, q / kSyT, c->nRB) * 2 * kSyPlaneHalfs +
                                 sy_offk(r % kSyT, q % kSyT, kSyT) / 2;
                const double v = (double)__half2float(t[o]) + (double)__half2float(t[o + kSyPlaneHalfs]);
                G[(size_t)i * N + j] = std::ldexp(v, -sg);
            }
    } else if (G) {
        if (int rc = fetch(c->dG, (size_t)b * gstride, gstride, h)) return rc;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j)
                G[(size_t)i * N + j] = h[((size_t)(i / RB) * ldJ + j) * RB + (i % RB)];
    }
    if (hz) {
        if (int rc = fetch(c->dhz, (size_t)b * ld, N, h)) return rc;
        std::copy(h.begin(), h.end(), hz);
    }
    if (D) {
        if (int rc = fetch(c->dD, (size_t)b * ld, N, h)) return rc;
        std::copy(h.begin(), h.end(), D);
    }
    return 0;
}

}  // extern "C"
