// mri_kernels.cuh -- matrix-free MRI coupling.
//
// The reference's transform-chain problem (mri.hpp:46-99, mri.cpp:209-315)
// never forms its N x N quadratic form
//     G = Re(A^H A) + gamma * Psi (Dv^T Dv + Dh^T Dh) Psi^T,   A = S F Psi^T
// (S: k-space mask, F: unitary 2-D DFT, Psi: orthonormal multi-level Haar in
// the Mallat layout, Dv / Dh: second differences with reflective ends): every
// apply_full(w) is inverse Haar -> FFT -> mask -> inverse FFT -> real part
// (+ gamma * fourth-difference smoothness of the Haar image) -> forward Haar.
// On the B200 one CTA owns one replica's whole image in shared memory
// (H x W complex fp32 = 128 KB at 128 x 128, plus the real Haar image):
// nothing of the chain touches HBM except w in and G w out.  Each 1-D FFT
// line lives in one warp's registers (4 elements per lane at 128 points,
// butterflies across lanes by shuffles): a 2-D transform is two passes over
// shared memory with one barrier each.  The forward transform is decimation-
// in-frequency (natural order in, bit-reversed out), the mask is applied in
// bit-reversed coordinates (pre-permuted on the host), and the inverse is
// decimation-in-time (bit-reversed in, natural out), so no permutation pass
// is ever needed.  G w lands in the slot buffer of the symmetric path
// ([N][NR], one slot) and sym_update_kernel runs the fused MFZ / CG / score
// epilogue on it.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

namespace cimcs {

constexpr int kMriThreads = 1024;
constexpr int kMriWarps = kMriThreads / 32;
constexpr int kMriMaxPix = 128 * 128;      // shared-memory image cap (~194 KB)
constexpr int kMriMaxLine = 128;           // longest FFT line (4 elements per lane)

enum { MRI_APPLY = 0, MRI_HZ = 1, MRI_DIAG = 2, MRI_COLS = 3 };

struct MriArgs {
    int H, W, N, NR, nact;         // nact: replica slots (or basis vectors) handled
    const unsigned char* mask_br;  // [H*W] sampled?  in bit-reversed (row, col) coordinates
    const float2* tw;              // exp(-2 pi i k / 128), k < 64 (every line length <= 128)
    int L;
    float gamma;
    float scale;                   // 1 / (H W): the two unitary scalings
    const float* in;               // MRI_APPLY: w [N][NR]; MRI_HZ: target image (row-major)
    float* out;                    // MRI_APPLY: G w [N][NR]; MRI_HZ: hz [N]; MRI_DIAG: D [N]; MRI_COLS: G rows
    int r0;                        // MRI_DIAG / MRI_COLS: first basis vector of this launch
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ float2 shfl2(float2 v, int m) {
    return make_float2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// One FFT pass over every line of the (padded) image, a warp per line held in
// registers: lines of length n = 2^LN (2 <= n <= 128) along an axis with
// element stride es and line stride ls.  n >= 32: element p = lane + 32 k
// (k < n / 32) of one line per lane; n < 32: 32 / n lines per warp, lane
// groups of n.  Butterfly spans >= 32 pair registers of a lane, spans < 32
// pair lanes (shuffles), so the whole transform needs no barrier; every
// lane's twiddles are loaded once per pass (tw = exp(-2 pi i k / 128)).
// DIF (forward): natural order in, bit-reversed out, (a, b) -> (a + b, (a - b) w);
// DIT (inverse, conj twiddles): bit-reversed in, natural out,
// (a, b) -> (a + b w*, a - b w*).  w = exp(-2 pi i pos / (2 span)).
template <bool DIF, int LN>
__device__ __noinline__ void fft_pass_t(float2* X, int nlines, int es, int ls,
                                        const float2* tw) {  // one copy per call site kind: i-cache
    constexpr int n = 1 << LN;
    constexpr int E = n >= 32 ? n / 32 : 1;          // elements per lane
    constexpr int G = n >= 32 ? 1 : 32 / n;          // lines per warp
    constexpr int LS = LN < 5 ? LN : 5;              // lane stages
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int p0 = lane & (n >= 32 ? 31 : n - 1);    // position of element 0
    // twiddles: lane stage s has span 2^s; register stage hk has span 32 hk
    float2 wl[LS > 0 ? LS : 1];
#pragma unroll
    for (int s2 = 0; s2 < LS; ++s2) {
        const int half = 1 << s2;
        wl[s2] = tw[(p0 & (half - 1)) * (64 >> s2)];
    }
    float2 wr1 = make_float2(1.f, 0.f), wr2a = wr1, wr2b = wr1;
    if constexpr (E >= 2) wr1 = tw[lane * 2];            // span 32: pos = lane
    if constexpr (E >= 4) {                               // span 64: pos = lane + 32 (k & 1)
        wr2a = tw[lane];
        wr2b = tw[lane + 32];
    }
    const int nwarps = blockDim.x >> 5;
    for (int l0 = warp * G; l0 < nlines; l0 += nwarps * G) {
        const int line = l0 + (n >= 32 ? 0 : lane >> LN);
        const bool on = line < nlines;
        float2* base = X + (size_t)(on ? line : 0) * ls;
        float2 v[E];
#pragma unroll
        for (int k = 0; k < E; ++k)
            v[k] = on ? base[(size_t)(p0 + 32 * k) * es] : make_float2(0.f, 0.f);
        auto lane_stage = [&](int s2) {
            const int half = 1 << s2;
            const float2 w = wl[s2];
            const bool upper = (p0 & half) != 0;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const float2 o = shfl2(v[k], half);
                if (DIF) {
                    v[k] = upper ? cmul(make_float2(o.x - v[k].x, o.y - v[k].y), w)
                                 : make_float2(v[k].x + o.x, v[k].y + o.y);
                } else {
                    const float2 bw = cmulc(upper ? v[k] : o, w);
                    v[k] = upper ? make_float2(o.x - bw.x, o.y - bw.y)
                                 : make_float2(v[k].x + bw.x, v[k].y + bw.y);
                }
            }
        };
        auto reg_bfly = [&](int k0, int k1, float2 w) {
            const float2 a = v[k0], b = v[k1];
            if (DIF) {
                v[k0] = make_float2(a.x + b.x, a.y + b.y);
                v[k1] = cmul(make_float2(a.x - b.x, a.y - b.y), w);
            } else {
                const float2 bw = cmulc(b, w);
                v[k0] = make_float2(a.x + bw.x, a.y + bw.y);
                v[k1] = make_float2(a.x - bw.x, a.y - bw.y);
            }
        };
        if (DIF) {
            if constexpr (E >= 4) {
                reg_bfly(0, 2, wr2a);
                reg_bfly(1, 3, wr2b);
            }
            if constexpr (E >= 2) {
#pragma unroll
                for (int k = 0; k < E; k += 2) reg_bfly(k, k + 1, wr1);
            }
#pragma unroll
            for (int s2 = LS - 1; s2 >= 0; --s2) lane_stage(s2);
        } else {
#pragma unroll
            for (int s2 = 0; s2 < LS; ++s2) lane_stage(s2);
            if constexpr (E >= 2) {
#pragma unroll
                for (int k = 0; k < E; k += 2) reg_bfly(k, k + 1, wr1);
            }
            if constexpr (E >= 4) {
                reg_bfly(0, 2, wr2a);
                reg_bfly(1, 3, wr2b);
            }
        }
        if (on) {
#pragma unroll
            for (int k = 0; k < E; ++k) base[(size_t)(p0 + 32 * k) * es] = v[k];
        }
    }
    __syncthreads();
}

template <bool DIF>
__device__ __forceinline__ void fft_pass(float2* X, int nlines, int ln, int es, int ls,
                                         const float2* tw) {
    switch (ln) {
        case 1: fft_pass_t<DIF, 1>(X, nlines, es, ls, tw); break;
        case 2: fft_pass_t<DIF, 2>(X, nlines, es, ls, tw); break;
        case 3: fft_pass_t<DIF, 3>(X, nlines, es, ls, tw); break;
        case 4: fft_pass_t<DIF, 4>(X, nlines, es, ls, tw); break;
        case 5: fft_pass_t<DIF, 5>(X, nlines, es, ls, tw); break;
        case 6: fft_pass_t<DIF, 6>(X, nlines, es, ls, tw); break;
        default: fft_pass_t<DIF, 7>(X, nlines, es, ls, tw); break;
    }
}

// One whole Haar level on the leading 2^lh x 2^lw block as 2 x 2 butterflies
// (row width 2^lW).  Forward = the reference's row split then column split
// (mri.cpp:122-141): block (2a..2a+1, 2b..2b+1) -> (a, b), (a, w/2 + b),
// (h/2 + a, b), (h/2 + a, w/2 + b), with the row sums rounded first exactly as
// the two-pass order does; inverse = column merge then row merge
// (mri.cpp:143-165).  Register-staged: all reads, barrier, all writes.
template <bool FWD, int NT>
__device__ __forceinline__ void haar_level(float* X, int lh, int lw, int lW) {
    const float s = 0.70710678118654752440f;
    const int h2 = 1 << (lh - 1), w2 = 1 << (lw - 1), nb = h2 << (lw - 1);
    constexpr int kReg = kMriMaxPix / 4 / NT;  // blocks per thread
    float o[kReg][4];
#pragma unroll
    for (int u = 0; u < kReg; ++u) {
        const int t = threadIdx.x + u * NT;
        if (t < nb) {
            const int aa = t >> (lw - 1), bb = t & (w2 - 1);
            if (FWD) {
                const float* r0 = X + ((size_t)(2 * aa) << lW) + 2 * bb;
                const float* r1 = r0 + ((size_t)1 << lW);
                const float x00 = r0[0], x01 = r0[1], x10 = r1[0], x11 = r1[1];
                const float p0 = (x00 + x01) * s, p1 = (x00 - x01) * s;  // row split, row 2a
                const float q0 = (x10 + x11) * s, q1 = (x10 - x11) * s;  // row split, row 2a+1
                o[u][0] = (p0 + q0) * s;  // (a, b)
                o[u][1] = (p1 + q1) * s;  // (a, w/2 + b)
                o[u][2] = (p0 - q0) * s;  // (h/2 + a, b)
                o[u][3] = (p1 - q1) * s;  // (h/2 + a, w/2 + b)
            } else {
                const float* t0 = X + ((size_t)aa << lW);
                const float* t1 = X + ((size_t)(h2 + aa) << lW);
                const float LL = t0[bb], HL = t0[w2 + bb], LH = t1[bb], HH = t1[w2 + bb];
                const float c00 = (LL + LH) * s, c10 = (LL - LH) * s;  // column merge
                const float c01 = (HL + HH) * s, c11 = (HL - HH) * s;
                o[u][0] = (c00 + c01) * s;  // (2a, 2b)
                o[u][1] = (c00 - c01) * s;  // (2a, 2b + 1)
                o[u][2] = (c10 + c11) * s;  // (2a + 1, 2b)
                o[u][3] = (c10 - c11) * s;  // (2a + 1, 2b + 1)
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kReg; ++u) {
        const int t = threadIdx.x + u * NT;
        if (t < nb) {
            const int aa = t >> (lw - 1), bb = t & (w2 - 1);
            if (FWD) {
                float* t0 = X + ((size_t)aa << lW);
                float* t1 = X + ((size_t)(h2 + aa) << lW);
                t0[bb] = o[u][0];
                t0[w2 + bb] = o[u][1];
                t1[bb] = o[u][2];
                t1[w2 + bb] = o[u][3];
            } else {
                float* r0 = X + ((size_t)(2 * aa) << lW) + 2 * bb;
                float* r1 = r0 + ((size_t)1 << lW);
                r0[0] = o[u][0];
                r0[1] = o[u][1];
                r1[0] = o[u][2];
                r1[1] = o[u][3];
            }
        }
    }
    __syncthreads();
}

// full multi-level transforms of an H x W image (H = 2^lH, W = 2^lW)
template <int NT>
__device__ __forceinline__ void haar_inverse(float* X, int lH, int lW) {
    for (int l = min(lH, lW) - 1; l >= 0; --l) haar_level<false, NT>(X, lH - l, lW - l, lW);
}
template <int NT>
__device__ __forceinline__ void haar_forward(float* X, int lH, int lW) {
    for (int lh = lH, lw = lW; lh >= 1 && lw >= 1; --lh, --lw) haar_level<true, NT>(X, lh, lw, lW);
}

// second difference along an axis with reflective ends (mri.cpp:51-63):
// element k of a line x of length n, stride es
__device__ __forceinline__ float d2(const float* x, int k, int n, int es) {
    if (n == 1) return 0.f;
    if (k == 0) return x[es] - x[0];
    if (k == n - 1) return x[(size_t)(n - 2) * es] - x[(size_t)(n - 1) * es];
    return x[(size_t)(k - 1) * es] - 2.f * x[(size_t)k * es] + x[(size_t)(k + 1) * es];
}
// D2(D2(x)) at k, the inner D2 evaluated on the fly
__device__ __forceinline__ float d4(const float* x, int k, int n, int es) {
    if (n == 1) return 0.f;
    if (k == 0) return d2(x, 1, n, es) - d2(x, 0, n, es);
    if (k == n - 1) return d2(x, n - 2, n, es) - d2(x, n - 1, n, es);
    return d2(x, k - 1, n, es) - 2.f * d2(x, k, n, es) + d2(x, k + 1, n, es);
}

// One CTA per replica slot (MRI_APPLY), per basis vector (MRI_DIAG /
// MRI_COLS) or the single target image (MRI_HZ).  Shared memory: the complex
// image with rows padded to W + 1 (column FFT lines hit distinct banks), the
// real Haar image, the twiddles.
__global__ void __launch_bounds__(kMriThreads, 1) mri_kernel(MriArgs a, int mode) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int H = a.H, W = a.W, N = a.N, KS = W + 1;
    float2* K = reinterpret_cast<float2*>(smem);          // [H][W + 1] complex
    float* B = reinterpret_cast<float*>(K + (size_t)H * KS);  // [H][W] real
    float2* tw = reinterpret_cast<float2*>(B + N);        // [64]
    const int q = blockIdx.x;
    const int lH = __ffs(H) - 1, lW = __ffs(W) - 1, wm = W - 1;
    for (int k = threadIdx.x; k < 64; k += blockDim.x) tw[k] = a.tw[k];
    // ---- input: Haar coefficients (or the target image for hz)
    if (mode == MRI_APPLY) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) B[i] = a.in[(size_t)i * a.NR + q];
    } else if (mode == MRI_DIAG || mode == MRI_COLS) {
        const int r = a.r0 + q;
        for (int i = threadIdx.x; i < N; i += blockDim.x) B[i] = i == r ? 1.f : 0.f;
    } else {
        for (int i = threadIdx.x; i < N; i += blockDim.x) B[i] = a.in[i];
    }
    __syncthreads();
    if (mode != MRI_HZ) haar_inverse<kMriThreads>(B, lH, lW);  // mri.cpp:143-165
    // ---- forward DFT (unitary scale folded into the mask step): DIF rows, DIF columns
    for (int p = threadIdx.x; p < N; p += blockDim.x)
        K[(size_t)(p >> lW) * KS + (p & wm)] = make_float2(B[p], 0.f);
    __syncthreads();
    fft_pass<true>(K, H, lW, 1, KS, tw);
    fft_pass<true>(K, W, lH, KS, 1, tw);
    // ---- mask (bit-reversed coordinates) and the two unitary scalings
    for (int p = threadIdx.x; p < N; p += blockDim.x) {
        const float m = a.mask_br[p] ? a.scale : 0.f;
        float2& z = K[(size_t)(p >> lW) * KS + (p & wm)];
        z = make_float2(z.x * m, z.y * m);
    }
    __syncthreads();
    // ---- inverse DFT: DIT rows, DIT columns (bit-reversed in, natural out)
    fft_pass<false>(K, H, lW, 1, KS, tw);
    fft_pass<false>(K, W, lH, KS, 1, tw);
    // ---- real part + gamma * (D2c D2c + D2r D2r) of the Haar image, into B
    {
        constexpr int kPer = kMriMaxPix / kMriThreads;
        float v[kPer];
        const bool smooth = mode != MRI_HZ && a.gamma > 0.f;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int p = threadIdx.x + u * kMriThreads;
            if (p < N) {
                const int i = p >> lW, j = p & wm;
                float x = K[(size_t)i * KS + j].x;
                if (smooth) x += a.gamma * (d4(B + j, i, H, W) + d4(B + ((size_t)i << lW), j, W, 1));
                v[u] = x;
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int p = threadIdx.x + u * kMriThreads;
            if (p < N) B[p] = v[u];
        }
        __syncthreads();
    }
    // ---- forward Haar (mri.cpp:122-141)
    haar_forward<kMriThreads>(B, lH, lW);
    if (mode == MRI_APPLY) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) a.out[(size_t)i * a.NR + q] = B[i];
    } else if (mode == MRI_DIAG) {
        if (threadIdx.x == 0) a.out[a.r0 + q] = B[a.r0 + q];
    } else if (mode == MRI_COLS) {  // column r0 + q of G (= row: G is symmetric)
        for (int i = threadIdx.x; i < N; i += blockDim.x) a.out[(size_t)(a.r0 + q) * N + i] = B[i];
    } else {
        for (int i = threadIdx.x; i < N; i += blockDim.x) a.out[i] = B[i];
    }
}

// ------------------------------------------------ cluster-distributed apply
// The per-step G w of MRI_APPLY on a thread-block cluster of CS = 8 CTAs per
// replica (H, W >= 16), so the 16 replicas of config 3 occupy 128 SMs instead
// of 16.  CTA k owns image rows [r0, r0 + RH) (RH = H / 8, even) and k-space
// columns [c0, c0 + CW) (CW = W / 8).  The Haar transform's first level is a
// 2 x 2 butterfly whose row pairs never straddle two CTAs, and every deeper
// level lives in the (H/2) x (W/2) low-pass quadrant:
//   1. the quadrant's coefficients are inverse-transformed redundantly in
//      every CTA (levels 2.., 1/4 of the work); the level-1 inverse is done
//      only for the CTA's rows and a two-row halo (the smoothness stencil's
//      reach), straight from the detail coefficients in global memory;
//   2. DIF FFT of the own rows; the slab is scattered by column ownership
//      into the peers' column slabs (DSMEM), cluster barrier;
//   3. DIF FFT of the own columns, mask x 1/(HW), DIT inverse, gathered back
//      by row ownership (DSMEM), cluster barrier;
//   4. DIT inverse of the own rows, real part + gamma * fourth differences;
//   5. level-1 forward Haar of the own rows: the detail quadrants are final
//      and go straight to global memory, the low-pass rows are broadcast into
//      every CTA's quadrant (DSMEM), cluster barrier, levels 2.. redundantly,
//      each CTA stores its share of the quadrant.
constexpr int kMriCThreads = 512;
constexpr int kMriCluster = 8;

inline int mri_cluster_size(int H, int W) { return std::min(kMriCluster, std::min(H, W)); }
inline size_t mri_cluster_smem_bytes(int H, int W) {
    const int RH = H / kMriCluster, CW = W / kMriCluster;
    return (size_t)(H / 2) * (W / 2) * 4     // low-pass quadrant
           + (size_t)(RH + 4) * W * 4        // inverse-Haar rows + halo
           + (size_t)RH * W * 4              // result rows
           + (size_t)RH * (W + 1) * 8        // own rows, complex
           + (size_t)H * (CW + 1) * 8        // own columns, complex
           + 64 * 8;
}

__global__ void __launch_bounds__(kMriCThreads, 1) mri_cluster_kernel(MriArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(1024) unsigned char smem[];
    const int H = a.H, W = a.W, NR = a.NR;
    const int CS = kMriCluster, k = (int)cl.block_rank();
    const int lH = __ffs(H) - 1, lW = __ffs(W) - 1;
    const int RH = H >> 3, CW = W >> 3, lRH = lH - 3, lCW = lW - 3;
    const int H2 = H >> 1, W2 = W >> 1, lW2 = lW - 1;
    const int RS = W + 1, CSt = CW + 1;
    const int r0 = k * RH, c0 = k * CW;
    const int s0 = max(0, r0 - 2), s1 = min(H, r0 + RH + 2);      // rows of Bs
    float* Q = reinterpret_cast<float*>(smem);                       // [H/2][W/2]
    float* Bs = Q + (size_t)H2 * W2;                                 // [RH + 4][W]
    float* Rr = Bs + (size_t)(RH + 4) * W;                           // [RH][W]
    float2* Kr = reinterpret_cast<float2*>(Rr + (size_t)RH * W);     // [RH][W + 1]
    float2* Kc = Kr + (size_t)RH * RS;                               // [H][CW + 1]
    float2* tw = Kc + (size_t)H * CSt;                               // [64]
    float* Bv = Bs - (size_t)s0 * W;  // virtual full image: rows [s0, s1) valid
    const int q = blockIdx.x / CS;
    const float* win = a.in;
    const float s = 0.70710678118654752440f;
    // arrival barriers of the three exchanges (st.async ... complete_tx): a CTA
    // proceeds as soon as ITS inputs have landed, no cluster-wide barrier
    __shared__ __align__(8) uint64_t mb[3];  // column slab, row slab, low-pass quadrant
    if (threadIdx.x == 0) {
        for (int e = 0; e < 3; ++e) mbar_init(&mb[e], 1);
        mbar_fence_init();
        mbar_arrive_expect_tx(&mb[0], (uint32_t)(H * CW * 8));
        mbar_arrive_expect_tx(&mb[1], (uint32_t)(RH * W * 8));
        mbar_arrive_expect_tx(&mb[2], (uint32_t)(H2 * W2 * 4));
    }
    for (int t = threadIdx.x; t < 64; t += blockDim.x) tw[t] = a.tw[t];
    cl.sync();  // every CTA's barriers are armed before any peer stores into it
    // programmatic dependent launch: the update kernel may be scheduled now; this
    // grid's reads of w wait for the previous step's update kernel
    sy_pdl_trigger();
    sy_pdl_wait();
    // 1. low-pass quadrant (redundant), levels 2.. of the inverse
    for (int t = threadIdx.x; t < H2 * W2; t += blockDim.x) {
        const int i = t >> lW2, j = t & (W2 - 1);
        Q[t] = win[((size_t)(i << lW) + j) * NR + q];
    }
    __syncthreads();
    haar_inverse<kMriCThreads>(Q, lH - 1, lW - 1);
    // level-1 inverse (column merge, then row merge) for rows [s0, s1)
    for (int t = threadIdx.x; t < ((s1 - s0) >> 1) * W2; t += blockDim.x) {
        const int aa = (s0 >> 1) + (t >> lW2), bb = t & (W2 - 1);
        const float LL = Q[(aa << lW2) + bb];
        const float HL = win[((size_t)(aa << lW) + W2 + bb) * NR + q];
        const float LH = win[((size_t)((H2 + aa) << lW) + bb) * NR + q];
        const float HH = win[((size_t)((H2 + aa) << lW) + W2 + bb) * NR + q];
        const float c00 = (LL + LH) * s, c10 = (LL - LH) * s;
        const float c01 = (HL + HH) * s, c11 = (HL - HH) * s;
        float* o0 = Bv + ((size_t)(2 * aa) << lW) + 2 * bb;
        float* o1 = o0 + W;
        o0[0] = (c00 + c01) * s;
        o0[1] = (c00 - c01) * s;
        o1[0] = (c10 + c11) * s;
        o1[1] = (c10 - c11) * s;
    }
    __syncthreads();
    // 2. DIF rows, scatter to the column owners
    for (int t = threadIdx.x; t < RH * W; t += blockDim.x)
        Kr[(size_t)(t >> lW) * RS + (t & (W - 1))] = make_float2(Bv[((size_t)r0 << lW) + t], 0.f);
    __syncthreads();
    fft_pass<true>(Kr, RH, lW, 1, RS, tw);
    for (int t = threadIdx.x; t < RH * W; t += blockDim.x) {
        const int r = t >> lW, j = t & (W - 1), m = j >> lCW;
        const float2 v = Kr[(size_t)r * RS + j];
        cl_st_async8(cl_mapa(smem_u32(Kc + (size_t)(r0 + r) * CSt + (j & (CW - 1))), m),
                     *reinterpret_cast<const uint64_t*>(&v), cl_mapa(smem_u32(&mb[0]), m));
    }
    cl_wait(&mb[0], 0);
    // 3. DIF columns, mask, DIT columns, gather back to the row owners
    fft_pass<true>(Kc, CW, lH, CSt, 1, tw);
    for (int t = threadIdx.x; t < H * CW; t += blockDim.x) {
        const int i = t >> lCW, jl = t & (CW - 1);
        const float m = a.mask_br[((size_t)i << lW) + c0 + jl] ? a.scale : 0.f;
        float2& z = Kc[(size_t)i * CSt + jl];
        z = make_float2(z.x * m, z.y * m);
    }
    __syncthreads();
    fft_pass<false>(Kc, CW, lH, CSt, 1, tw);
    for (int t = threadIdx.x; t < H * CW; t += blockDim.x) {
        const int i = t >> lCW, jl = t & (CW - 1), m = i >> lRH;
        const float2 v = Kc[(size_t)i * CSt + jl];
        cl_st_async8(cl_mapa(smem_u32(Kr + (size_t)(i & (RH - 1)) * RS + c0 + jl), m),
                     *reinterpret_cast<const uint64_t*>(&v), cl_mapa(smem_u32(&mb[1]), m));
    }
    cl_wait(&mb[1], 0);
    // 4. DIT rows; real part + smoothness
    fft_pass<false>(Kr, RH, lW, 1, RS, tw);
    const bool smooth = a.gamma > 0.f;
    for (int t = threadIdx.x; t < RH * W; t += blockDim.x) {
        const int i = r0 + (t >> lW), j = t & (W - 1);
        float x = Kr[(size_t)(t >> lW) * RS + j].x;
        if (smooth) x += a.gamma * (d4(Bv + j, i, H, W) + d4(Bv + ((size_t)i << lW), j, W, 1));
        Rr[t] = x;
    }
    __syncthreads();
    // 5. level-1 forward of the own rows (row split, then column split)
    for (int t = threadIdx.x; t < (RH >> 1) * W2; t += blockDim.x) {
        const int al = t >> lW2, bb = t & (W2 - 1), aa = (r0 >> 1) + al;
        const float* p = Rr + ((size_t)(2 * al) << lW) + 2 * bb;
        const float x00 = p[0], x01 = p[1], x10 = p[W], x11 = p[W + 1];
        const float p0 = (x00 + x01) * s, p1 = (x00 - x01) * s;
        const float q0 = (x10 + x11) * s, q1 = (x10 - x11) * s;
        const float LL = (p0 + q0) * s;
        a.out[((size_t)(aa << lW) + W2 + bb) * NR + q] = (p1 + q1) * s;          // HL
        a.out[((size_t)((H2 + aa) << lW) + bb) * NR + q] = (p0 - q0) * s;        // LH
        a.out[((size_t)((H2 + aa) << lW) + W2 + bb) * NR + q] = (p1 - q1) * s;   // HH
        const uint32_t dst = smem_u32(Q + (aa << lW2) + bb), bar = smem_u32(&mb[2]);
        for (int m = 0; m < CS; ++m)
            cl_st_async4(cl_mapa(dst, m), __float_as_uint(LL), cl_mapa(bar, m));
    }
    cl_wait(&mb[2], 0);
    haar_forward<kMriCThreads>(Q, lH - 1, lW - 1);
    for (int t = threadIdx.x; t < (RH >> 1) * W2; t += blockDim.x) {
        const int idx = ((r0 >> 1) << lW2) + t, i = idx >> lW2, j = idx & (W2 - 1);
        a.out[((size_t)(i << lW) + j) * NR + q] = Q[idx];
    }
}

// ---------------------------------------------------------------- LASSO
// lasso_normal_form (mri.cpp:345-370) as used by lasso_init(t, lambda)
// (mri.cpp:372-377): FISTA on 1/2 x'Gx - hz.x + lambda |x|_1 with
// G = Re(A^H A) (the chain without smoothness), step 1.  Each iteration is
// one mri_kernel launch over the two slots [z | x] followed by this
// one-CTA kernel: it first evaluates the objective of the x produced by the
// previous update (its G x is the second slot) and stops on the reference's
// test |f - f_prev| <= tol max(1, |f_prev|) (f_prev starts at 0) or after
// max_iters updates; otherwise it applies the next update.  Reductions are
// in fp64 in a fixed order.
struct LassoState {
    double t, f_prev, f;
    int it, done;
};

constexpr int kLassoThreads = 1024;

__global__ void __launch_bounds__(kLassoThreads) lasso_kernel(
    const float* __restrict__ Gzx,  // [N][2]: G z, G x
    float* __restrict__ zx,         // [N][2]: z, x (the next apply's input)
    const float* __restrict__ hz, int N, double lambda, double step, double tol,
    int max_iters, LassoState* st) {
    __shared__ double red[3][kLassoThreads / 32];
    __shared__ int s_stop;
    if (st->done) return;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int it = st->it;
    if (it >= 1) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int i = tid; i < N; i += kLassoThreads) {
            const double x = zx[2 * i + 1];
            a += x * (double)Gzx[2 * i + 1];
            b += (double)hz[i] * x;
            c += fabs(x);
        }
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (lane == 0) {
            red[0][wid] = a;
            red[1][wid] = b;
            red[2][wid] = c;
        }
        __syncthreads();
        if (tid == 0) {
            double A = 0.0, Bv = 0.0, Cv = 0.0;
            for (int w = 0; w < kLassoThreads / 32; ++w) {
                A += red[0][w];
                Bv += red[1][w];
                Cv += red[2][w];
            }
            const double f = 0.5 * A - Bv + lambda * Cv;
            const double fp = st->f_prev;
            int stop = fabs(f - fp) <= tol * fmax(1.0, fabs(fp)) || it >= max_iters;
            st->f = f;
            st->f_prev = f;
            if (stop) st->done = 1;
            s_stop = stop;
        }
        __syncthreads();
        if (s_stop) return;
    }
    const double t = st->t, tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t)), mom = (t - 1.0) / tn;
    const double thr = step * lambda;
    for (int i = tid; i < N; i += kLassoThreads) {
        const double z = zx[2 * i], x = zx[2 * i + 1];
        const double g = (double)Gzx[2 * i] - (double)hz[i];
        const double v = z - step * g, m = fabs(v) - thr;
        const double xn = m > 0.0 ? (v > 0.0 ? m : -m) : 0.0;  // soft_threshold, mri.cpp:67-74
        zx[2 * i] = (float)(xn + mom * (xn - x));
        zx[2 * i + 1] = (float)xn;
    }
    __syncthreads();
    if (tid == 0) {
        st->t = tn;
        st->it = it + 1;
    }
}

inline size_t mri_smem_bytes(int H, int W, int L) {
    return (size_t)H * (W + 1) * 8 + (size_t)H * W * 4 + 64 * 8;
}

}  // namespace cimcs
