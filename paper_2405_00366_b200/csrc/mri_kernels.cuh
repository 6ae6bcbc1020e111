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
// nothing of the chain touches HBM except w in and G w out.  The FFTs are
// radix-2 over shared memory: the forward transform is decimation-in-
// frequency (natural order in, bit-reversed out), the mask is applied in
// bit-reversed coordinates (pre-permuted on the host), and the inverse is
// decimation-in-time (bit-reversed in, natural out), so no permutation pass
// is ever needed.  G w lands in the slot buffer of the symmetric path
// ([N][NR], one slot) and sym_update_kernel runs the fused MFZ / CG / score
// epilogue on it.
#pragma once

#include <cuda_runtime.h>

namespace cimcs {

constexpr int kMriThreads = 512;
constexpr int kMriMaxPix = 128 * 128;      // shared-memory image cap (192 KB)

enum { MRI_APPLY = 0, MRI_HZ = 1, MRI_DIAG = 2, MRI_COLS = 3 };

struct MriArgs {
    int H, W, N, NR, nact;         // nact: replica slots (or basis vectors) handled
    const unsigned char* mask_br;  // [H*W] sampled?  in bit-reversed (row, col) coordinates
    const float2* tw;              // exp(-2 pi i k / L), k < L / 2, L = max(H, W)
    int L;
    float gamma;
    float scale;                   // 1 / (H W): the two unitary scalings
    const float* in;               // MRI_APPLY: w [N][NR]; MRI_HZ: target image (row-major)
    float* out;                    // MRI_APPLY: G w [N][NR]; MRI_HZ: hz [N]; MRI_DIAG: D [N]
    int r0;                        // MRI_DIAG: first basis vector of this launch
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// One radix-2 stage over every line of the image.  Lines of length n along
// an axis with element stride es (1: rows, W: columns) and line stride ls;
// `half` = butterfly span.  DIF: (a, b) -> (a + b, (a - b) w); DIT with conj
// twiddles: (a, b) -> (a + b w*, a - b w*).
template <bool DIF>
__device__ __forceinline__ void fft_stage(float2* X, int nlines, int n, int es, int ls, int half,
                                          const float2* tw, int L) {
    const int nb = nlines * (n / 2);
    const int tstep = L / (2 * half);
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
        const int line = t / (n / 2), bi = t % (n / 2);
        const int grp = bi / half, pos = bi % half;
        const int i0 = grp * 2 * half + pos;
        float2* p0 = X + (size_t)line * ls + (size_t)i0 * es;
        float2* p1 = p0 + (size_t)half * es;
        const float2 a = *p0, b = *p1, w = tw[pos * tstep];
        if (DIF) {
            *p0 = make_float2(a.x + b.x, a.y + b.y);
            *p1 = cmul(make_float2(a.x - b.x, a.y - b.y), w);
        } else {
            const float2 bw = cmulc(b, w);
            *p0 = make_float2(a.x + bw.x, a.y + bw.y);
            *p1 = make_float2(a.x - bw.x, a.y - bw.y);
        }
    }
    __syncthreads();
}

// Haar level on the first `cnt` lines (stride ls) of length n (element
// stride es): split (forward) or merge (inverse), staged through registers.
// mri.cpp:29-48 (s = 1/sqrt(2), (a + b) s and (a - b) s).
template <bool SPLIT>
__device__ __forceinline__ void haar_pass(float* X, int cnt, int n, int es, int ls) {
    const float s = 0.70710678118654752440f;
    const int np = cnt * (n / 2);
    constexpr int kReg = kMriMaxPix / 2 / kMriThreads;  // pairs per thread (16)
    float ra[kReg], rb[kReg];
#pragma unroll
    for (int u = 0; u < kReg; ++u) {
        const int t = threadIdx.x + u * kMriThreads;
        if (t < np) {
            const int line = t / (n / 2), k = t % (n / 2);
            const float* L = X + (size_t)line * ls;
            float a, b;
            if (SPLIT) {
                a = L[(size_t)(2 * k) * es];
                b = L[(size_t)(2 * k + 1) * es];
            } else {
                a = L[(size_t)k * es];
                b = L[(size_t)(n / 2 + k) * es];
            }
            ra[u] = (a + b) * s;
            rb[u] = (a - b) * s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kReg; ++u) {
        const int t = threadIdx.x + u * kMriThreads;
        if (t < np) {
            const int line = t / (n / 2), k = t % (n / 2);
            float* L = X + (size_t)line * ls;
            if (SPLIT) {
                L[(size_t)k * es] = ra[u];
                L[(size_t)(n / 2 + k) * es] = rb[u];
            } else {
                L[(size_t)(2 * k) * es] = ra[u];
                L[(size_t)(2 * k + 1) * es] = rb[u];
            }
        }
    }
    __syncthreads();
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

// One CTA per replica slot (MRI_APPLY), per basis vector (MRI_DIAG) or the
// single target image (MRI_HZ).
__global__ void __launch_bounds__(kMriThreads, 1) mri_kernel(MriArgs a, int mode) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int H = a.H, W = a.W, N = a.N;
    float2* K = reinterpret_cast<float2*>(smem);          // [H][W] complex
    float* B = reinterpret_cast<float*>(K + N);           // [H][W] real
    float2* tw = reinterpret_cast<float2*>(B + N);        // [L / 2]
    const int q = blockIdx.x;
    for (int k = threadIdx.x; k < a.L / 2; k += blockDim.x) tw[k] = a.tw[k];
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
    if (mode != MRI_HZ) {
        // inverse Haar, deepest level first: columns then rows (mri.cpp:143-165)
        int nl = 0;
        for (int h = H, w = W; h >= 2 && w >= 2; h /= 2, w /= 2) ++nl;
        for (int l = nl - 1; l >= 0; --l) {
            const int h = H >> l, w = W >> l;
            haar_pass<false>(B, w, h, W, 1);  // columns j < w, length h
            haar_pass<false>(B, h, w, 1, W);  // rows i < h, length w
        }
    }
    // ---- forward unitary DFT (scale folded into the mask step): DIF rows, DIF columns
    for (int i = threadIdx.x; i < N; i += blockDim.x) K[i] = make_float2(B[i], 0.f);
    __syncthreads();
    for (int half = W / 2; half >= 1; half /= 2) fft_stage<true>(K, H, W, 1, W, half, tw, a.L);
    for (int half = H / 2; half >= 1; half /= 2) fft_stage<true>(K, W, H, W, 1, half, tw, a.L);
    // ---- mask (bit-reversed coordinates) and the two unitary scalings
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const float m = a.mask_br[i] ? a.scale : 0.f;
        K[i] = make_float2(K[i].x * m, K[i].y * m);
    }
    __syncthreads();
    // ---- inverse DFT: DIT rows, DIT columns (bit-reversed in, natural out)
    for (int half = 1; half < W; half *= 2) fft_stage<false>(K, H, W, 1, W, half, tw, a.L);
    for (int half = 1; half < H; half *= 2) fft_stage<false>(K, W, H, W, 1, half, tw, a.L);
    // ---- real part + gamma * (D2c D2c + D2r D2r) of the Haar image, into B
    {
        constexpr int kPer = kMriMaxPix / kMriThreads;
        float v[kPer];
        const bool smooth = mode != MRI_HZ && a.gamma > 0.f;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int p = threadIdx.x + u * kMriThreads;
            if (p < N) {
                float x = K[p].x;
                if (smooth) {
                    const int i = p / W, j = p % W;
                    x += a.gamma * (d4(B + j, i, H, W) + d4(B + (size_t)i * W, j, W, 1));
                }
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
    // ---- forward Haar: rows then columns per level (mri.cpp:122-141)
    for (int h = H, w = W; h >= 2 && w >= 2; h /= 2, w /= 2) {
        haar_pass<true>(B, h, w, 1, W);
        haar_pass<true>(B, w, h, W, 1);
    }
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

inline size_t mri_smem_bytes(int N, int L) { return (size_t)N * 12 + (size_t)(L / 2) * 8; }

}  // namespace cimcs
