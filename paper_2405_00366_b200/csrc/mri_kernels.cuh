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

#include <cuda_runtime.h>

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
__device__ __forceinline__ void fft_pass_t(float2* X, int nlines, int es, int ls,
                                           const float2* tw) {
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
    for (int l0 = warp * G; l0 < nlines; l0 += kMriWarps * G) {
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

// Haar level on the first 2^lcnt lines of length 2^ln: split (forward) or merge
// (inverse), staged through registers (mri.cpp:29-48: s = 1/sqrt(2),
// (a + b) s and (a - b) s).  cols: lines are columns (stride W) and the line
// index runs fastest across threads, so a warp touches consecutive columns.
template <bool SPLIT>
__device__ __forceinline__ void haar_pass(float* X, int lcnt, int ln, int lW, bool cols) {
    const float s = 0.70710678118654752440f;
    const int n = 1 << ln, np = 1 << (lcnt + ln - 1), hm = (n >> 1) - 1, cm = (1 << lcnt) - 1;
    constexpr int kReg = kMriMaxPix / 2 / kMriThreads;  // pairs per thread (8)
    float ra[kReg], rb[kReg];
    auto at = [&](int line, int k) -> float* {
        return cols ? X + ((size_t)k << lW) + line : X + ((size_t)line << lW) + k;
    };
#pragma unroll
    for (int u = 0; u < kReg; ++u) {
        const int t = threadIdx.x + u * kMriThreads;
        if (t < np) {
            const int line = cols ? t & cm : t >> (ln - 1), k = cols ? t >> lcnt : t & hm;
            const float a = SPLIT ? *at(line, 2 * k) : *at(line, k);
            const float b = SPLIT ? *at(line, 2 * k + 1) : *at(line, (n >> 1) + k);
            ra[u] = (a + b) * s;
            rb[u] = (a - b) * s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kReg; ++u) {
        const int t = threadIdx.x + u * kMriThreads;
        if (t < np) {
            const int line = cols ? t & cm : t >> (ln - 1), k = cols ? t >> lcnt : t & hm;
            if (SPLIT) {
                *at(line, k) = ra[u];
                *at(line, (n >> 1) + k) = rb[u];
            } else {
                *at(line, 2 * k) = ra[u];
                *at(line, 2 * k + 1) = rb[u];
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
    if (mode != MRI_HZ) {
        // inverse Haar, deepest level first: columns then rows (mri.cpp:143-165)
        const int nl = min(lH, lW);
        for (int l = nl - 1; l >= 0; --l) {
            const int lh = lH - l, lw = lW - l;
            haar_pass<false>(B, lw, lh, lW, true);   // columns j < w, length h
            haar_pass<false>(B, lh, lw, lW, false);  // rows i < h, length w
        }
    }
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
    // ---- forward Haar: rows then columns per level (mri.cpp:122-141)
    for (int lh = lH, lw = lW; lh >= 1 && lw >= 1; --lh, --lw) {
        haar_pass<true>(B, lh, lw, lW, false);
        haar_pass<true>(B, lw, lh, lW, true);
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
