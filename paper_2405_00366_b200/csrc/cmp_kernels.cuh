// cmp_kernels.cuh -- the compacted Jacobi refit of the fp32 symmetric path.
//
// cdp_minimize (cdp.cpp:132-139) only touches the active spins: the refit of
// a trajectory is damped Jacobi on G[act, act] (`jacobi_solve` :48-64) and an
// inactive spin's R is kept bitwise (:109-120).  All R replicas of an instance
// share its gram, so per alternation the refit runs on the UNION U_b of the
// replicas' supports (config 1: |U| ~ 0.39 N): the union's rows / columns of the
// stored fp16 hi/lo tiles are gathered into a compacted symmetric tile set
// (padded to the largest union of the batch), the state (R, sigma, D, hz) is
// gathered, the unchanged symmetric-tile kernels run the 100 sweeps on the
// compacted problem (~(|U| / N)^2 of the bytes, mostly L2-resident), and R is
// scattered back.  A spin of U that is inactive in a replica keeps its R and
// contributes w = 0 exactly as in the full refit.
#pragma once

#include "sym_kernels.cuh"
#include "sym64_kernels.cuh"

namespace cimcs {

// union of the live replicas' supports of instance b (one CTA per instance):
// cU[b][0..cnt) = the union's spins ascending, cU[b][cnt..ldN) = -1
template <int NR>
__global__ void __launch_bounds__(1024) cmp_union_kernel(const int8_t* __restrict__ sig, int N,
                                                         int ldN, int* cU, int* cnt, int* cmax) {
    const int b = blockIdx.x;
    __shared__ int s_base;
    __shared__ int s_warp[32];
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i0 = 0; i0 < ldN; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        bool f = false;
        if (i < N) {
            const int8_t* sp = sig + ((size_t)b * ldN + i) * NR;
#pragma unroll
            for (int q = 0; q < NR; ++q) f |= sp[q] != 0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_warp[wid] = __popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {  // exclusive scan over the warps
            int acc = s_base;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                const int v = s_warp[w];
                s_warp[w] = acc;
                acc += v;
            }
            s_base = acc;
        }
        __syncthreads();
        if (f) cU[(size_t)b * ldN + s_warp[wid] + __popc(m & ((1u << lane) - 1u))] = i;
        __syncthreads();
    }
    const int n = s_base;
    for (int k = n + threadIdx.x; k < ldN; k += blockDim.x) cU[(size_t)b * ldN + k] = -1;
    if (threadIdx.x == 0) {
        cnt[b] = n;
        atomicMax(cmax, n);
    }
}

// compacted tiles: tile (I, J), I <= J < nRBc, element (r, c) = G[u_r][u_c]
// from the full tiles (pad rows / columns: 0); one CTA per (tile, instance)
__global__ void __launch_bounds__(256) cmp_gather_tiles_kernel(const __half* __restrict__ Gs,
                                                               int ntri, int nRB,
                                                               const int* __restrict__ cU, int ldN,
                                                               int nRBc, int ntric, __half* Gc) {
    const int b = blockIdx.y;
    int t = blockIdx.x, I = 0;
    while (t >= nRBc - I) {  // row-major upper-triangle index -> (I, J)
        t -= nRBc - I;
        ++I;
    }
    const int J = I + t;
    const int* ub = cU + (size_t)b * ldN;
    const __half* Gb = Gs + (size_t)b * ntri * 2 * kSyPlaneHalfs;
    __half* out = Gc + ((size_t)b * ntric + sy_tri(I, J, nRBc)) * 2 * kSyPlaneHalfs;
    for (int e = threadIdx.x; e < kSyT * kSyT / 8; e += blockDim.x) {
        const int r = e / (kSyT / 8), c0 = (e % (kSyT / 8)) * 8;
        const int i = ub[I * kSyT + r];
        __align__(16) __half hi[8], lo[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = ub[J * kSyT + c0 + u];
            __half h = __float2half(0.f), l = __float2half(0.f);
            if (i >= 0 && j >= 0) {
                int p = i, q = j;  // stored upper triangle
                if (p / kSyT > q / kSyT) {
                    p = j;
                    q = i;
                }
                const size_t o = (size_t)sy_tri(p / kSyT, q / kSyT, nRB) * 2 * kSyPlaneHalfs +
                                 sy_offk(p % kSyT, q % kSyT, kSyT) / 2;
                h = Gb[o];
                l = Gb[o + kSyPlaneHalfs];
            }
            hi[u] = h;
            lo[u] = l;
        }
        const int o = sy_offk(r, c0, kSyT) / 2;  // 8 consecutive K = 16 contiguous bytes
        *reinterpret_cast<uint4*>(out + o) = *reinterpret_cast<const uint4*>(hi);
        *reinterpret_cast<uint4*>(out + kSyPlaneHalfs + o) = *reinterpret_cast<const uint4*>(lo);
    }
}

// compacted state: Rc, sigc, Dc, hzc, and the refit's first input Wc = Rc o sigc
template <int NR>
__global__ void cmp_gather_state_kernel(const float* __restrict__ Rs, const int8_t* __restrict__ sig,
                                        const float* __restrict__ D, const float* __restrict__ hz,
                                        const int* __restrict__ cU, int ldN, int B, float* Rc,
                                        int8_t* sigc, float* Dc, float* hzc, float* Wc) {
    const size_t total = (size_t)B * ldN;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(t / ldN);
        const int i = cU[t];
        if (i >= 0) {
            const size_t si = (size_t)b * ldN + i;
            Dc[t] = D[si];
            hzc[t] = hz[si];
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                const float r = Rs[si * NR + q];
                const int8_t s = sig[si * NR + q];
                Rc[t * NR + q] = r;
                sigc[t * NR + q] = s;
                Wc[t * NR + q] = r * (s ? 1.f : 0.f);
            }
        } else {
            Dc[t] = 0.f;
            hzc[t] = 0.f;
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                Rc[t * NR + q] = 0.f;
                sigc[t * NR + q] = 0;
                Wc[t * NR + q] = 0.f;
            }
        }
    }
}

// refitted R back to the full state (union rows only)
template <int NR>
__global__ void cmp_scatter_kernel(const float* __restrict__ Rc, const int* __restrict__ cU,
                                   int ldN, int B, float* Rs) {
    const size_t total = (size_t)B * ldN;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int i = cU[t];
        if (i < 0) continue;
        const size_t si = (size_t)(t / ldN) * ldN + i;
#pragma unroll
        for (int q = 0; q < NR; ++q) Rs[si * NR + q] = Rc[t * NR + q];
    }
}

// ---------------------------------------------------------------------------
// The fp64 (DMMA) path's compacted refit keeps the oracle order BITWISE: the
// canonical order sums 512-column segments left to right, each an ascending
// fma chain, and fma(g, +-0, acc) == acc exactly (acc is never -0: chains
// start at +0), so dropping the zero w of non-union spins changes nothing as
// long as no compacted 64-column block mixes two original segments.  Each
// original segment s is therefore compacted on its own, padded to a multiple of
// 64 (the batch maximum), and segments no instance uses are dropped (their
// partial is an exact +0).  The DMMA kernels then run on the variable-width
// segments (Sym64Args::seg).
namespace cmp64 {
constexpr int kSeg = 512;     // the canonical segment (oracle CANON gran)
constexpr int kMaxSeg = 256;  // oracle P[256]: N <= 131072
}

// per (instance, original segment): union spins in it
__global__ void cmp64_segcount_kernel(const int* __restrict__ cU, const int* __restrict__ cnt,
                                      int ldN, int nseg, int B, int* segc) {
    const size_t total = (size_t)B * ldN;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(t / ldN), k = (int)(t % ldN);
        if (k < cnt[b]) atomicAdd(&segc[b * nseg + cU[t] / cmp64::kSeg], 1);
    }
}

// compacted index -> original spin: segment s of instance b starts at segoff[s]
// (-1: dropped) and holds its union spins in ascending order
__global__ void cmp64_map_kernel(const int* __restrict__ cU, const int* __restrict__ cnt,
                                 const int* __restrict__ segpfx, const int* __restrict__ segoff,
                                 int ldN, int nseg, int B, int* cU6) {
    const size_t total = (size_t)B * ldN;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(t / ldN), k = (int)(t % ldN);
        if (k >= cnt[b]) continue;
        const int i = cU[t], s = i / cmp64::kSeg;
        const int rank = k - segpfx[b * nseg + s];  // position inside the segment
        cU6[(size_t)b * ldN + segoff[s] + rank] = i;
    }
}

// compacted fp64 tiles (64 x 64, XOR-swizzled as sym64), element (r, c) = G[u_r][u_c]
__global__ void __launch_bounds__(256) cmp64_gather_tiles_kernel(
    const double* __restrict__ Gt, int ntri, int nRB, const int* __restrict__ cU6, int ldN,
    int nRBc, int ntric, double* Gc) {
    const int b = blockIdx.y;
    int t = blockIdx.x, I = 0;
    while (t >= nRBc - I) {
        t -= nRBc - I;
        ++I;
    }
    const int J = I + t;
    const int* ub = cU6 + (size_t)b * ldN;
    const double* Gb = Gt + (size_t)b * ntri * (kT6 * kT6);
    double* out = Gc + ((size_t)b * ntric + sy_tri(I, J, nRBc)) * (kT6 * kT6);
    for (int e = threadIdx.x; e < kT6 * kT6; e += blockDim.x) {
        const int r = e / kT6, cc = e % kT6;
        const int i = ub[I * kT6 + r], j = ub[J * kT6 + cc];
        double v = 0.0;
        if (i >= 0 && j >= 0) {
            int p = i, q = j;
            if (p / kT6 > q / kT6) {
                p = j;
                q = i;
            }
            v = Gb[(size_t)sy_tri(p / kT6, q / kT6, nRB) * (kT6 * kT6) + s6_gofs(p % kT6, q % kT6)];
        }
        out[s6_gofs(r, cc)] = v;
    }
}

template <int NR>
__global__ void cmp64_gather_state_kernel(const double* __restrict__ Rs,
                                          const int8_t* __restrict__ sig,
                                          const double* __restrict__ D,
                                          const double* __restrict__ hz, const int* __restrict__ cU,
                                          int ldN, int B, double* Rc, int8_t* sigc, double* Dc,
                                          double* hzc, double* Wc) {
    const size_t total = (size_t)B * ldN;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(t / ldN);
        const int i = cU[t];
        const bool on = i >= 0;
        const size_t si = (size_t)b * ldN + (on ? i : 0);
        Dc[t] = on ? D[si] : 0.0;
        hzc[t] = on ? hz[si] : 0.0;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
            const double r = on ? Rs[si * NR + q] : 0.0;
            const int8_t s = on ? sig[si * NR + q] : 0;
            Rc[t * NR + q] = r;
            sigc[t * NR + q] = s;
            Wc[t * NR + q] = r * (s ? 1.0 : 0.0);
        }
    }
}

template <int NR>
__global__ void cmp64_scatter_kernel(const double* __restrict__ Rc, const int* __restrict__ cU,
                                     int ldN, int B, double* Rs) {
    const size_t total = (size_t)B * ldN;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int i = cU[t];
        if (i < 0) continue;
        const size_t si = (size_t)(t / ldN) * ldN + i;
#pragma unroll
        for (int q = 0; q < NR; ++q) Rs[si * NR + q] = Rc[t * NR + q];
    }
}

}  // namespace cimcs
