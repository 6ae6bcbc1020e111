// gram_tc_kernels.cuh -- K1 for large N on the 5th-gen tensor cores: the fp32
// symmetric path's gram G = A^T A (model.cpp:54-63, orchestrator.cpp:84-85)
// written straight into its fp16 hi/lo upper-triangle 128 x 128 tiles (SymOut).
// No library GEMM is involved (configs 3 and 4 used cuBLAS panels in round 1).
//
// The tiles keep ~22 bits, so the GEMM must be fp32-accurate.  A (fp64, scaled
// by an exact 2^s_A per instance) is split once into fp16 hi/lo planes,
// x ~= hi + lo (~22 bits), stored PRE-TILED per 32-row k-chunk, plane and 128-column
// block in the UMMA canonical no-swizzle K-major layout (M/N = 128, K = 32):
//     plane(c, p)[ (j/128) * 8 KB + (k/8) * 2 KB + ((j%128)/8) * 128 B + (j%8) * 16 B + (k%8) * 2 B ]
// so one operand plane of a stage is ONE contiguous 8 KB bulk copy (4 per stage).
// Per k-step (K = 16) the MMA warp issues
//     D += A_hi_I^T A_hi_J + A_hi_I^T A_lo_J + A_lo_I^T A_hi_J     (kind::f16, M = N = 128)
// (the lo*lo term is below fp32 resolution).
//
// Accuracy: the tensor core's fp32 accumulation truncates once per MMA relative
// to the accumulator (measured: a K = 550 gram chain accumulated whole in TMEM
// is off by ~3e-6 relative -- ~1 ulp per MMA, linear in K).  So every 32-row
// k-chunk starts a FRESH accumulator (2 hi*hi MMAs deep: ~2.4e-7, the tiles' own
// resolution), double-buffered in TMEM; eight epilogue warps drain each chunk
// into fp32 registers with a two-level sum (16 chunks, then a running total),
// so the fp32 rounding of the long K sum stays at ~sqrt(K / 512) ulp.
// Measured on the kernel (tools/gram_pipeline.py, tools/gram_time.py): a k-chunk costs
// 0.55 us per CTA, 0.35 us of it the six MMAs themselves -- each reads 8 KB of operands
// from shared memory while the ring's bulk copies write 32 KB per chunk into it, so the
// chunk moves 80 KB through a 128 B/clk port: the kernel is bound by shared-memory
// bandwidth, not by loads (a 7-stage ring with the second-level sums moved to TMEM gave
// 0.56 us) nor by the tensor pipe (6 x 64 clk).
// Persistent CTAs walk the upper-triangle tiles super-block by super-block (kGtSB x
// kGtSB tiles, about one per wave of 148 CTAs), so the CTAs of a wave share 2 x kGtSB
// operand blocks in L2 instead of streaming one A_J block each from HBM; warp 0
// produces (bulk copies into a 4-stage ring), warps 1 and 10 issue the MMAs (alternate k-chunks), warps 2-9
// drain TMEM and finally store the fp16 hi/lo SymOut values (G * 2^s_G).  Producer
// and MMA warps run convergently on warp-uniform operands with one elected lane
// issuing (see sym_step_kernel: issuing from inside `if (lane == 0)` costs an
// ELECT / R2UR / BRA.U.ANY loop per instruction).
#pragma once

#include "sym_kernels.cuh"

namespace cimcs {

constexpr int kGtK = 32;                          // k per chunk / pipeline stage
constexpr int kGtStages = 4;
constexpr int kGtEpi = 8;                         // epilogue warps (2 per TMEM lane quadrant)
constexpr int kGtMma2 = 2 + kGtEpi;                // second MMA issuer warp (odd chunks)
constexpr int kGtThreads = (3 + kGtEpi) * 32;
constexpr int kGtInner = 16;                      // chunks per first-level sum
constexpr uint32_t kGtPlane = kSyT * kGtK * 2;    // 8 KB: one plane of one 128-column block
constexpr uint32_t kGtStage = 4 * kGtPlane;       // A_I hi, lo; A_J hi, lo
// + the second-level sums of the epilogue threads ([64][256] fp32, conflict-free)
constexpr size_t kGtS2 = (size_t)64 * kGtEpi * 32 * 4;
constexpr size_t kGtSmem = (size_t)kGtStages * kGtStage + kGtS2 + 256;
constexpr int kGtTmemCols = 256;                  // 2 x 128 accumulator columns

constexpr int kGtSB = 12;                         // super-block edge in tiles (L2 reuse)

// byte offset of (column j, k within the chunk) in one plane of a k-chunk
__host__ __device__ inline size_t gt_off(int j, int k, int /*Np*/) {
    return (size_t)(j / kSyT) * kGtPlane + (size_t)(k / 8) * ((kSyT / 8) * 128) +
           (size_t)((j % kSyT) / 8) * 128 + (j % 8) * 16 + (k % 8) * 2;
}

// per-instance exact scale: max|A| * 2^s in [2^14, 2^15)
__global__ void gt_absmax_kernel(const double* __restrict__ A, size_t n,
                                 unsigned long long* out) {
    double m = 0.0;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
         t += (size_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(A[t]));
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__device__ __forceinline__ int gt_scale(const unsigned long long* amax) {
    const double m = __longlong_as_double((long long)*amax);
    if (!(m > 0.0)) return 0;
    int ex;
    frexp(m, &ex);  // m = f * 2^ex, f in [0.5, 1): m * 2^(15 - ex) in [2^14, 2^15)
    return 15 - ex;
}

// A (column-major M x N, ld M) -> hi/lo planes [nch][2][Np x 32 canonical]
__global__ void gt_split_kernel(const double* __restrict__ A, int M, int N, int Np, int nch,
                                const unsigned long long* amax, __half* __restrict__ P) {
    const int e = gt_scale(amax);
    const size_t plane = (size_t)Np * kGtK;  // halfs per plane
    const size_t total = (size_t)nch * Np * (kGtK / 8);  // one thread per (chunk, j, k-group)
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(t % Np);
        const size_t r = t / Np;
        const int kg = (int)(r % (kGtK / 8));
        const int c = (int)(r / (kGtK / 8));
        __align__(16) __half hi[8], lo[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = c * kGtK + kg * 8 + u;
            const double v = (j < N && k < M) ? ldexp(A[(size_t)j * M + k], e) : 0.0;
            hi[u] = __double2half(v);
            lo[u] = __double2half(v - (double)__half2float(hi[u]));
        }
        const size_t o = gt_off(j, kg * 8, Np) / 2;
        __half* ph = P + (size_t)c * 2 * plane;
        *reinterpret_cast<uint4*>(ph + o) = *reinterpret_cast<const uint4*>(hi);
        *reinterpret_cast<uint4*>(ph + plane + o) = *reinterpret_cast<const uint4*>(lo);
    }
}

struct GtArgs {
    const __half* P;                 // split planes of this instance
    const unsigned long long* amax;  // its max|A|
    SymOut out;                      // the fp32 path's tiles (its own scale s_G)
    int b;                           // instance index of `out`
    int N, Np, nch;
    int I0, I1;                      // row blocks built by this rank [I0, I1)
    int nRB;                         // column blocks (ceil(N / 128))
    long long ntile;                 // tiles (I, J), I0 <= I < I1, I <= J < nRB
    unsigned* round;                 // zeroed per launch: producers that finished issuing a round
    unsigned long long* tlog;        // option "timeline": CTA 0's per-chunk stamps (sym_kernels.cuh rows)
};

// tile t -> (I, J): super-blocks of kGtSB x kGtSB tiles, row-major over the super-
// block triangle of the rows [I0, I1); inside a super-block row-major (I <= J)
__device__ __forceinline__ void gt_tile(const GtArgs& a, long long t, int& I, int& J) {
    for (int R0 = a.I0; R0 < a.I1; R0 += kGtSB) {
        const int nI = min(kGtSB, a.I1 - R0);
        // this super-row: the diagonal block (columns R0 .. R0 + nI), then full blocks
        const long long diag = (long long)nI * (nI + 1) / 2;
        const long long rest = (long long)nI * (a.nRB - R0 - nI);
        if (t >= diag + rest) {
            t -= diag + rest;
            continue;
        }
        if (t < diag) {  // row i has nI - i tiles
            int i = 0;
            while (t >= nI - i) {
                t -= nI - i;
                ++i;
            }
            I = R0 + i;
            J = I + (int)t;
            return;
        }
        t -= diag;
        const long long per = (long long)nI * kGtSB;  // tiles of a full super-block
        const int sb = (int)(t / per);
        t -= sb * per;
        const int C0 = R0 + nI + sb * kGtSB;
        const int nJ = min(kGtSB, a.nRB - C0);
        I = R0 + (int)(t / nJ);
        J = C0 + (int)(t % nJ);
        return;
    }
    I = J = a.I1 - 1;  // not reached for t < ntile
}

__global__ void __launch_bounds__(kGtThreads, 1) gram_tc_kernel(GtArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    float* s2all = reinterpret_cast<float*>(smem + kGtStages * kGtStage);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGtStages * kGtStage + kGtS2);
    uint64_t* empty = full + kGtStages;
    uint64_t* tm_full = empty + kGtStages;  // [2]
    uint64_t* tm_empty = tm_full + 2;       // [2]
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kGtStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&tm_full[k], 1);
            mbar_init(&tm_empty[k], kGtEpi);
        }
        mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kGtTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const size_t plane = (size_t)a.Np * kGtK * 2;  // bytes per plane
    const unsigned char* Pb = reinterpret_cast<const unsigned char*>(a.P);
    constexpr uint32_t kBlk = (kSyT / 8) * 128;    // 2 KB: one k-group of one 128-column block

    if (warp == 0) {  // -------------------------------------------------- producer
        const uint64_t pol = sy_policy_last();
        const uint32_t smem0 = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
        const uint32_t full0 = __shfl_sync(0xffffffffu, smem_u32(full), 0);
        long long it = 0;
        unsigned rnd = 0;
        for (long long t = blockIdx.x; t < a.ntile; t += gridDim.x, ++rnd) {
            // Round gate (a locality hint, never needed for correctness): start round r
            // only when every CTA's producer has issued all of round r - 1, so the CTAs
            // of a wave walk the k-chunks of ONE super-block together and its 2 x kGtSB
            // operand blocks are read from HBM once and from L2 by everyone else.  Without
            // it the CTAs drift apart by whole tiles and each streams its own operands
            // from HBM (measured: 32 KB per chunk-step at the HBM rate).  The wait is
            // bounded (~0.5 ms); on expiry the CTA simply goes on.
            if (rnd && lane == 0) {
                const unsigned want = rnd * gridDim.x;
                const long long t0 = clock64();
                unsigned v;
                do {
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.round) : "memory");
                } while (v < want && clock64() - t0 < (1ll << 20));
            }
            __syncwarp();
            int I, J;
            gt_tile(a, t, I, J);
            I = __shfl_sync(0xffffffffu, I, 0);
            J = __shfl_sync(0xffffffffu, J, 0);
            const unsigned char* srcI = Pb + (size_t)I * kGtPlane;
            const unsigned char* srcJ = Pb + (size_t)J * kGtPlane;
            for (int c = 0; c < a.nch; ++c, ++it) {
                const int s = (int)(it % kGtStages);
                if (it >= kGtStages) mbar_wait(&empty[s], (uint32_t)(((it / kGtStages) - 1) & 1));
                if (a.tlog && blockIdx.x == 0 && it < 128 && lane == 0)
                    a.tlog[(kTlTile + it) * 4 + 3] = sy_gtime();
                if (sy_elect_one()) {
                    const uint32_t st = smem0 + s * kGtStage, fb = full0 + s * 8;
                    sy_expect_tx_u(fb, kGtStage);
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        const size_t o = ((size_t)c * 2 + p) * plane;
                        sy_bulk_u(st + p * kGtPlane, srcI + o, kGtPlane, fb, pol);
                        sy_bulk_u(st + (2 + p) * kGtPlane, srcJ + o, kGtPlane, fb, pol);
                    }
                }
                __syncwarp();
            }
            if (lane == 0) atomicAdd(a.round, 1u);
        }
    } else if (warp == 1 || warp == kGtMma2) {  // ------------------------ MMA issuers
        // Two issuer warps take alternate k-chunks (each owns one TMEM accumulator): the
        // ~0.2 us a warp spends between chunks (barrier waits, fences, descriptors) is
        // hidden behind the other warp's six MMAs.  The chunks of the two warps touch
        // different stages and accumulators, so their relative issue order is free; each
        // warp commits its own MMAs.
        const int par = warp == 1 ? 0 : 1;
        constexpr uint32_t idesc = sy_idesc(kSyT, 0);  // F32 += F16 x F16, M = N = 128
        const uint32_t smem0 = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
        long long it = 0;
        for (long long t = blockIdx.x; t < a.ntile; t += gridDim.x) {
            for (int c = 0; c < a.nch; ++c, ++it) {
                const int s = (int)(it % kGtStages), buf = (int)(it & 1);
                if (buf != par) continue;
                const bool tl = a.tlog && blockIdx.x == 0 && it < 128 && lane == 0;
                if (it >= 2) mbar_wait(&tm_empty[buf], (uint32_t)(((it >> 1) - 1) & 1));
                if (tl) a.tlog[(kTlTile + it) * 4 + 0] = sy_gtime();
                mbar_wait(&full[s], (uint32_t)((it / kGtStages) & 1));
                if (tl) a.tlog[(kTlTile + it) * 4 + 1] = sy_gtime();
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t aHi = smem0 + s * kGtStage;
                const uint32_t d = tmem_u + buf * kSyT;
                // descriptors of k-step 0; planes and k-steps only move the start address
                const uint64_t dAh0 = umma_desc(aHi, kBlk, 128);
                if (sy_elect_one()) {
#pragma unroll
                    for (int kb = 0; kb < kGtK / 16; ++kb) {
                        const uint64_t dAh = dAh0 + (uint64_t)(kb * 2 * kBlk >> 4);
                        const uint64_t dAl = dAh + (uint64_t)(kGtPlane >> 4);
                        const uint64_t dBh = dAh + (uint64_t)(2 * kGtPlane >> 4);
                        const uint64_t dBl = dAh + (uint64_t)(3 * kGtPlane >> 4);
                        sy_mma(d, dAh, dBh, idesc, kb ? 1u : 0u);  // a fresh accumulator per chunk
                        sy_mma(d, dAh, dBl, idesc, 1u);
                        sy_mma(d, dAl, dBh, idesc, 1u);
                    }
                    tc_commit(&empty[s]);
                    tc_commit(&tm_full[buf]);
                }
                __syncwarp();
                if (tl) a.tlog[(kTlTile + it) * 4 + 2] = sy_gtime();
            }
        }
    } else if (warp < kGtMma2) {  // ------------------------------------ epilogue
        const int q = warp & 3;           // TMEM lane quadrant (warps 2..9)
        const int h = (warp - 2) >> 2;    // column half: 64 columns each
        const int row = q * 32 + lane;
        const int e = gt_scale(a.amax);
        long long it = 0;
        for (long long t = blockIdx.x; t < a.ntile; t += gridDim.x) {
            int I, J;
            gt_tile(a, t, I, J);
            float s1[64];
            float* s2 = s2all + (threadIdx.x - 64);  // element u at s2[u * 256]
#pragma unroll
            for (int u = 0; u < 64; ++u) {
                s1[u] = 0.f;
                s2[u * kGtEpi * 32] = 0.f;
            }
            for (int c = 0; c < a.nch; ++c, ++it) {
                const int buf = (int)(it & 1);
                mbar_wait(&tm_full[buf], (uint32_t)((it >> 1) & 1));
                const bool tle = a.tlog && blockIdx.x == 0 && it < 128 && threadIdx.x == 64;
                if (tle) a.tlog[(kTlTile + 128 + it) * 4 + 0] = sy_gtime();
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t ta = tmem + buf * kSyT + h * 64 + ((uint32_t)(q * 32) << 16);
#pragma unroll
                for (int gh = 0; gh < 2; ++gh) {  // 2 x 32 columns (register budget)
                    uint32_t v[2][16];
                    tmem_ld16(ta + gh * 32, v[0]);
                    tmem_ld16(ta + gh * 32 + 16, v[1]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int g = 0; g < 2; ++g)
#pragma unroll
                        for (int u = 0; u < 16; ++u)
                            s1[gh * 32 + g * 16 + u] += __uint_as_float(v[g][u]);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&tm_empty[buf]);
                if (tle) a.tlog[(kTlTile + 128 + it) * 4 + 1] = sy_gtime();
                if ((c + 1) % kGtInner == 0) {
#pragma unroll
                    for (int u = 0; u < 64; ++u) {
                        s2[u * kGtEpi * 32] += s1[u];
                        s1[u] = 0.f;
                    }
                }
            }
            // tile done: G = (s2 + s1) * 2^(-2 s_A) -> fp16 hi/lo * 2^s_G, 8 columns per store
            __half* tb = a.out.G + ((size_t)a.b * a.out.ntri + sy_tri(I, J, a.out.nRB)) * 2 * kSyPlaneHalfs;
            const int es = a.out.sg[a.b] - 2 * e;
#pragma unroll
            for (int g8 = 0; g8 < 8; ++g8) {
                __align__(16) __half hi[8], lo[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double gs =
                        ldexp((double)s2[(g8 * 8 + u) * kGtEpi * 32] + (double)s1[g8 * 8 + u], es);
                    hi[u] = __double2half(gs);
                    lo[u] = __double2half(gs - (double)__half2float(hi[u]));
                }
                const int k0 = h * 64 + g8 * 8;  // column within the tile (K of the canonical layout)
                const int o = sy_offk(row, k0, kSyT) / 2;
                *reinterpret_cast<uint4*>(tb + o) = *reinterpret_cast<const uint4*>(hi);
                *reinterpret_cast<uint4*>(tb + kSyPlaneHalfs + o) = *reinterpret_cast<const uint4*>(lo);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kGtTmemCols));
}

}  // namespace cimcs
