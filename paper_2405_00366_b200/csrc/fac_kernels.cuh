// fac_kernels.cuh -- fp32 fused MFZ step on the FACTORED coupling: G w =
// A^T (A w), the reference's own matrix-free form (orchestrator.cpp:84-88,
// apply_gram closure), with A held on the device as fp16 hi/lo 128 x 128 tiles.
//
// When M is at most about N/2 the M x N tiles of A hold no more bytes than the
// upper triangle of G (config 1: 8 x 16 = 128 tiles vs 136), and the
// contraction needs NO partial products: a task owns one whole output block.
//   phase 1, task (b, I):  u[I]  = sum_J A[I,J]   w[J]   (A tile K-major)
//   phase 2, task (b, Jc): Gw[J] = sum_I A[I,J]^T u[I]   (same bytes, MN-major
//                          view, as the symmetric kernel's use 2), 1-2 column
//                          blocks per task so both phases have ~equal tiles
// A phase-2 task of instance b starts once every phase-1 task of b has
// published its u block (per-instance counter, release/acquire + async-proxy
// fence, since u is read back by bulk copies).  Tasks are laid out so that
// phase 2 of instance b comes `skew` instances after its phase 1: the wait is
// normally already satisfied, and A[b] is re-read while it is still in L2, so
// HBM sees A about once per step.  Deadlock freedom: the kernel is launched
// cooperatively (all CTAs resident) and every task only waits on tasks with a
// smaller index, which their CTAs reach first (induction on the index).
//
// Each tile's product goes to its own TMEM buffer (4 in flight); the epilogue
// unscales it exactly (2^-(s_A + s_B)) and accumulates in registers in a FIXED
// tile order, so results do not depend on scheduling.  Phase 1 emits u as the
// fp16 hi/lo B tile format of the symmetric kernel (sy_emit_block); phase 2
// runs the fused update of tc_row_update (step / Jacobi / matvec / score) and
// emits the next w tiles.  The counters reset themselves (the last phase-2
// task of an instance zeroes them), so the kernel can be replayed in graphs.
#pragma once

#include "sym_kernels.cuh"

namespace cimcs {

constexpr int kFaStages = 3;
constexpr int kFaTmemBufs = 4;
constexpr int kFaThreads = 6 * 32;
constexpr int kFaTmemCols = 128;
constexpr int kFaW2 = 2;  // max column blocks per phase-2 task

// task table entry: phase (bit 31), instance (bits 16-30), block index (0-15)
__host__ __device__ inline int fa_task(int phase, int b, int idx) {
    return (phase << 31) | (b << 16) | idx;
}

struct FacArgs {
    TcArgs t;
    const __half* As;     // [B][nMB][nRB][hi | lo][128 x 128], element (m, n) at sy_offk(m, n)
    const int* sa;        // [B] scale exponent of A
    const __half* WBin;   // [B][nRB][2NR x 128] fp16 B tiles of w (and scales)
    const int* WSin;
    __half* WBout;
    int* WSout;
    __half* UB;           // [B][nMB][2NR x 128] fp16 B tiles of u = A w
    int* US;
    int* cnt;             // [2B]: phase-1 tasks done, phase-2 tasks done
    const int* task;      // [ntask]
    int ntask, nMB, W2;
};

template <int NR>
__host__ __device__ constexpr size_t fa_stage_bytes() {
    return 2 * (size_t)kSyPlaneBytes + sy_bbytes<NR>();
}
template <int NR>
__host__ __device__ constexpr size_t fa_smem_bytes() {
    return kFaStages * fa_stage_bytes<NR>() + 64 * 8;
}

__device__ __forceinline__ int fa_ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fa_fence_proxy() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// tiles of the task: phase 1: J = 0..nRB-1; phase 2: I-major over nc columns
struct FaTask {
    int phase, b, idx, ntiles, nc;
};
__device__ __forceinline__ FaTask fa_decode(const FacArgs& f, int t) {
    const int e = f.task[t];
    FaTask k;
    k.phase = (e >> 31) & 1;
    k.b = (e >> 16) & 0x7fff;
    k.idx = e & 0xffff;
    if (k.phase == 0) {
        k.nc = 1;
        k.ntiles = f.t.nRB;
    } else {
        k.nc = min(f.W2, f.t.nRB - k.idx * f.W2);
        k.ntiles = f.nMB * k.nc;
    }
    return k;
}

template <int NR, int MODE>
__global__ void __launch_bounds__(kFaThreads, 1) fac_step_kernel(FacArgs f) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const TcArgs& a = f.t;
    constexpr uint32_t kBB = (uint32_t)sy_bbytes<NR>();
    constexpr uint32_t kStage = (uint32_t)fa_stage_bytes<NR>();
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kFaStages * kStage);
    uint64_t* empty = full + kFaStages;
    uint64_t* tm_full = empty + kFaStages;
    uint64_t* tm_empty = tm_full + kFaTmemBufs;
    __shared__ uint32_t s_tmem;
    __shared__ unsigned s_max[4][NR];
    __shared__ double s_part[4][NR][3];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nRB = a.nRB, nMB = f.nMB;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kFaStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int k = 0; k < kFaTmemBufs; ++k) {
            mbar_init(&tm_full[k], 1);
            mbar_init(&tm_empty[k], 4);
        }
        mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kFaTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const size_t tileH = 2 * (size_t)kSyPlaneHalfs;  // halfs per A tile (hi | lo)
    const size_t bH = (size_t)2 * NR * kSyT;          // halfs per B tile

    if (warp == 0) {
        // ------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pF = sy_policy_first(), pL = sy_policy_last();
            int tt = 0;
            for (int t = blockIdx.x; t < f.ntask; t += gridDim.x) {
                const FaTask k = fa_decode(f, t);
                const __half* Ab = f.As + (size_t)k.b * nMB * nRB * tileH;
                if (k.phase == 1) {  // u of instance b complete?
                    const int* c1 = f.cnt + 2 * k.b;
                    while (fa_ld_acquire(c1) < nMB) __nanosleep(64);
                    fa_fence_proxy();
                }
                for (int x = 0; x < k.ntiles; ++x, ++tt) {
                    const int s = tt % kFaStages;
                    int I, J;
                    const __half* bt;
                    if (k.phase == 0) {
                        I = k.idx;
                        J = x;
                        bt = f.WBin + ((size_t)k.b * nRB + J) * bH;
                    } else {
                        I = x / k.nc;
                        J = k.idx * f.W2 + x % k.nc;
                        bt = f.UB + ((size_t)k.b * nMB + I) * bH;
                    }
                    if (tt >= kFaStages) mbar_wait(&empty[s], ((tt / kFaStages) - 1) & 1);
                    unsigned char* st = smem + s * kStage;
                    mbar_arrive_expect_tx(&full[s], 2 * kSyPlaneBytes + kBB);
                    // phase 1 leaves A in L2 for phase 2, which drops it
                    sy_bulk_g2s(st, Ab + ((size_t)I * nRB + J) * tileH, 2 * kSyPlaneBytes,
                                &full[s], k.phase ? pF : pL);
                    sy_bulk_g2s(st + 2 * kSyPlaneBytes, bt, kBB, &full[s], pL);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t id_cat = sy_idesc(2 * NR, 0), id_hi = sy_idesc(NR, 0);
            constexpr uint32_t id_catT = sy_idesc(2 * NR, 1), id_hiT = sy_idesc(NR, 1);
            constexpr uint32_t kstr = (kSyT / 8) * 128;
            constexpr uint32_t lboB = (2 * NR / 8) * 128;
            int tt = 0;
            for (int t = blockIdx.x; t < f.ntask; t += gridDim.x) {
                const FaTask k = fa_decode(f, t);
                for (int x = 0; x < k.ntiles; ++x, ++tt) {
                    const int s = tt % kFaStages, buf = tt % kFaTmemBufs;
                    if (tt >= kFaTmemBufs) mbar_wait(&tm_empty[buf], ((tt / kFaTmemBufs) - 1) & 1);
                    mbar_wait(&full[s], (tt / kFaStages) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t aHi = smem_u32(smem + s * kStage), aLo = aHi + kSyPlaneBytes;
                    const uint32_t bB = aHi + 2 * kSyPlaneBytes;
                    const uint32_t d = tmem + buf * 2 * NR;
                    if (k.phase == 0) {
#pragma unroll
                        for (int kb = 0; kb < kSyT / 16; ++kb) {
                            const uint64_t dB = umma_desc(bB + kb * 2 * lboB, lboB, 128);
                            sy_mma(d, umma_desc(aHi + kb * 2 * kstr, kstr, 128), dB, id_cat,
                                   kb ? 1u : 0u);
                            sy_mma(d, umma_desc(aLo + kb * 2 * kstr, kstr, 128), dB, id_hi, 1u);
                        }
                    } else {
#pragma unroll
                        for (int kb = 0; kb < kSyT / 16; ++kb) {
                            const uint64_t dB = umma_desc(bB + kb * 2 * lboB, lboB, 128);
                            sy_mma(d, umma_desc(aHi + kb * 256, 128, kstr), dB, id_catT,
                                   kb ? 1u : 0u);
                            sy_mma(d, umma_desc(aLo + kb * 256, 128, kstr), dB, id_hiT, 1u);
                        }
                    }
                    tc_commit(&empty[s]);
                    tc_commit(&tm_full[buf]);
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (4 warps)
        const int ew = warp & 3;
        const int row = ew * 32 + lane;
        int tt = 0;
        for (int t = blockIdx.x; t < f.ntask; t += gridDim.x) {
            const FaTask k = fa_decode(f, t);
            const int b = k.b;
            const float fA = sy_pow2(-f.sa[b]);
            float acc[kFaW2][NR];
#pragma unroll
            for (int c = 0; c < kFaW2; ++c)
#pragma unroll
                for (int q = 0; q < NR; ++q) acc[c][q] = 0.f;
            for (int x = 0; x < k.ntiles; ++x, ++tt) {
                const int buf = tt % kFaTmemBufs;
                mbar_wait(&tm_full[buf], (tt / kFaTmemBufs) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                float g[NR];
                tmem_ld_row<NR>(tmem + buf * 2 * NR + ((uint32_t)(ew * 32) << 16), g);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&tm_empty[buf]);
                const int* sB = k.phase == 0 ? f.WSin + ((size_t)b * nRB + x) * NR
                                             : f.US + ((size_t)b * nMB + x / k.nc) * NR;
                const int c = k.phase == 0 ? 0 : x % k.nc;
#pragma unroll
                for (int cc = 0; cc < kFaW2; ++cc)
                    if (cc == c) {
#pragma unroll
                        for (int q = 0; q < NR; ++q)
                            acc[cc][q] = acc[cc][q] + g[q] * fA * sy_pow2(-__ldg(sB + q));
                    }
            }
            if (k.phase == 0) {
                // u block I: fp16 hi/lo B tile + scales, then publish
                sy_emit_block<NR>(acc[0], row, lane, ew, s_max,
                                  f.UB + ((size_t)b * nMB + k.idx) * (2 * NR * kSyT),
                                  f.US + ((size_t)b * nMB + k.idx) * NR, 1);
                if (row == 0) {
                    fa_fence_proxy();
                    __threadfence();
                    atomicAdd(f.cnt + 2 * b, 1);
                }
            } else {
#pragma unroll
                for (int cc = 0; cc < kFaW2; ++cc) {
                    if (cc >= k.nc) break;
                    const int J = k.idx * f.W2 + cc;
                    float wn[NR];
                    tc_row_update<NR, MODE, false>(a, b, J, row, lane, ew, acc[cc], s_part, 1, wn);
                    if constexpr (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN ||
                                  MODE == EPI_JACOBI)
                        sy_emit_block<NR>(wn, row, lane, ew, s_max,
                                          f.WBout + ((size_t)b * nRB + J) * (2 * NR * kSyT),
                                          f.WSout + ((size_t)b * nRB + J) * NR, 1);
                }
                if (row == 0) {  // last phase-2 task of b: reset the counters
                    const int nP2 = (nRB + f.W2 - 1) / f.W2;
                    if (atomicAdd(f.cnt + 2 * b + 1, 1) == nP2 - 1) {
                        f.cnt[2 * b] = 0;
                        f.cnt[2 * b + 1] = 0;
                        __threadfence();
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kFaTmemCols));
}

// A tiles (fp16 hi/lo, exact 2^s_A scale) from the fp64 column-major A of
// instances b0.. (one thread per element, m fastest: coalesced reads)
__global__ void fac_tiles_kernel(const double* __restrict__ A, const int* __restrict__ M, int N,
                                 size_t astride, int nMB, int nRB, const int* __restrict__ sa,
                                 __half* out, int B) {
    const size_t rows = (size_t)nMB * kSyT, cols = (size_t)nRB * kSyT;
    const size_t total = (size_t)B * rows * cols;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int m = (int)(t % rows);
        const int n = (int)((t / rows) % cols);
        const int b = (int)(t / (rows * cols));
        const int Mb = M[b];
        const double v = (m < Mb && n < N) ? A[(size_t)b * astride + (size_t)n * Mb + m] : 0.0;
        const double vs = ldexp(v, sa[b]);
        const __half hi = __double2half(vs);
        const __half lo = __double2half(vs - (double)__half2float(hi));
        __half* tile = out + (((size_t)b * nMB + m / kSyT) * nRB + n / kSyT) * 2 * kSyPlaneHalfs;
        const int o = sy_offk(m % kSyT, n % kSyT, kSyT) / 2;
        tile[o] = hi;
        tile[kSyPlaneHalfs + o] = lo;
    }
}

// s_A[b]: max |A| * 2^s_A in [2^14, 2^15)
__global__ void fac_scale_kernel(const double* __restrict__ A, const int* __restrict__ M, int N,
                                 size_t astride, int* sa) {
    const int b = blockIdx.x;
    const size_t n = (size_t)M[b] * N;
    const double* Ab = A + (size_t)b * astride;
    float m = 0.f;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, (float)fabs(Ab[i]));
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    __shared__ float s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, s[w]);
        m = fmaxf(m, s[0]);
        // (float)max rounds to nearest: a value that rounds up to 2^15 still
        // fits fp16 (max 65504) after the exact 2^s scaling
        sa[b] = sy_exp14(m);
    }
}

}  // namespace cimcs
