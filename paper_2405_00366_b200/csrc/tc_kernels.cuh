// tc_kernels.cuh -- fp32 fused MFZ step on the 5th-gen tensor cores (tcgen05).
//
// G*W for R replicas is a GEMM with M = 128 spins (rows), N = NR slots (8 or
// 16), K = N spins.  fp32 accuracy is held with a 3xTF32 split:
//     G W ~= G_hi W_hi + G_hi W_lo + G_lo W_hi,   x_hi = trunc_tf32(x), x_lo = x - x_hi
// The tensor core reads raw fp32 operands and truncates them to tf32 (measured
// by tools/tc_probe.cu), so G_hi / W_hi are the raw arrays.  Per k-block:
//   MMA1  D[0:2NR)  += G_hi (smem) x [W | W_lo] (smem, N = 2 NR)   one read of G_hi
//   MMA2  D[0:NR)   += G_lo (TMEM) x W (smem, N = NR)
// W_lo is produced by the previous step's epilogue (the contraction input is
// stored as the concatenated operand); G_lo = G - trunc(G) is computed per
// stage by four "split" warps on CUDA cores and written straight to TMEM, so
// shared memory carries only the bulk-copied G and W tiles.
//
// Persistent, warp-specialised CTA (one per SM, 10 warps):
//   warp 0      producer: per stage one bulk copy of the G panel chunk
//               (64 j x 128 i, 32 KB, stored in HBM in the UMMA canonical
//               layout) + one of the [W | W_lo] chunk (2 NR x 64)
//   warps 1-4   split: G_lo rows -> TMEM (tcgen05.st), double buffered
//   warp 5      MMA issuer (one thread), accumulators double buffered in TMEM
//   warps 6-9   epilogue: tcgen05.ld of the accumulator (one spin row per
//               thread, NR replicas) + the fused Euler / Jacobi / score update
// The epilogue of tile t overlaps the main loop of tile t+1.
//
// Canonical no-swizzle K-major layouts (core matrix = 8 rows x 16 bytes):
//   A tile (128 i x 64 j): float offset (j/4)*512 + (i/8)*32 + (i%8)*4 + j%4
//   B tile (2NR x 64 j)  : float offset (j/4)*8*NR + (r/8)*32 + (r%8)*4 + j%4
// TMEM columns: accumulators [0, 4 NR), G_lo buffers at 64 and 128 (64 each).
#pragma once

#include "kernels.cuh"

namespace cimcs {

constexpr int kTcRows = 128;           // M of the MMA, spins per tile
constexpr int kTcChunk = kTcChunkJ;    // j per pipeline stage
constexpr int kTcStages = 4;
constexpr int kTcThreads = 10 * 32;
constexpr int kTcTileFloats = kTcRows * kTcChunk;  // 8192
constexpr int kTcLoCol = 64;           // first TMEM column of the G_lo buffers
constexpr int kTcTmemCols = 256;

// G panels: [B][nRB][nch][8192] in the canonical A layout
__host__ __device__ inline size_t tc_gofs(int nRB, int nch, int b, int i, int j) {
    const int rb = i / kTcRows, il = i % kTcRows, c = j / kTcChunk, jl = j % kTcChunk;
    return (((size_t)b * nRB + rb) * nch + c) * kTcTileFloats + (jl / 4) * 512 + (il / 8) * 32 +
           (il % 8) * 4 + (jl % 4);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // SWIZZLE_NONE, base offset 0
}

// F32 accumulate, A/B = TF32, both K-major, N, M = 128
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(kTcRows >> 4) << 24);
}

__device__ __forceinline__ void tc_mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t ta, uint64_t db, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
        "r"(ta), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[16], int off) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[off + 0]), "=r"(r[off + 1]), "=r"(r[off + 2]), "=r"(r[off + 3]),
          "=r"(r[off + 4]), "=r"(r[off + 5]), "=r"(r[off + 6]), "=r"(r[off + 7])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15]));
}

// accumulator row of this thread: gw[q] = D[q] + D[NR + q]  (hi*W + lo*W  +  hi*W_lo)
template <int NR>
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, float (&gw)[NR]) {
    uint32_t a[16], b[16];
    if constexpr (NR == 16) {
        tmem_ld16(taddr, a);
        tmem_ld16(taddr + 16, b);
    } else {
        tmem_ld8(taddr, a, 0);
        tmem_ld8(taddr + 8, b, 0);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < NR; ++q) gw[q] = __uint_as_float(a[q]) + __uint_as_float(b[q]);
}

struct TcArgs {
    const float* G;        // panels, canonical A layout
    const float* D;        // [B][ldN]
    const float* hz;
    const float* Win;      // [W | W_lo] canonical, [B][ldJ * 2NR]
    float* Wout;
    float* Rs;             // [B][ldN][NR]
    float* C;
    float* E;
    float* Hdbg;
    double* Mv;            // EPI_MATVEC output [B][ldN][NR]
    const int8_t* sigma;   // [B][ldN][NR]
    int* fail_gstep;
    int* fail_idx;
    unsigned long long* minE;
    double* part;          // [B][nRB][NR][4]
    const double* pump;
    const AltParams* alt;
    const double* xtrue;
    const int8_t* xitrue;
    int* err;
    double p_scalar;
    int step;
    int N, ldN, ldJ, B, nRB, nch, ntiles;  // nRB: LOCAL row blocks per instance
    int rb0;                               // first global row block of this rank
    StepScalars s;
};

// Per-row fused update after the contraction: thread `row` of the four
// epilogue warps owns spin i = (rb0 + rb) * 128 + row of instance b and all NR
// replicas; gw[q] = (G w)_iq.  Shared by the streaming kernel below and the
// symmetric-tile kernel (sym_kernels.cuh).  kWLo: also store the tf32 residue
// half of [W | W_lo] (only the streaming kernel reads it); wnv (optional)
// receives the new contraction input of this row (0 where nothing was written).
template <int NR, int MODE, bool kWLo = true>
__device__ __forceinline__ void tc_row_update(const TcArgs& a, int b, int rb, int row, int lane,
                                              int ep, const float (&gw)[NR],
                                              double (*s_part)[NR][3], int bar = 2,
                                              float* wnv = nullptr) {
    const StepScalars& sc = a.s;
    const int N = a.N;
    const int i = (a.rb0 + rb) * kTcRows + row;
    if (wnv) {
#pragma unroll
        for (int q = 0; q < NR; ++q) wnv[q] = 0.f;
    }
    bool fz[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        const int fg = a.fail_gstep[b * NR + q];
        if (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN)
            fz[q] = fg < a.alt->gstep_base + a.step;
        else
            fz[q] = fg != kFreeTraj;
    }
    const bool valid = i < N;
    const size_t si = (size_t)b * a.ldN + i;
    const size_t vi0 = si * NR;
    if constexpr (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) {
        float lmin[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) lmin[q] = INFINITY;
        if (valid) {
            float wv[NR], Rv[NR], cv[NR], ev[NR];
#pragma unroll
            for (int q = 0; q < NR; ++q) wv[q] = __ldg(a.Win + tc_wofs(a.ldJ, NR, b, i, q));
#pragma unroll
            for (int q = 0; q < NR; q += 4) {
                const float4 r4 = __ldg(reinterpret_cast<const float4*>(a.Rs + vi0 + q));
                const float4 c4 = *reinterpret_cast<const float4*>(a.C + vi0 + q);
                const float4 e4 = *reinterpret_cast<const float4*>(a.E + vi0 + q);
                Rv[q] = r4.x; Rv[q + 1] = r4.y; Rv[q + 2] = r4.z; Rv[q + 3] = r4.w;
                cv[q] = c4.x; cv[q + 1] = c4.y; cv[q + 2] = c4.z; cv[q + 3] = c4.w;
                ev[q] = e4.x; ev[q + 1] = e4.y; ev[q + 2] = e4.z; ev[q + 3] = e4.w;
            }
            const float Dv = __ldg(a.D + si), hzv = __ldg(a.hz + si);
            const float half_rt = (float)sc.half_rt, rt = (float)sc.rt, dt = (float)sc.dt;
            const float Kj = (float)sc.Kj, nbeta = (float)sc.nbeta, tau = (float)sc.tau;
            const double pd = a.pump ? a.pump[a.step] : a.p_scalar;
            const float loss = sc.minus_j != 0.0 ? (float)((-1.0 + pd) - sc.minus_j)
                                                 : (float)(-1.0 + pd);
            const float thresh = (float)a.alt->thresh;
            float cn[NR], en[NR];
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                const float c = cv[q], e = ev[q];
                const float Jw = Dv * wv[q] - gw[q];
                float h;
                if constexpr (MODE == EPI_STEP_BN)
                    h = half_rt * (Jw + hzv);
                else
                    h = Jw + half_rt * hzv;
                if (a.Hdbg) a.Hdbg[vi0 + q] = h;
                const float inj = (Kj * e) * (Rv[q] * h - thresh);
                cn[q] = c + dt * ((loss - c * c) * c + inj);
                en[q] = e + dt * ((nbeta * (c * c - tau)) * e);
                if (fz[q]) {
                    cn[q] = c;
                    en[q] = e;
                } else if (!isfinite(cn[q]) || !isfinite(en[q])) {
                    atomicMin(&a.fail_gstep[b * NR + q], a.alt->gstep_base + a.step);
                    atomicMin(&a.fail_idx[b * NR + q], i);
                    cn[q] = c;
                    en[q] = e;
                } else {
                    lmin[q] = en[q];
                    float wn;
                    if constexpr (MODE == EPI_STEP_BN)
                        wn = Rv[q] * (cn[q] > 0.f ? 1.f : 0.f);
                    else
                        wn = (Rv[q] * 0.25f) * (cn[q] + rt);
                    a.Wout[tc_wofs(a.ldJ, NR, b, i, q)] = wn;
                    if (kWLo) a.Wout[tc_wofs(a.ldJ, NR, b, i, NR + q)] = wn - trunc_tf32(wn);
                    if (wnv) wnv[q] = wn;
                }
            }
#pragma unroll
            for (int q = 0; q < NR; q += 4) {
                *reinterpret_cast<float4*>(a.C + vi0 + q) =
                    make_float4(cn[q], cn[q + 1], cn[q + 2], cn[q + 3]);
                *reinterpret_cast<float4*>(a.E + vi0 + q) =
                    make_float4(en[q], en[q + 1], en[q + 2], en[q + 3]);
            }
        }
        // per-replica min of e: warp reduce, one atomic per (warp, replica)
#pragma unroll
        for (int q = 0; q < NR; ++q) {
            float m = lmin[q];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
                m = fminf(m, __shfl_xor_sync(0xffffffffu, m, off));
            if (lane == q && m != INFINITY) atomicMin(&a.minE[b * NR + q], ord_key(m));
        }
    } else if constexpr (MODE == EPI_JACOBI) {
        if (valid) {
            const float Dv = __ldg(a.D + si), bv = __ldg(a.hz + si);
            const float omd = (float)sc.one_minus_dtc, dtc = (float)sc.dt_c;
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                if (fz[q]) continue;
                const float Rv = a.Rs[vi0 + q];
                const bool on = a.sigma[vi0 + q] != 0;
                float rn = Rv;
                if (on) {
                    if (Dv == 0.f) {
                        atomicMin(a.err, i);
                        continue;
                    }
                    const float off = gw[q] - Dv * Rv;
                    rn = omd * Rv + dtc * ((bv - off) / Dv);
                    a.Rs[vi0 + q] = rn;
                }
                const float wn = rn * (on ? 1.f : 0.f);
                a.Wout[tc_wofs(a.ldJ, NR, b, i, q)] = wn;
                if (kWLo) a.Wout[tc_wofs(a.ldJ, NR, b, i, NR + q)] = wn - trunc_tf32(wn);
                if (wnv) wnv[q] = wn;
            }
        }
    } else if constexpr (MODE == EPI_MATVEC) {
        if (valid) {
#pragma unroll
            for (int q = 0; q < NR; ++q)
                if (!fz[q]) a.Mv[vi0 + q] = (double)gw[q];
        }
    } else {  // EPI_SCORE
        double pa[NR], pb[NR], pc[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) {
            pa[q] = pb[q] = pc[q] = 0.0;
            if (valid && !fz[q]) {
                const double wv = a.Win[tc_wofs(a.ldJ, NR, b, i, q)];
                pa[q] = wv * (double)gw[q];
                pb[q] = (double)a.hz[si] * wv;
                if (a.xtrue) {
                    const double xt = a.xitrue[si] ? a.xtrue[si] : 0.0;
                    pc[q] = (wv - xt) * (wv - xt);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                pa[q] += __shfl_xor_sync(0xffffffffu, pa[q], off);
                pb[q] += __shfl_xor_sync(0xffffffffu, pb[q], off);
                pc[q] += __shfl_xor_sync(0xffffffffu, pc[q], off);
            }
        }
        if (lane < NR) {
            s_part[ep][lane][0] = pa[lane];
            s_part[ep][lane][1] = pb[lane];
            s_part[ep][lane][2] = pc[lane];
        }
        asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
        if (ep == 0 && lane < NR) {
            double A_ = 0, B_ = 0, C_ = 0;
            for (int w = 0; w < 4; ++w) {
                A_ += s_part[w][lane][0];
                B_ += s_part[w][lane][1];
                C_ += s_part[w][lane][2];
            }
            double* p = a.part + (((size_t)b * a.nRB + rb) * NR + lane) * 4;
            p[0] = A_;
            p[1] = B_;
            p[2] = C_;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
    }
}

template <int NR, int MODE>
__global__ void __launch_bounds__(kTcThreads, 1) tc_step_kernel(TcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr uint32_t kABytes = kTcTileFloats * 4;            // 32 KB
    constexpr uint32_t kBBytes = kTcChunk * 2 * NR * 4;        // 8 KB (NR=16)
    constexpr uint32_t kStageBytes = kABytes + kBBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTcStages * kStageBytes);
    uint64_t* full = bars;                  // [S]  TMA landed
    uint64_t* empty = bars + kTcStages;     // [S]  MMAs of the stage retired
    uint64_t* lo_full = empty + kTcStages;  // [2]  G_lo in TMEM
    uint64_t* lo_empty = lo_full + 2;       // [2]  MMAs reading G_lo retired
    uint64_t* tm_full = lo_empty + 2;       // [2]  accumulator complete
    uint64_t* tm_empty = tm_full + 2;       // [2]  accumulator drained
    __shared__ uint32_t s_tmem;
    __shared__ double s_part[4][NR][3];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N, nch = a.nch;
    const int nchunks = (N + kTcChunk - 1) / kTcChunk;  // chunks actually streamed

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&lo_full[k], 4);
            mbar_init(&lo_empty[k], 1);
            mbar_init(&tm_full[k], 1);
            mbar_init(&tm_empty[k], 4);
        }
        mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kTcTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        // ------------------------------------------------------ producer
        if (lane == 0) {
            int g = 0;
            for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
                const int b = tile / a.nRB, rb = tile % a.nRB;
                const float* Gp = a.G + ((size_t)b * a.nRB + rb) * nch * kTcTileFloats;
                const float* Wp = a.Win + (size_t)b * a.ldJ * 2 * NR;
                for (int c = 0; c < nchunks; ++c, ++g) {
                    const int s = g % kTcStages;
                    if (g >= kTcStages) mbar_wait(&empty[s], ((g / kTcStages) - 1) & 1);
                    unsigned char* st = smem + s * kStageBytes;
                    mbar_arrive_expect_tx(&full[s], kStageBytes);
                    bulk_g2s(st, Gp + (size_t)c * kTcTileFloats, kABytes, &full[s]);
                    bulk_g2s(st + kABytes, Wp + (size_t)c * kTcChunk * 2 * NR, kBBytes, &full[s]);
                }
            }
        }
    } else if (warp <= 4) {
        // ------------------------------- split: G_lo = G - trunc(G) -> TMEM
        const int quad = warp & 3;          // TMEM lane quadrant of this warp
        const int m = quad * 32 + lane;     // A row handled by this thread
        int g = 0;
        for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
            for (int c = 0; c < nchunks; ++c, ++g) {
                const int s = g % kTcStages, k = g & 1;
                mbar_wait(&full[s], (g / kTcStages) & 1);
                if (g >= 2) mbar_wait(&lo_empty[k], ((g / 2) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const float* At = reinterpret_cast<const float*>(smem + s * kStageBytes) +
                                  (m / 8) * 32 + (m % 8) * 4;
                const uint32_t tdst = tmem + ((uint32_t)(quad * 32) << 16) + kTcLoCol + k * 64;
#pragma unroll
                for (int h = 0; h < 4; ++h) {  // 16 j per tcgen05.st
                    uint32_t v[16];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float4 x = *reinterpret_cast<const float4*>(At + (h * 4 + u) * 512);
                        v[4 * u + 0] = __float_as_uint(x.x - trunc_tf32(x.x));
                        v[4 * u + 1] = __float_as_uint(x.y - trunc_tf32(x.y));
                        v[4 * u + 2] = __float_as_uint(x.z - trunc_tf32(x.z));
                        v[4 * u + 3] = __float_as_uint(x.w - trunc_tf32(x.w));
                    }
                    tmem_st16(tdst + h * 16, v);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&lo_full[k]);
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t id_cat = tc_idesc(2 * NR), id_hi = tc_idesc(NR);
            constexpr uint32_t lboB = 4 * 2 * NR * 4;  // K-group stride of [W | W_lo]
            int g = 0, tt = 0;
            for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++tt) {
                const int acc = tt & 1;
                if (tt >= 2) mbar_wait(&tm_empty[acc], ((tt / 2) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dtm = tmem + acc * 2 * NR;
                for (int c = 0; c < nchunks; ++c, ++g) {
                    const int s = g % kTcStages, k = g & 1;
                    mbar_wait(&full[s], (g / kTcStages) & 1);
                    mbar_wait(&lo_full[k], (g / 2) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t aH = smem_u32(smem + s * kStageBytes);
                    const uint32_t bW = aH + kABytes;
                    const uint32_t tLo = tmem + kTcLoCol + k * 64;
#pragma unroll
                    for (int kb = 0; kb < kTcChunk / 8; ++kb) {
                        // K = 8 per MMA = two 4-wide K groups
                        const uint64_t dA = umma_desc(aH + kb * 2 * 2048, 2048, 128);
                        const uint64_t dB = umma_desc(bW + kb * 2 * lboB, lboB, 128);
                        const uint32_t first = (c | kb) ? 1u : 0u;
                        tc_mma_ss(dtm, dA, dB, id_cat, first);      // G_hi [W | W_lo]
                        tc_mma_ts(dtm, tLo + kb * 8, dB, id_hi, 1u);  // G_lo W
                    }
                    tc_commit(&empty[s]);
                    tc_commit(&lo_empty[k]);
                }
                tc_commit(&tm_full[acc]);
            }
        }
    } else {
        // ------------------------------------------------------ epilogue
        const int ew = warp & 3;                // TMEM lane quadrant of this warp
        const int row = ew * 32 + lane;         // spin row inside the tile
        const int ep = warp - 6;                // 0..3, stable order for reductions
        int tt = 0;
        for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++tt) {
            const int acc = tt & 1;
            const int b = tile / a.nRB, rb = tile % a.nRB;
            mbar_wait(&tm_full[acc], (tt / 2) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            float gw[NR];
            tmem_ld_row<NR>(tmem + acc * 2 * NR + ((uint32_t)(ew * 32) << 16), gw);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tm_empty[acc]);

            tc_row_update<NR, MODE>(a, b, rb, row, lane, ep, gw, s_part);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTcTmemCols));
}

constexpr size_t tc_smem_bytes(int NR) {
    return (size_t)kTcStages * (kTcTileFloats * 4 + 2 * kTcChunk * NR * 4) + 16 * 8 + 64;
}

// canonical tcgen05 A-operand output of the gram builder (fp32)
struct TcPanelOut {
    float* G;
    int nRB, nch, row0;  // nRB: local row blocks; row0: first local row
    __device__ __forceinline__ void store(int b, int i, int j, double v) const {
        G[tc_gofs(nRB, nch, b, i - row0, j)] = (float)v;
    }
};

// G panels in the canonical A layout, fp32 (gram rounded from the fp64 chain)
__global__ void __launch_bounds__(256) tc_gram_kernel(const double* __restrict__ A, int M, int N,
                                                      size_t a_stride, float* G, int nRB,
                                                      int nch) {
    const int b = blockIdx.z;
    const int bi = blockIdx.y, bj = blockIdx.x;
    if (bj < bi) return;
    const double* Ab = A + (size_t)b * a_stride;
    __shared__ double As[kGK][kGT + 2];
    __shared__ double Bs[kGK][kGT + 2];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int i0 = bi * kGT, j0 = bj * kGT;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    const int lc = threadIdx.x / 4, lk = (threadIdx.x % 4) * 4;
    for (int k0 = 0; k0 < M; k0 += kGK) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = k0 + lk + u;
            const int ci = i0 + lc, cj = j0 + lc;
            As[lk + u][lc] = (k < M && ci < N) ? Ab[(size_t)ci * M + k] : 0.0;
            Bs[lk + u][lc] = (k < M && cj < N) ? Ab[(size_t)cj * M + k] : 0.0;
        }
        __syncthreads();
        const int kn = min(kGK, M - k0);
        for (int kk = 0; kk < kn; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = As[kk][ty * 4 + r];
#pragma unroll
            for (int c = 0; c < 4; ++c) bv[c] = Bs[kk][tx * 4 + c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = __fma_rn(av[r], bv[c], acc[r][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int i = i0 + ty * 4 + r, j = j0 + tx * 4 + c;
            if (i < N && j < N) {
                const float v = (float)acc[r][c];
                G[tc_gofs(nRB, nch, b, i, j)] = v;
                G[tc_gofs(nRB, nch, b, j, i)] = v;
            }
        }
}

}  // namespace cimcs
