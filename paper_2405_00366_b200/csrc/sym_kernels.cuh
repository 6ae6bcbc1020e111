// sym_kernels.cuh -- fp32 fused MFZ step that reads each gram entry ONCE per
// step by exploiting G = G^T (tcgen05 kind::f16, fp16 hi/lo split).
//
// The streaming kernel (tc_kernels.cuh) is bound by HBM bytes: every step
// reads the whole N x N gram.  Here only the upper-triangle 128 x 128 tiles
// (I <= J) are stored, and one tile in shared memory feeds TWO products:
//     use 1:  out[I] += G[I,J]   * w[J]     A = tile, K-major
//     use 2:  out[J] += G[I,J]^T * w[I]     A = the same bytes as an MN-major
//                                           operand (tools/tc_probe_f16.cu)
// which halves the gram bytes per step.  The transposed view needs a 16-bit
// MMA kind (tf32 is K-major only), so fp32 accuracy is kept with a split
//     x ~= hi + lo,  hi = fp16(x * 2^s), lo = fp16(x * 2^s - hi)   (~22 bits)
// with exact power-of-two scales: s_G per instance (max |G| = max diag in
// [2^14, 2^15)) and s_w per (128-row block, replica) computed on the fly, so
// no value leaves fp16's normal range.  G w ~= G_hi [w_hi | w_lo] + G_lo w_hi,
// accumulated in fp32 in TMEM, and unscaled exactly.
//
// Work is split into super-block ITEMS of up to kSyS x kSyS tiles (rows
// [I0, I0 + kSyS) x columns [J0, J0 + kSyS) of the tile triangle).  The tile
// epilogue sums the unscaled products of an item in registers, so an item
// emits one partial per row block (use 1) and one per column block (use 2)
// instead of one per tile and use: a row block K receives nSB = ceil(nRB /
// kSyS) partials, written to [B][nRB][slot = nSB][128][NR] (4x fewer bytes at
// N = 2000, small enough to stay in L2 until the update reads them).  Items
// are placed on the persistent CTAs by a host LPT schedule (largest first onto
// the least-loaded CTA), so every role of a CTA walks the same static list.
// A second, evenly spread kernel (sym_update_kernel, one CTA per block, 4
// replicas per thread) sums the slots in a FIXED order (deterministic) and runs
// the fused Euler / Jacobi / score / matvec update (the arithmetic of
// tc_row_update of round 1); no CTA waits for another.
// (Fusing the finish into the tile kernel -- last-arriving CTA, or owner-CTA
// finisher warps with an L2-resident ring of partials -- was measured slower:
// each finish is a chain of dependent L2 round trips behind the tile stream.)
//
// The contraction input w is kept, next to the fp32 [W | W_lo] array the other
// kernels use, as per-block fp16 B tiles [w_hi | w_lo] (2NR x 128, canonical
// K-major) with one scale exponent per (block, replica): written once per
// block by the finisher that produces w (or by sym_wconvert_kernel after any
// other writer), so a tile only bulk-copies them.
//
// Persistent, warp-specialised CTA (one per SM, 6 warps):
//   warp 0      producer: per tile bulk copies of G_hi, G_lo (32 KB each) and
//               the two 8 KB B tiles
//   warp 1      MMA issuer: 8 k-steps x (2 + 2) MMAs, kSyAcc (4) TMEM accumulators
//   warps 2-5   tile epilogue: TMEM -> unscaled products, summed per item
#pragma once

#include <cuda_fp16.h>

#include "tc_kernels.cuh"

namespace cimcs {

#ifndef SY_UPD_OCC
#define SY_UPD_OCC 2  // update-kernel CTAs per SM the register cap allows (3 / 4 spill; measured)
#endif
constexpr int kSyT = 128;                              // tile edge
constexpr int kSyStages = 2;
constexpr int kSyPlaneHalfs = kSyT * kSyT;             // 16384
constexpr uint32_t kSyPlaneBytes = kSyPlaneHalfs * 2;  // 32 KB
constexpr int kSyThreads = 6 * 32;
constexpr int kSyS = 4;                                // item edge in tiles
constexpr int kSyAcc = 4;                              // TMEM accumulator buffers (4 vs 2: 104.8 vs 105.3 us per step)
constexpr int kSyBarBytes = 256;                       // mbarriers after the stages
template <int NR>
__host__ __device__ constexpr int sy_tmem_cols() { return kSyAcc * 4 * NR; }  // 256 (NR 16) / 128 (NR 8)

// byte offset of element (mn, k) of an fp16 operand in the canonical no-swizzle
// K-major layout (core matrix = 8 MN rows x 8 K = 16 bytes per row)
__host__ __device__ inline int sy_offk(int mn, int k, int MN) {
    return (k / 8) * (MN / 8) * 128 + (mn / 8) * 128 + (mn % 8) * 16 + (k % 8) * 2;
}
// index of tile (I, J), I <= J, in the row-major upper triangle of nRB x nRB
__host__ __device__ inline int sy_tri(int I, int J, int nRB) {
    return I * nRB - I * (I - 1) / 2 + (J - I);
}

// gram builder output: tile (i/128, j/128) of the upper triangle, planes hi|lo
struct SymOut {
    __half* G;
    const int* sg;  // per-instance scale exponent
    int nRB, ntri;
    __device__ __forceinline__ void store(int b, int i, int j, double v) const {
        const int I = i / kSyT, J = j / kSyT;
        if (I > J) return;
        __half* t = G + ((size_t)b * ntri + sy_tri(I, J, nRB)) * 2 * kSyPlaneHalfs;
        const int o = sy_offk(i % kSyT, j % kSyT, kSyT) / 2;
        const double gs = ldexp(v, sg[b]);
        const __half hi = __double2half(gs);
        t[o] = hi;
        t[kSyPlaneHalfs + o] = __double2half(gs - (double)__half2float(hi));
    }
};

// e such that m * 2^e is in [2^14, 2^15) (0 for m = 0 / non-finite / subnormal),
// clamped to [-100, 100]
__host__ __device__ inline int sy_exp14(float m) {
    if (!(m > 0.f) || !(m < INFINITY)) return 0;
    int u;
    memcpy(&u, &m, 4);
    const int ex = (u >> 23) & 0xff;  // biased exponent
    const int e = ex == 0 ? 0 : 14 - (ex - 127);
    return e < -100 ? -100 : (e > 100 ? 100 : e);  // 2^-(s_G + s_w) stays representable
}
// exact 2^e as a float, |e| <= 126
__device__ __forceinline__ float sy_pow2(int e) { return __int_as_float((127 + e) << 23); }

// s_G[b]: max |G| (= max diag) * 2^s_G in [2^14, 2^15)
template <typename TS>
__global__ void sym_scale_kernel(const TS* __restrict__ D, int N, int ldN, int* sg) {
    const int b = blockIdx.x;
    float m = 0.f;
    for (int i = threadIdx.x; i < N; i += blockDim.x) m = fmaxf(m, fabsf((float)D[(size_t)b * ldN + i]));
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    __shared__ float s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, s[w]);
        m = fmaxf(m, s[0]);
        sg[b] = sy_exp14(m);
    }
}

__host__ __device__ constexpr uint32_t sy_idesc(int n, int amn) {
    return (1u << 4) | ((uint32_t)amn << 15) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(kSyT >> 4) << 24);  // F32 accumulate, A = B = F16
}
__device__ __forceinline__ void sy_mma(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ bool sy_elect_one() { return elect_one_sync(); }
__device__ __forceinline__ uint64_t sy_policy_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t sy_policy_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// programmatic dependent launch (no-ops without the launch attribute)
__device__ __forceinline__ void sy_pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void sy_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// bulk copy global -> shared with an L2 eviction-priority hint
__device__ __forceinline__ void sy_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// the same with shared addresses as 32-bit values (warp-uniform: uniform registers)
__device__ __forceinline__ void sy_bulk_u(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void sy_expect_tx_u(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void sy_st_last(float4* p, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}

struct SymArgs {
    TcArgs t;              // state, scalars, fp32 W (other kernels), outputs
    const __half* Gs;      // [B][ntri][hi | lo][128 x 128]
    const int* sg;         // [B]
    const __half* WBin;    // [B][nRB][2NR x 128] fp16 B tiles of the input w
    const int* WSin;       // [B][nRB][NR] their scale exponents
    __half* WBout;         // same for the output w (step / Jacobi modes)
    int* WSout;
    float* spart;          // [B][nRB][nSB][128][NR]
    const int2* items;     // (b - b0, P << 16 | Q): super-block (P, Q), P <= Q
    const int* sched;      // [grid + 1] item range of each CTA
    int ntri, nSB;         // tiles per instance, super-blocks per row
    int b0;                // first instance of this launch (instance groups)
    int keep_w;            // step modes: also store the fp32 w (a consumer reads it)
    int gram_keep;         // tiles t < gram_keep of each triangle copied with evict_last
    int S;                 // item edge in tiles (kSyS; 2 for the compacted refit)
    const int* rowmap;     // compacted refit: row -> original spin (error reports), or null
    // measurement aid (option "timeline"): %globaltimer stamps of the last launch pair,
    // 4 per CTA: tile CTA x at [x] = (entry, past the PDL wait, last item stored, SM id << 32 | tiles),
    // update CTA (K, b) at [kTlUpd + b * nRB + K] = (entry, past the PDL wait, exit, -)
    unsigned long long* tlog;
};
// per-tile stamps of tile CTA 0 at [kTlTile + tt] = (MMA thread: accumulator free, tile
// landed, MMAs issued; producer: refill of the tile's stage issued) and [kTlTile + 128 +
// tt] = (epilogue warp 2: accumulator complete, accumulator read + released, -, -)
constexpr int kTlUpd = 256, kTlTile = 8192, kTlCap = kTlTile + 256;
__device__ __forceinline__ unsigned long long sy_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int NR>
__host__ __device__ constexpr size_t sy_bbytes() { return (size_t)2 * NR * kSyT * 2; }
template <int NR>
__host__ __device__ constexpr size_t sy_stage_bytes() {
    return 2 * (size_t)kSyPlaneBytes + 2 * sy_bbytes<NR>();
}
template <int NR>
__host__ __device__ constexpr size_t sy_smem_bytes() {
    return kSyStages * sy_stage_bytes<NR>() + kSyBarBytes + (size_t)kSyS * NR * kSyT * 4;
}

// item k -> instance, first row / column block, extents
struct SyItem {
    int b, P, Q, I0, J0, nI, nJ;
    bool diag;
};
__device__ __forceinline__ SyItem sy_item(const SymArgs& sa, int k, int nRB) {
    const int2 it = sa.items[k];
    SyItem r;
    r.b = sa.b0 + it.x;
    r.P = it.y >> 16;
    r.Q = it.y & 0xffff;
    r.I0 = r.P * sa.S;
    r.J0 = r.Q * sa.S;
    r.nI = min(sa.S, nRB - r.I0);
    r.nJ = min(sa.S, nRB - r.J0);
    r.diag = r.P == r.Q;
    return r;
}

// fp16 hi/lo split of w * 2^e (e from the per-replica block max): exact scaling,
// rounded to nearest in both halves (a double input is split from its double
// value)
__device__ __forceinline__ void sy_split(float w, int e, __half& hi, __half& lo) {
    const float ws = w * sy_pow2(e);
    hi = __float2half_rn(ws);
    lo = __float2half_rn(ws - __half2float(hi));
}
__device__ __forceinline__ void sy_split(double w, int e, __half& hi, __half& lo) {
    const double ws = ldexp(w, e);
    hi = __double2half(ws);
    lo = __double2half(ws - (double)__half2float(hi));
}

// fp16 B tile + scales of one 128-row block from the values w[q] of row k
// (called by all 128 threads of a group synchronised on named barrier `bar`).
template <int NR, typename TS>
__device__ __forceinline__ void sy_emit_block(const TS (&w)[NR], int k, int lane, int wq,
                                              unsigned (*s_max)[NR], __half* WB, int* WS,
                                              int bar) {
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        const unsigned m =
            __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf((float)w[q])));
        if (lane == 0) s_max[wq][q] = m;
    }
    asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        const unsigned m = max(max(s_max[0][q], s_max[1][q]), max(s_max[2][q], s_max[3][q]));
        const int e = sy_exp14(__uint_as_float(m));
        __half hi, lo;
        sy_split(w[q], e, hi, lo);
        unsigned char* B = reinterpret_cast<unsigned char*>(WB);
        *reinterpret_cast<__half*>(B + sy_offk(q, k, 2 * NR)) = hi;
        *reinterpret_cast<__half*>(B + sy_offk(NR + q, k, 2 * NR)) = lo;
        if (k == q) WS[q] = e;
    }
    asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");  // s_max reusable
}

// B tiles of a whole W array [b][i][r] -- after any writer of W other than
// the symmetric update kernel (init, support, mask, CG).
template <int NR, typename TS>
__global__ void __launch_bounds__(128) sym_wconvert_kernel(const TS* __restrict__ W, int N,
                                                           int ldN, int nRB, __half* WB, int* WS) {
    __shared__ unsigned s_max[4][NR];
    const int X = blockIdx.x, b = blockIdx.y, k = threadIdx.x;
    const int j = X * kSyT + k;
    TS w[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) w[q] = j >= N ? TS(0) : W[((size_t)b * ldN + j) * NR + q];
    sy_emit_block<NR, TS>(w, k, k & 31, k >> 5, s_max,
                          WB + ((size_t)b * nRB + X) * (2 * NR * kSyT),
                          WS + ((size_t)b * nRB + X) * NR, 1);
}

template <int NR, int MODE>
__global__ void __launch_bounds__(kSyThreads, 1) sym_step_kernel(SymArgs sa) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr uint32_t kBB = (uint32_t)sy_bbytes<NR>();
    constexpr uint32_t kStage = (uint32_t)sy_stage_bytes<NR>();
    constexpr int kCols = sy_tmem_cols<NR>();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSyStages * kStage);
    uint64_t* full = bars;                    // [2] G planes + B tiles landed
    uint64_t* empty = full + kSyStages;       // [2] MMAs of the stage retired
    uint64_t* tm_full = empty + kSyStages;    // [kSyAcc] accumulators complete
    uint64_t* tm_empty = tm_full + kSyAcc;    // [kSyAcc] accumulators drained
    __shared__ uint32_t s_tmem;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nRB = sa.t.nRB;
    const int it0 = sa.sched[blockIdx.x], it1 = sa.sched[blockIdx.x + 1];

    if (threadIdx.x == 0) {
        for (int s = 0; s < kSyStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int k = 0; k < kSyAcc; ++k) {
            mbar_init(&tm_full[k], 1);
            mbar_init(&tm_empty[k], 4);
        }
        mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    // programmatic dependent launch: the update kernel may be scheduled now (its
    // CTAs wait for this grid in griddepcontrol.wait); this grid's own reads of
    // w and writes of the partial products wait for the previous update kernel.
    // In the step modes the producer warp waits later: every CIM call starts
    // with a plain (non-PDL) launch issued after the gram was built, and nothing
    // writes the gram tiles during the call, so the planes of the first stages
    // are copied while the previous update kernel finishes.
    constexpr bool kEarly = MODE == EPI_STEP_BN || MODE == EPI_STEP_CN;
    if (sa.tlog && threadIdx.x == 0) sa.tlog[blockIdx.x * 4 + 0] = sy_gtime();
    sy_pdl_trigger();
    if (!kEarly || warp != 0) sy_pdl_wait();

    if (warp == 0) {
        // ------------------------------------------------------ producer
        // (convergent warp, warp-uniform operands, one elected lane issues: see the
        // MMA issuer below for why)
        const uint64_t pGf = sy_policy_first(), pW = sy_policy_last();
        const uint32_t smem0 = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
        const uint32_t full0 = __shfl_sync(0xffffffffu, smem_u32(full), 0);
        const int k0 = __shfl_sync(0xffffffffu, it0, 0), k1 = __shfl_sync(0xffffffffu, it1, 0);
        // this CTA's item descriptors, one per lane, loaded BEFORE the PDL wait: right after
        // it the memory system is busy with the update kernel's write-back and a dependent
        // global load on the way to the first w copies measured 1 - 2 us
        const int2 mine = lane < k1 - k0 ? sa.items[k0 + lane] : make_int2(0, 0);
        auto item_u = [&](int k, int& b, int& I0, int& J0, int& nI, int& nJ, bool& diag) {
            int2 itv;
            if (k - k0 < 32) {
                itv.x = __shfl_sync(0xffffffffu, mine.x, k - k0);
                itv.y = __shfl_sync(0xffffffffu, mine.y, k - k0);
            } else {
                itv = sa.items[k];
            }
            b = sa.b0 + __shfl_sync(0xffffffffu, itv.x, 0);
            const int iy = __shfl_sync(0xffffffffu, itv.y, 0);
            const int P = iy >> 16, Q = iy & 0xffff;
            I0 = P * sa.S;
            J0 = Q * sa.S;
            nI = min(sa.S, nRB - I0);
            nJ = min(sa.S, nRB - J0);
            diag = P == Q;
        };
        // stage s of a tile: expect its bytes, copy the two gram planes
        auto g_part = [&](int s, int b, int I, int J) {
            const int tri = sy_tri(I, J, nRB);
            const __half* src = sa.Gs + ((size_t)b * sa.ntri + tri) * 2 * kSyPlaneHalfs;
            const uint64_t pG = tri < sa.gram_keep ? pW : pGf;
            if (sy_elect_one()) {
                const uint32_t st = smem0 + s * kStage, fb = full0 + s * 8;
                sy_expect_tx_u(fb, 2 * kSyPlaneBytes + (I != J ? 2 : 1) * kBB);
                // the gram streams through L2 once per step; w tiles are re-read
                sy_bulk_u(st, src, kSyPlaneBytes, fb, pG);
                sy_bulk_u(st + kSyPlaneBytes, src + kSyPlaneHalfs, kSyPlaneBytes, fb, pG);
            }
            __syncwarp();
        };
        int tt = 0;
        for (int k = k0; k < k1 && tt < kSyStages; ++k) {
            int b, I0, J0, nI, nJ;
            bool diag;
            item_u(k, b, I0, J0, nI, nJ, diag);
            for (int ii = 0; ii < nI && tt < kSyStages; ++ii)
                for (int jj = diag ? ii : 0; jj < nJ && tt < kSyStages; ++jj, ++tt)
                    g_part(tt, b, I0 + ii, J0 + jj);
        }
        if (kEarly) sy_pdl_wait();
        if (sa.tlog && lane == 0) sa.tlog[blockIdx.x * 4 + 1] = sy_gtime();
        tt = 0;
        for (int k = k0; k < k1; ++k) {
            int b, I0, J0, nI, nJ;
            bool diag;
            item_u(k, b, I0, J0, nI, nJ, diag);
            const __half* wb = sa.WBin + (size_t)b * nRB * (2 * NR * kSyT);
            for (int ii = 0; ii < nI; ++ii)
                for (int jj = diag ? ii : 0; jj < nJ; ++jj, ++tt) {
                    const int I = I0 + ii, J = J0 + jj, s = tt % kSyStages;
                    if (tt >= kSyStages) {
                        mbar_wait(&empty[s], ((tt / kSyStages) - 1) & 1);
                        g_part(s, b, I, J);
                    }
                    if (sa.tlog && blockIdx.x == 0 && tt < 128 && lane == 0)
                        sa.tlog[(kTlTile + tt) * 4 + 3] = sy_gtime();
                    if (sy_elect_one()) {
                        const uint32_t st = smem0 + s * kStage, fb = full0 + s * 8;
                        sy_bulk_u(st + 2 * kSyPlaneBytes, wb + (size_t)J * (2 * NR * kSyT), kBB, fb, pW);
                        if (I != J)
                            sy_bulk_u(st + 2 * kSyPlaneBytes + kBB, wb + (size_t)I * (2 * NR * kSyT),
                                      kBB, fb, pW);
                    }
                    __syncwarp();
                }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        // The whole warp walks the tile list convergently and every operand is
        // warp-uniform (loaded values go through __shfl_sync(.., 0) so the compiler
        // keeps them in uniform registers); one elected lane issues.  Issuing from
        // inside an `if (lane == 0)` branch instead made ptxas wrap EVERY tcgen05.mma
        // in an ELECT / 5 x R2UR / BRA.U.ANY loop: 1.37 us of issue per tile, which
        // bound the whole kernel (tools/tile_pipeline.py).
        constexpr uint32_t id_cat = sy_idesc(2 * NR, 0), id_hi = sy_idesc(NR, 0);
        constexpr uint32_t id_catT = sy_idesc(2 * NR, 1), id_hiT = sy_idesc(NR, 1);
        constexpr uint32_t kstr = (kSyT / 8) * 128;   // K-group stride of the tile (2 KB)
        constexpr uint32_t lboB = (2 * NR / 8) * 128;  // K-group stride of a B tile
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
        const uint32_t smem0 = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
        const int k0 = __shfl_sync(0xffffffffu, it0, 0), k1 = __shfl_sync(0xffffffffu, it1, 0);
        int tt = 0;
        for (int k = k0; k < k1; ++k) {
            const int2 itv = sa.items[k];
            const int iy = __shfl_sync(0xffffffffu, itv.y, 0);
            const int P = iy >> 16, Q = iy & 0xffff;
            const int nI = min(sa.S, nRB - P * sa.S), nJ = min(sa.S, nRB - Q * sa.S);
            const bool diag = P == Q;
            for (int ii = 0; ii < nI; ++ii)
                for (int jj = diag ? ii : 0; jj < nJ; ++jj, ++tt) {
                    const int s = tt % kSyStages, acc = tt % kSyAcc;
                    const bool off = !(diag && ii == jj);
                    const bool tlt = sa.tlog && blockIdx.x == 0 && tt < 128 && lane == 0;
                    if (tt >= kSyAcc) mbar_wait(&tm_empty[acc], ((tt / kSyAcc) - 1) & 1);
                    if (tlt) sa.tlog[(kTlTile + tt) * 4 + 0] = sy_gtime();
                    mbar_wait(&full[s], (tt / kSyStages) & 1);
                    if (tlt) sa.tlog[(kTlTile + tt) * 4 + 1] = sy_gtime();
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t aHi = smem0 + s * kStage, aLo = aHi + kSyPlaneBytes;
                    const uint32_t bJ = aHi + 2 * kSyPlaneBytes, bI = bJ + kBB;
                    const uint32_t d1 = tmem_u + acc * 4 * NR, d2 = d1 + 2 * NR;
                    // descriptors of k-step 0; a k-step only moves the 14-bit start
                    // address field (>> 4), which cannot carry out (smem < 256 KB)
                    const uint64_t dA1h = umma_desc(aHi, kstr, 128), dA1l = umma_desc(aLo, kstr, 128);
                    const uint64_t dA2h = umma_desc(aHi, 128, kstr), dA2l = umma_desc(aLo, 128, kstr);
                    const uint64_t dBJ0 = umma_desc(bJ, lboB, 128), dBI0 = umma_desc(bI, lboB, 128);
                    if (sy_elect_one()) {
#pragma unroll
                        for (int kb = 0; kb < kSyT / 16; ++kb) {
                            const uint32_t first = kb ? 1u : 0u;
                            const uint64_t dBJ = dBJ0 + (uint64_t)(kb * 2 * lboB >> 4);
                            sy_mma(d1, dA1h + (uint64_t)(kb * 2 * kstr >> 4), dBJ, id_cat, first);
                            sy_mma(d1, dA1l + (uint64_t)(kb * 2 * kstr >> 4), dBJ, id_hi, 1u);
                            if (off) {  // transposed view: K' = tile rows, 16 per k-step = 256 B
                                const uint64_t dBI = dBI0 + (uint64_t)(kb * 2 * lboB >> 4);
                                sy_mma(d2, dA2h + (uint64_t)(kb * 256 >> 4), dBI, id_catT, first);
                                sy_mma(d2, dA2l + (uint64_t)(kb * 256 >> 4), dBI, id_hiT, 1u);
                            }
                        }
                        tc_commit(&empty[s]);
                        tc_commit(&tm_full[acc]);
                    }
                    __syncwarp();
                    if (tlt) sa.tlog[(kTlTile + tt) * 4 + 2] = sy_gtime();
                }
        }
    } else {
        // ------------------------------------------------ tile epilogue
        // Thread `row` owns row `row` of every row block of the item (use 1)
        // and column `row` of every column block (use 2); products are unscaled
        // exactly (2^-(s_G + s_w)) and summed per item in tile order: the row
        // block in registers, the column blocks in shared memory (own row only,
        // [kSyS][NR][128]: conflict-free), so the loops need no unrolling.
        const int ew = warp & 3;         // TMEM lane quadrant of this warp
        const int row = ew * 32 + lane;
        const uint64_t pP = sy_policy_last();
        const int nSB = sa.nSB;
        float* cs = reinterpret_cast<float*>(smem + kSyStages * kStage + kSyBarBytes) + row;
        auto put = [&](int b, int K, int slot, const float (&v)[NR]) {
            float4* p = reinterpret_cast<float4*>(
                sa.spart + ((((size_t)b * nRB + K) * nSB + slot) * kSyT + row) * NR);
#pragma unroll
            for (int q = 0; q < NR; q += 4)
                sy_st_last(p + q / 4, make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]), pP);
        };
        auto put_cs = [&](int b, int K, int slot, int jj) {
            float v[NR];
#pragma unroll
            for (int q = 0; q < NR; ++q) v[q] = cs[(jj * NR + q) * kSyT];
            put(b, K, slot, v);
        };
        int tt = 0;
        for (int k = it0; k < it1; ++k) {
            const SyItem m = sy_item(sa, k, nRB);
            const float fG = sy_pow2(-sa.sg[m.b]);
            const int* ws = sa.WSin + (size_t)m.b * nRB * NR;
            for (int jj = 0; jj < m.nJ; ++jj)
#pragma unroll
                for (int q = 0; q < NR; ++q) cs[(jj * NR + q) * kSyT] = 0.f;
            for (int ii = 0; ii < m.nI; ++ii) {
                float racc[NR];
#pragma unroll
                for (int q = 0; q < NR; ++q) racc[q] = 0.f;
                for (int jj = m.diag ? ii : 0; jj < m.nJ; ++jj, ++tt) {
                    const int I = m.I0 + ii, J = m.J0 + jj;
                    const bool off = I != J;
                    const int acc = tt % kSyAcc;
                    mbar_wait(&tm_full[acc], (tt / kSyAcc) & 1);
                    const bool tle = sa.tlog && blockIdx.x == 0 && tt < 128 && row == 0;
                    if (tle) sa.tlog[(kTlTile + 128 + tt) * 4 + 0] = sy_gtime();
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    float g1[NR], g2[NR];
                    const uint32_t tq = tmem + acc * 4 * NR + ((uint32_t)(ew * 32) << 16);
                    tmem_ld_row<NR>(tq, g1);
                    if (off) tmem_ld_row<NR>(tq + 2 * NR, g2);
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tm_empty[acc]);
                    if (tle) sa.tlog[(kTlTile + 128 + tt) * 4 + 1] = sy_gtime();
                    if (m.diag) {  // both uses land in the item's own blocks
#pragma unroll
                        for (int q = 0; q < NR; ++q)
                            cs[(ii * NR + q) * kSyT] += g1[q] * (fG * sy_pow2(-__ldg(ws + J * NR + q)));
                    } else {
#pragma unroll
                        for (int q = 0; q < NR; ++q)
                            racc[q] += g1[q] * (fG * sy_pow2(-__ldg(ws + J * NR + q)));
                    }
                    if (off) {
#pragma unroll
                        for (int q = 0; q < NR; ++q)
                            cs[(jj * NR + q) * kSyT] += g2[q] * (fG * sy_pow2(-__ldg(ws + I * NR + q)));
                    }
                }
                // row block I0 + ii is complete: all its tiles of this item are done
                if (m.diag)
                    put_cs(m.b, m.I0 + ii, m.P, ii);
                else
                    put(m.b, m.I0 + ii, m.Q, racc);
            }
            if (!m.diag)
                for (int jj = 0; jj < m.nJ; ++jj) put_cs(m.b, m.J0 + jj, m.P, jj);
        }
        if (sa.tlog && row == 0) {
            sa.tlog[blockIdx.x * 4 + 2] = sy_gtime();
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            sa.tlog[blockIdx.x * 4 + 3] = ((unsigned long long)smid << 32) | (unsigned)tt;  // SM, tiles
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kCols));
}

// Tile-sharded contexts (one rank per GPU, replicated state): the slot sums
// of the rank's own items, in the update kernel's slot order, into a one-slot
// buffer [B][nRB][128][NR] that NCCL all-reduces before the update.
template <int NR>
__global__ void __launch_bounds__(kSyT * NR / 4) sym_slotsum_kernel(const float* __restrict__ spart,
                                                                     float* __restrict__ H, int nRB,
                                                                     int nSB, int b0) {
    constexpr int QG = NR / 4;
    const int K = blockIdx.x, b = b0 + blockIdx.y, t = threadIdx.x, g = t % QG, row = t / QG;
    const float4* src = reinterpret_cast<const float4*>(
                            spart + (((size_t)b * nRB + K) * nSB * kSyT + row) * NR) + g;
    constexpr size_t kSlot4 = (size_t)kSyT * NR / 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nSB; ++s) {
        const float4 v = __ldcs(src + s * kSlot4);
        acc.x = acc.x + v.x;
        acc.y = acc.y + v.y;
        acc.z = acc.z + v.z;
        acc.w = acc.w + v.w;
    }
    reinterpret_cast<float4*>(H + (((size_t)b * nRB + K) * kSyT + row) * NR)[g] = acc;
}

// 4 consecutive state values (one thread's replicas q0..q0+3) in the state type
__device__ __forceinline__ void sy_ld4(const float* p, float (&v)[4]) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void sy_ld4(const double* p, double (&v)[4]) {
    const double2 x = reinterpret_cast<const double2*>(p)[0], y = reinterpret_cast<const double2*>(p)[1];
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
}
__device__ __forceinline__ void sy_ldg4(const float* p, float (&v)[4]) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void sy_ldg4(const double* p, double (&v)[4]) {
    const double2 x = __ldg(reinterpret_cast<const double2*>(p)),
                  y = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
}
__device__ __forceinline__ void sy_st4(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void sy_st4(double* p, const double (&v)[4]) {
    reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
}

// Second pass of a step in ONE kernel, 4 replicas per thread: block (b, K) is
// handled by 128 x (NR / 4) threads; thread (row, g), g = t % (NR / 4) fastest
// so a warp reads whole state rows (coalesced 16-byte vectors), sums its 4
// replicas' nSB partial products in slot order (deterministic, fp32), runs the
// fused update for replicas 4g..4g+3 in the state type TS (float; a double
// instantiation gives an fp64-state variant) and, in step / Jacobi modes, emits the fp16
// B tile of the new w (staged in shared memory, stored with 16-byte vectors).
template <int NR, int MODE, typename TS = float>
__global__ void __launch_bounds__(kSyT * NR / 4, SY_UPD_OCC) sym_update_kernel(SymArgs sa) {
    constexpr int QG = NR / 4;
    constexpr int NW = kSyT * QG / 32;         // warps per CTA
    __shared__ unsigned s_max[NW][NR];          // per warp, per replica max |w|
    __shared__ int s_exp[NR];
    __shared__ TS s_min[NW][NR];                // per warp, per replica min e (step modes)
    __shared__ double s_sc[NW][NR][3];          // score partials
    __shared__ __align__(16) __half s_B[2 * NR * kSyT];
    const TcArgs& a = sa.t;
    const StepScalars& sc = a.s;
    const TS* __restrict__ Dp = static_cast<const TS*>(a.D);
    const TS* __restrict__ Hp = static_cast<const TS*>(a.hz);
    const TS* __restrict__ Win = static_cast<const TS*>(a.Win);
    TS* __restrict__ Wout = static_cast<TS*>(a.Wout);
    TS* __restrict__ Rp = static_cast<TS*>(a.Rs);
    TS* __restrict__ Cp = static_cast<TS*>(a.C);
    TS* __restrict__ Ep = static_cast<TS*>(a.E);
    TS* __restrict__ Hd = static_cast<TS*>(a.Hdbg);
    const int K = blockIdx.x, b = sa.b0 + blockIdx.y, nRB = a.nRB, N = a.N;
    const int t = threadIdx.x, g = t % QG, row = t / QG;
    const int lane = t & 31, wid = t >> 5;
    const int i = K * kSyT + row, q0 = 4 * g;
    const bool valid = i < N;
    const size_t si = (size_t)b * a.ldN + i, vi0 = si * NR + q0;
    unsigned long long* tl = sa.tlog && t == 0 ? sa.tlog + (kTlUpd + (size_t)b * nRB + K) * 4 : nullptr;
    if (tl) tl[0] = sy_gtime();
    sy_pdl_wait();  // the tile kernel's partial products
    // dependents may launch as soon as every CTA of this grid has STARTED: the next tile
    // kernel's CTAs take over SMs as they drain and run their prologue / gram prefetch under
    // the last update CTAs (105.5 vs 105.8 us per config-1 step against triggering at exit)
    sy_pdl_trigger();
    if (tl) tl[1] = sy_gtime();
    // state of the step modes first: its loads are in flight with the slot loads
    TS Rv[4] = {TS(0), TS(0), TS(0), TS(0)}, cv[4] = {TS(0), TS(0), TS(0), TS(0)};
    TS ev[4] = {TS(0), TS(0), TS(0), TS(0)};
    TS st_D = TS(0), st_hz = TS(0);
    if constexpr (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) {
        if (valid) {
            // the input w is never loaded: in step modes it is a function of the
            // stored c and R (init_state_kernel and every update write them so)
            sy_ldg4(Rp + vi0, Rv);
            sy_ld4(Cp + vi0, cv);
            sy_ld4(Ep + vi0, ev);
            st_D = __ldg(Dp + si);
            st_hz = __ldg(Hp + si);
        }
    }
    // ---- slot sums (fp32, fixed slot order)
    TS gw[4];
    {
        const int nSB = sa.nSB;
        const float4* src = reinterpret_cast<const float4*>(
                                sa.spart + (((size_t)b * nRB + K) * nSB * kSyT + row) * NR) +
                            g;
        constexpr size_t kSlot4 = (size_t)kSyT * NR / 4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        // groups of 4 slots (config 1 has exactly 4: no predicated-off loads / adds, which
        // still cost issue slots in this issue-bound kernel); same slot order either way
        for (int s0 = 0; s0 < nSB; s0 += 4) {
            float4 v[4];
            if (s0 + 4 <= nSB) {
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldcs(src + (s0 + u) * kSlot4);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc.x = acc.x + v[u].x;
                    acc.y = acc.y + v[u].y;
                    acc.z = acc.z + v[u].z;
                    acc.w = acc.w + v[u].w;
                }
            } else {
                for (int u = 0; s0 + u < nSB; ++u) {
                    const float4 w1 = __ldcs(src + (s0 + u) * kSlot4);
                    acc.x = acc.x + w1.x;
                    acc.y = acc.y + w1.y;
                    acc.z = acc.z + w1.z;
                    acc.w = acc.w + w1.w;
                }
            }
        }
        gw[0] = (TS)acc.x; gw[1] = (TS)acc.y; gw[2] = (TS)acc.z; gw[3] = (TS)acc.w;
    }
    bool fz[4];
    const int4 fg4 = *reinterpret_cast<const int4*>(a.fail_gstep + b * NR + q0);
    const int fga[4] = {fg4.x, fg4.y, fg4.z, fg4.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int fg = fga[u];
        fz[u] = (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN || MODE == EPI_STEP_PP)
                    ? fg < a.alt->gstep_base + a.step
                    : fg != kFreeTraj;
    }
    TS wn[4] = {TS(0), TS(0), TS(0), TS(0)};  // new contraction input (0: frozen / padding)
    if constexpr (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) {
        TS lmin[4] = {TS(INFINITY), TS(INFINITY), TS(INFINITY), TS(INFINITY)};
        if (valid) {
            const TS Dv = st_D, hzv = st_hz;
            const TS half_rt = (TS)sc.half_rt, rt = (TS)sc.rt, dt = (TS)sc.dt;
            TS wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                wv[u] = MODE == EPI_STEP_BN ? Rv[u] * (cv[u] > TS(0) ? TS(1) : TS(0))
                                            : (Rv[u] * TS(0.25)) * (cv[u] + rt);
            const TS Kj = (TS)sc.Kj, nbeta = (TS)sc.nbeta, tau = (TS)sc.tau;
            const double pd = a.pump ? a.pump[a.step] : a.p_scalar;
            const TS loss = sc.minus_j != 0.0 ? (TS)((-1.0 + pd) - sc.minus_j) : (TS)(-1.0 + pd);
            const TS thresh = (TS)a.alt->thresh;
            TS cn[4], en[4], wo[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const TS c = cv[u], e = ev[u];
                const TS Jw = Dv * wv[u] - gw[u];
                TS h;
                if constexpr (MODE == EPI_STEP_BN)
                    h = half_rt * (Jw + hzv);
                else
                    h = Jw + half_rt * hzv;
                if (Hd) Hd[vi0 + u] = h;
                const TS inj = (Kj * e) * (Rv[u] * h - thresh);
                cn[u] = c + dt * ((loss - c * c) * c + inj);
                en[u] = e + dt * ((nbeta * (c * c - tau)) * e);
                wo[u] = wv[u];  // frozen / failing trajectories keep their output w
                if (fz[u]) {
                    cn[u] = c;
                    en[u] = e;
                } else if (!isfinite(cn[u]) || !isfinite(en[u])) {
                    atomicMin(&a.fail_gstep[b * NR + q0 + u], a.alt->gstep_base + a.step);
                    atomicMin(&a.fail_idx[b * NR + q0 + u], i);
                    cn[u] = c;
                    en[u] = e;
                } else {
                    lmin[u] = en[u];
                    TS w;
                    if constexpr (MODE == EPI_STEP_BN)
                        w = Rv[u] * (cn[u] > TS(0) ? TS(1) : TS(0));
                    else
                        w = (Rv[u] * TS(0.25)) * (cn[u] + rt);
                    wo[u] = w;
                    wn[u] = w;
                }
            }
            sy_st4(Cp + vi0, cn);
            sy_st4(Ep + vi0, en);
            if (sa.keep_w) sy_st4(Wout + vi0, wo);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // min e: warp, then CTA (one atomic per replica)
            TS m = lmin[u];
#pragma unroll
            for (int off = 16; off >= QG; off >>= 1) {
                const TS o = __shfl_xor_sync(0xffffffffu, m, off);
                m = o < m ? o : m;
            }
            if (lane < QG) s_min[wid][q0 + u] = m;
        }
    } else if constexpr (MODE == EPI_STEP_PP) {
        // Positive-P step (pp_elem, kernels.cuh): the same element update as the CUDA-core
        // epilogue on this path's G w; the plain w is read and written as well as its B tile
        TS lmin[4] = {TS(INFINITY), TS(INFINITY), TS(INFINITY), TS(INFINITY)};
        if (valid) {
            TS* __restrict__ Np = static_cast<TS*>(a.Pn);
            TS* __restrict__ Mp = static_cast<TS*>(a.Pm);
            TS* __restrict__ MTp = static_cast<TS*>(a.MT);
            const double pd = a.pump ? a.pump[a.step] : a.p_scalar;
            const PpConsts<TS> pc(sc, *a.alt, pd);
            const TS Dv = __ldg(Dp + si), hzv = __ldg(Hp + si);
            TS wv[4], Rr[4], mu[4], nn[4], mm[4], ee[4], mt[4];
            double z0[4], z1[4];
            sy_ld4(Win + vi0, wv);
            sy_ldg4(Rp + vi0, Rr);
            sy_ld4(Cp + vi0, mu);
            sy_ld4(Np + vi0, nn);
            sy_ld4(Mp + vi0, mm);
            sy_ld4(Ep + vi0, ee);
            sy_ld4(MTp + vi0, mt);
            sy_ldg4(a.nz + vi0, z0);
            sy_ldg4(a.nz_next + vi0, z1);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                wn[u] = wv[u];  // frozen / failing trajectories keep their w
                if (fz[u]) continue;
                const PpElem<TS> o = pp_elem(pc, wv[u], Dv, hzv, Rr[u], gw[u], mu[u], nn[u],
                                             mm[u], ee[u], (TS)z0[u]);
                if (!o.finite) {
                    atomicMin(&a.fail_gstep[b * NR + q0 + u], a.alt->gstep_base + a.step);
                    atomicMin(&a.fail_idx[b * NR + q0 + u], i);  // kind 0: non-finite (pp_step)
                    continue;
                }
                mu[u] = o.mu;
                nn[u] = o.n;
                mm[u] = o.m;
                ee[u] = o.e;
                mt[u] = o.mt;
                lmin[u] = o.e;
                if (fabs((double)o.mu) > (double)pc.mu_abort) {  // run_pp :119-124, kind 1
                    atomicMin(&a.fail_gstep[b * NR + q0 + u], a.alt->gstep_base + a.step);
                    atomicMin(&a.fail_idx[b * NR + q0 + u], (1 << 30) + i);
                }
                wn[u] = pp_next_w(pc, Rr[u], o.mu, (TS)z1[u]);
            }
            sy_st4(Cp + vi0, mu);
            sy_st4(Np + vi0, nn);
            sy_st4(Mp + vi0, mm);
            sy_st4(Ep + vi0, ee);
            sy_st4(MTp + vi0, mt);
            sy_st4(Wout + vi0, wn);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // min e: warp, then CTA (one atomic per replica)
            TS m = lmin[u];
#pragma unroll
            for (int off = 16; off >= QG; off >>= 1) {
                const TS o = __shfl_xor_sync(0xffffffffu, m, off);
                m = o < m ? o : m;
            }
            if (lane < QG) s_min[wid][q0 + u] = m;
        }
    } else if constexpr (MODE == EPI_JACOBI) {
        if (valid) {
            const TS Dv = __ldg(Dp + si), bv = __ldg(Hp + si);
            const TS omd = (TS)sc.one_minus_dtc, dtc = (TS)sc.dt_c;
            TS Rj[4], wo[4];
            sy_ld4(Rp + vi0, Rj);
            sy_ld4(Win + vi0, wo);
            const char4 s4 = *reinterpret_cast<const char4*>(a.sigma + vi0);
            const bool on4[4] = {s4.x != 0, s4.y != 0, s4.z != 0, s4.w != 0};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (fz[u]) continue;
                const bool on = on4[u];
                TS rn = Rj[u];
                if (on) {
                    if (Dv == TS(0)) {
                        atomicMin(a.err, sa.rowmap ? sa.rowmap[(size_t)b * a.ldN + i] : i);
                        continue;
                    }
                    const TS off = gw[u] - Dv * Rj[u];
                    rn = omd * Rj[u] + dtc * ((bv - off) / Dv);
                    Rj[u] = rn;
                }
                const TS w = rn * (on ? TS(1) : TS(0));
                wo[u] = w;
                wn[u] = w;
            }
            sy_st4(Rp + vi0, Rj);
            sy_st4(Wout + vi0, wo);
        }
    } else if constexpr (MODE == EPI_MATVEC) {
        if (valid) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (!fz[u]) a.Mv[vi0 + u] = (double)gw[u];
        }
    } else {  // EPI_SCORE: w.Gw, hz.w, |w - x|^2 partials of this 128-row block
        double pa[4], pb[4], pc[4];
        TS wv4[4] = {TS(0), TS(0), TS(0), TS(0)};
        if (valid) sy_ld4(Win + vi0, wv4);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pa[u] = pb[u] = pc[u] = 0.0;
            if (valid && !fz[u]) {
                const double wv = wv4[u];
                pa[u] = wv * (double)gw[u];
                pb[u] = (double)Hp[si] * wv;
                if (a.xtrue) {
                    const double xt = a.xitrue[si] ? a.xtrue[si] : 0.0;
                    pc[u] = (wv - xt) * (wv - xt);
                }
            }
#pragma unroll
            for (int off = 16; off >= QG; off >>= 1) {
                pa[u] += __shfl_xor_sync(0xffffffffu, pa[u], off);
                pb[u] += __shfl_xor_sync(0xffffffffu, pb[u], off);
                pc[u] += __shfl_xor_sync(0xffffffffu, pc[u], off);
            }
        }
        if (lane < QG) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                s_sc[wid][q0 + u][0] = pa[u];
                s_sc[wid][q0 + u][1] = pb[u];
                s_sc[wid][q0 + u][2] = pc[u];
            }
        }
        __syncthreads();
        if (t < NR) {  // thread t writes replica t: warps summed in a fixed order
            double A_ = 0, B_ = 0, C_ = 0;
            for (int w = 0; w < NW; ++w) {
                A_ += s_sc[w][t][0];
                B_ += s_sc[w][t][1];
                C_ += s_sc[w][t][2];
            }
            double* p = a.part + (((size_t)b * nRB + K) * NR + t) * 4;
            p[0] = A_;
            p[1] = B_;
            p[2] = C_;
        }
    }
    if constexpr (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN || MODE == EPI_STEP_PP ||
                  MODE == EPI_JACOBI) {
        // fp16 B tile of the new w of block K: per-replica max over the 128 rows
        // (no tile when the contraction does not read them: transform chains)
        const bool emit = sa.WBout != nullptr;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            unsigned m = __float_as_uint(fabsf((float)wn[u]));
#pragma unroll
            for (int off = 16; off >= QG; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
            if (lane < QG) s_max[wid][q0 + u] = m;
        }
        __syncthreads();
        if (t < NR) {
            if constexpr (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN || MODE == EPI_STEP_PP) {
                TS mn = TS(INFINITY);
                for (int w = 0; w < NW; ++w) mn = s_min[w][t] < mn ? s_min[w][t] : mn;
                if (mn != TS(INFINITY)) atomicMin(&a.minE[b * NR + t], ord_key(mn));
            }
            unsigned m = 0;
            for (int w = 0; w < NW; ++w) m = max(m, s_max[w][t]);
            const int e = sy_exp14(__uint_as_float(m));
            s_exp[t] = e;
            if (emit) sa.WSout[((size_t)b * nRB + K) * NR + t] = e;
        }
        if (!emit) {
            sy_pdl_trigger();
            return;
        }
        __syncthreads();
        unsigned char* Bs = reinterpret_cast<unsigned char*>(s_B);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            __half hi, lo;
            sy_split(wn[u], s_exp[q0 + u], hi, lo);
            *reinterpret_cast<__half*>(Bs + sy_offk(q0 + u, row, 2 * NR)) = hi;
            *reinterpret_cast<__half*>(Bs + sy_offk(NR + q0 + u, row, 2 * NR)) = lo;
        }
        __syncthreads();
        uint4* dst = reinterpret_cast<uint4*>(sa.WBout + ((size_t)b * nRB + K) * (2 * NR * kSyT));
        const uint4* srcB = reinterpret_cast<const uint4*>(s_B);
        for (int o = t; o < 2 * NR * kSyT / 8; o += kSyT * QG) dst[o] = srcB[o];
    }
    if (tl) tl[2] = sy_gtime();
}

}  // namespace cimcs
