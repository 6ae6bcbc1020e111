// tc_kernels.cuh -- shared tcgen05 building blocks of the fp32 symmetric-tile
// path (sym_kernels.cuh): UMMA shared-memory descriptors, MMA commit, TMEM
// loads and the TcArgs argument block of the fused update kernel.
//
// (Round 1 also shipped a streaming 3xTF32 kernel here that read the dense
// gram every step; its tensor-core truncation of the raw fp32 operands biased
// |G w| by ~2^-20 per step and it lost to the symmetric path on bytes, so it was
// removed.  The measurements are in DESIGN.md section 4.)
#pragma once

#include "kernels.cuh"

namespace cimcs {

constexpr int kTcRows = 128;           // M of the MMA, spins per tile
constexpr int kTcChunk = kTcChunkJ;    // j per pipeline stage

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // SWIZZLE_NONE, base offset 0
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
    // state arrays in the context's state type (float on the fp32 path)
    const void* D;         // [B][ldN]
    const void* hz;
    const void* Win;       // [B][ldN][NR]
    void* Wout;
    void* Rs;              // [B][ldN][NR]
    void* C;
    void* E;
    void* Hdbg;
    double* Mv;            // EPI_MATVEC output [B][ldN][NR]
    void* Pn;              // Positive-P moments n, m and the measured amplitude [B][ldN][NR]
    void* Pm;
    void* MT;
    const double* nz;      // this step's unit normals [B][ldN][NR] (host stream), the next step's
    const double* nz_next;
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

}  // namespace cimcs
