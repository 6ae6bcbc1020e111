// sym64_kernels.cuh -- fp64 fused MFZ step on the FP64 tensor cores (DMMA,
// mma.sync m8n8k4 f64) reading each gram entry ONCE per step (G = G^T).
//
// The fp64 path is the bitwise-reproducible one, so its contraction order is a
// contract with the oracle.  Measured on the B200 (tools/peaks_probe.cu,
// profiles/r02_peaks.json): one m8n8k4 DMMA computes, for every output, the
// sequential fma chain d = fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c)))),
// bit for bit (262144 / 262144 random cases).  Chaining DMMAs over k therefore
// gives ONE sequential fma chain, so the order below is exactly the oracle's
// canonical segmented order ORC_CANON with gran = 512, nseg = ceil(N / 512):
//     (G w)_i = sum_s P_s,  P_s = fma chain over j in [512 s, 512 s + 512),
//     j ascending, from +0;  the P_s added left to right.
// (Proof sketch: the gram is stored as upper-triangle 64 x 64 tiles; an ITEM is
// a 512 x 512 super-block (P, Q), P <= Q.  For a row block K of super-row P0:
// items (P0, Q > P0) give use 1 (G[I,J] w[J]) chains over the columns of Q in
// ascending J; items (P < P0, P0) give use 2 (G[I,J]^T w[I]) chains over the rows
// of P, which by symmetry are columns 512 P.. of row i, ascending; the diagonal
// item (P0, P0) walks its tiles row-major, so block K first receives use 2 of
// the rows above it and then use 1 of its own row: again columns ascending.
// Each item's chain is one partial ("slot"); the update kernel adds the nSB
// slots in order.)  DMMA peak 37 TFLOP/s = DFMA peak on this chip, but one
// instruction does 256 FMAs, so the issue slots and shared-memory operand loads
// that bound the CUDA-core kernel (gemv_fused_kernel<double>: FP64 pipe 55 %)
// drop by 8x; and the symmetric tiles halve the HBM bytes (1.1 GB/step at
// config 1 instead of 2.05 GB), leaving the step compute-bound.
//
// Layouts (per instance b):
//   G tiles   [ntri][64 x 64] fp64, tile (I, J), I <= J, row-major upper
//             triangle order (sy_tri); element (r, c) at r*64 + (c ^ ((r&3)<<2))
//             -- an XOR swizzle that makes the A-fragment loads of BOTH uses
//             (rows g / cols t, and the transposed cols g / rows t) hit 16
//             distinct 8-byte banks per half-warp; a tile is ONE 32 KB bulk copy
//   W tiles   [nRB][64][NR] fp64, element (k, n) at k*NR + (n ^ swz_w(k))
//   partials  [nRB][nSB][64][NR] fp64 (slot = item of the block, see above)
// Persistent warp-specialised CTA (one per SM): warp 8 produces (bulk copies
// into a 3-stage mbarrier ring), warps 0-3 run use 1 (16 rows x NR each),
// warps 4-7 run use 2; use-1 accumulators of an off-diagonal item's row live
// in registers, use-2 (and diagonal-item) accumulators in shared memory.
#pragma once

#include "sym_kernels.cuh"

namespace cimcs {

constexpr int kT6 = 64;                         // tile edge
constexpr int kS6 = 8;                          // item edge in tiles (512 = one segment)
constexpr int kT6Stages = 3;
constexpr uint32_t kT6TileBytes = kT6 * kT6 * 8;  // 32 KB
constexpr int kT6Seg = kT6 * kS6;               // canonical segment (512)

__host__ __device__ inline int s6_gofs(int r, int c) { return r * kT6 + (c ^ ((r & 3) << 2)); }
template <int NR>
__host__ __device__ inline int s6_wofs(int k, int n) {
    return k * NR + (n ^ (NR == 16 ? (k & 3) << 2 : ((k >> 1) & 1) << 2));
}

// gram builder output: upper-triangle 64 x 64 tiles (gram128_kernel mirrors, so
// the diagonal tiles are complete)
struct Sym64Out {
    double* G;
    int nRB, ntri;
    __device__ __forceinline__ void store(int b, int i, int j, double v) const {
        const int I = i / kT6, J = j / kT6;
        if (I > J) return;
        G[((size_t)b * ntri + sy_tri(I, J, nRB)) * (kT6 * kT6) + s6_gofs(i % kT6, j % kT6)] = v;
    }
};

struct Sym64Args {
    TcArgs t;              // fp64 state arrays, scalars, outputs
    const double* Gt;      // [B][ntri][64 x 64]
    const double* WTin;    // [B][nRB][64][NR] fp64 w tiles of the input
    double* WTout;         // same for the output w (step / Jacobi modes)
    double* part;          // [B][nRB][nSB][64][NR]
    const int2* items;     // (b, P << 16 | Q)
    const int* sched;      // [grid + 1]
    int ntri, nSB;
    int keep_w;            // step modes: also store the plain [b][i][r] w
    const int2* seg;       // compacted refit: per segment (first block, blocks), or null
    const int* rowmap;     // compacted refit: row -> original spin (error reports), or null
    // Item flags (null: the update kernel waits for the whole tile grid).  The tile
    // kernel is bound by the DMMA pipe and leaves HBM and the other pipes idle, so the
    // update CTAs of instance b run under it as soon as b's `ipi` items are published:
    // done[b] counts published items, taken[b] the update CTAs that saw it complete.
    unsigned* done;
    unsigned* taken;
    unsigned ipi;
    unsigned long long* tlog;  // option "timeline": per-CTA stamps (rows as in sym_kernels.cuh)
};

// The tile kernel's consumers of an item meet on the item's last barrier after their
// partial-product stores; one thread then fences (gpu scope, cumulative) and publishes
// (s6_item_done).  An update CTA of
// instance b waits for all `ipi` items of b (s6_wait_items); the last of the
// instance's `nblk` update CTAs to pass zeroes both counters, and the next tile
// kernel publishes nothing before that update grid has completed (its threads
// trigger their dependents only after their own griddepcontrol.wait, so the next
// update grid cannot even become resident earlier).  The wait is bounded: on expiry
// the CTA reports through *err (-2) instead of hanging the GPU.
__device__ __forceinline__ void s6_item_done(unsigned* done, int b) {
    __threadfence();
    atomicAdd(done + b, 1u);
}
__device__ __forceinline__ void s6_wait_items(unsigned* done, unsigned* taken, int b, unsigned ipi,
                                              unsigned nblk, int* err) {
    unsigned v;
    const long long t0 = clock64();
    for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + b) : "memory");
        if (v >= ipi) break;
        __nanosleep(256);
        if (clock64() - t0 > (1ll << 32)) {
            if (err) atomicMin(err, -2);
            break;
        }
    }
    if (atomicAdd(taken + b, 1u) == nblk - 1) {
        taken[b] = 0;
        done[b] = 0;
        __threadfence();
    }
}

template <int NR>
__host__ __device__ constexpr size_t s6_wbytes() { return (size_t)kT6 * NR * 8; }
template <int NR>
__host__ __device__ constexpr size_t s6_stage_bytes() { return kT6TileBytes + 2 * s6_wbytes<NR>(); }
template <int NR>
__host__ __device__ constexpr size_t s6_smem_bytes() {
    // stages + use-2 / diagonal accumulators (kS6 blocks) + mbarriers
    return kT6Stages * s6_stage_bytes<NR>() + (size_t)kS6 * kT6 * NR * 8 + 256;
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Warp tiling of one use: WPU warps per use split the 64 x NR output block into
// RW rows x (NT x 8) replicas each (MT = RW / 8 row fragments).  WPU = 4: 16 rows
// x NR; WPU = 8 (NR 16): 16 rows x 8 replicas (more warps to hide the DMMA
// issue latency, same chains per SM sub-partition).
template <int NR, int WPU>
struct S6Map {
    static constexpr int NSPLIT = (NR / 8 >= 2 && WPU == 8) ? 2 : 1;  // warps across replicas
    static constexpr int NT = NR / 8 / NSPLIT;
    static constexpr int RW = 64 * NSPLIT / WPU;
    static constexpr int MT = RW / 8;
    __device__ static int m0(int u) { return (u / NSPLIT) * RW; }
    __device__ static int n0(int u) { return (u % NSPLIT) * NT * 8; }
};

// One use of one tile for one warp: acc (MT x NT fragments, 2 doubles each)
// += A(rows m0.. of the warp) * B(w tile, replicas n0..).  use 1: A[m][k] =
// tile[m][k]; use 2: A[m][k] = tile[k][m].  k runs 0..63 ascending (4 per DMMA).
template <int NR, int MT, int NT, bool kT>
__device__ __forceinline__ void s6_tile_mma(const double* __restrict__ tile,
                                            const double* __restrict__ wt, int m0, int n0,
                                            int lane, double (&acc)[MT][NT][2]) {
    const int g = lane >> 2, t = lane & 3;
    double a[MT], b[NT], an[MT], bn[NT];
    auto load = [&](int k0, double (&aa)[MT], double (&bb)[NT]) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int m = m0 + 8 * mt + g, k = k0 + t;
            aa[mt] = kT ? tile[s6_gofs(k, m)] : tile[s6_gofs(m, k)];
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bb[nt] = wt[s6_wofs<NR>(k0 + t, n0 + 8 * nt + g)];
    };
    load(0, a, b);
#pragma unroll
    for (int k0 = 0; k0 < kT6; k0 += 4) {
        if (k0 + 4 < kT6) load(k0 + 4, an, bn);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
        if (k0 + 4 < kT6) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) a[mt] = an[mt];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) b[nt] = bn[nt];
        }
    }
}

// accumulator fragments <-> a [64][NR] block (row-major; the C-fragment
// pattern g*NR + 2t hits 8 distinct 16-B columns per quarter-warp)
template <int NR, int MT, int NT>
__device__ __forceinline__ void s6_acc_ld(const double* blk, int m0, int n0, int lane,
                                          double (&acc)[MT][NT][2]) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const double2 v = *reinterpret_cast<const double2*>(
                blk + (m0 + 8 * mt + g) * NR + n0 + 8 * nt + 2 * t);
            acc[mt][nt][0] = v.x;
            acc[mt][nt][1] = v.y;
        }
}
template <int NR, int MT, int NT>
__device__ __forceinline__ void s6_acc_st(double* blk, int m0, int n0, int lane,
                                          const double (&acc)[MT][NT][2]) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
            *reinterpret_cast<double2*>(blk + (m0 + 8 * mt + g) * NR + n0 + 8 * nt + 2 * t) =
                make_double2(acc[mt][nt][0], acc[mt][nt][1]);
}
template <int MT, int NT>
__device__ __forceinline__ void s6_acc_zero(double (&acc)[MT][NT][2]) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
}

template <int NC>
__device__ __forceinline__ void s6_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NC * 32) : "memory");
}

// NC = DMMA warps (NC / 2 per use); one more warp produces.
template <int NR, int MODE, int NC>
__global__ void __launch_bounds__((NC + 1) * 32, 1) sym64_step_kernel(Sym64Args sa) {
    constexpr int kT6Compute = NC;
    using Map = S6Map<NR, NC / 2>;
    constexpr int MT = Map::MT, NT = Map::NT;
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr size_t kStage = s6_stage_bytes<NR>();
    constexpr size_t kWB = s6_wbytes<NR>();
    constexpr int kBlk = kT6 * NR;  // doubles per accumulator block
    double* accs = reinterpret_cast<double*>(smem + kT6Stages * kStage);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kT6Stages * kStage + kS6 * kBlk * 8);
    uint64_t* empty = full + kT6Stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nRB = sa.t.nRB, nSB = sa.nSB;
    const int it0 = sa.sched[blockIdx.x], it1 = sa.sched[blockIdx.x + 1];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kT6Stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kT6Compute);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // PDL: the update kernel may launch now; this grid's w reads / partial
    // writes wait for the previous update kernel (the gram is never written
    // inside a CIM call, so the first stages' gram copies may start earlier)
    constexpr bool kEarly = MODE == EPI_STEP_BN || MODE == EPI_STEP_CN;
    if (sa.tlog && threadIdx.x == 0) sa.tlog[blockIdx.x * 4 + 0] = sy_gtime();
    if (!sa.done) sy_pdl_trigger();
    if (!kEarly || warp != kT6Compute) {
        sy_pdl_wait();
        if (sa.done) sy_pdl_trigger();  // item flags: only after the previous update grid
    }

    auto item = [&](int k, int& b, int& P, int& Q, int& nI, int& nJ) {
        const int2 it = sa.items[k];
        b = it.x;
        P = it.y >> 16;
        Q = it.y & 0xffff;
        nI = sa.seg ? sa.seg[P].y : min(kS6, nRB - P * kS6);
        nJ = sa.seg ? sa.seg[Q].y : min(kS6, nRB - Q * kS6);
    };
    // first 64-row block of segment P (fixed 8-block segments, or the compacted
    // refit's variable ones: each compacted segment is one original 512-column
    // segment, so the canonical order is unchanged)
    auto blk0 = [&](int P) { return sa.seg ? sa.seg[P].x : P * kS6; };

    if (warp == kT6Compute) {
        // ------------------------------------------------------ producer
        // (convergent warp, warp-uniform operands, one elected lane issues: a bulk copy
        // issued from inside `if (lane == 0)` is wrapped in an ELECT / R2UR / BRA.U.ANY
        // loop by ptxas -- sym_kernels.cuh)
        const uint64_t pG = sy_policy_first(), pW = sy_policy_last();
        const uint32_t smem0 = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
        const uint32_t full0 = __shfl_sync(0xffffffffu, smem_u32(full), 0);
        const int k0 = __shfl_sync(0xffffffffu, it0, 0), k1 = __shfl_sync(0xffffffffu, it1, 0);
        // item descriptors one per lane, loaded before the PDL wait (sym_kernels.cuh)
        const int2 mine = lane < k1 - k0 ? sa.items[k0 + lane] : make_int2(0, 0);
        auto item_u = [&](int k, int& b, int& P, int& Q, int& nI, int& nJ) {
            int2 itv;
            if (k - k0 < 32) {
                itv.x = __shfl_sync(0xffffffffu, mine.x, k - k0);
                itv.y = __shfl_sync(0xffffffffu, mine.y, k - k0);
            } else {
                itv = sa.items[k];
            }
            b = __shfl_sync(0xffffffffu, itv.x, 0);
            const int iy = __shfl_sync(0xffffffffu, itv.y, 0);
            P = iy >> 16;
            Q = iy & 0xffff;
            nI = sa.seg ? __shfl_sync(0xffffffffu, sa.seg[P].y, 0) : min(kS6, nRB - P * kS6);
            nJ = sa.seg ? __shfl_sync(0xffffffffu, sa.seg[Q].y, 0) : min(kS6, nRB - Q * kS6);
        };
        auto blk0_u = [&](int P) {
            return sa.seg ? __shfl_sync(0xffffffffu, sa.seg[P].x, 0) : P * kS6;
        };
        // stage s of a tile: expect its bytes, copy the gram tile
        auto g_part = [&](int s, int b, int I, int J) {
            const double* src = sa.Gt + ((size_t)b * sa.ntri + sy_tri(I, J, nRB)) * (kT6 * kT6);
            if (sy_elect_one()) {
                const uint32_t fb = full0 + s * 8;
                sy_expect_tx_u(fb, kT6TileBytes + (I != J ? 2 : 1) * (uint32_t)kWB);
                sy_bulk_u(smem0 + s * (uint32_t)kStage, src, kT6TileBytes, fb, pG);
            }
            __syncwarp();
        };
        int tt = 0;
        for (int k = k0; k < k1 && tt < kT6Stages; ++k) {  // fill before the PDL wait
            int b, P, Q, nI, nJ;
            item_u(k, b, P, Q, nI, nJ);
            const int bP = blk0_u(P), bQ = blk0_u(Q);
            for (int ii = 0; ii < nI && tt < kT6Stages; ++ii)
                for (int jj = P == Q ? ii : 0; jj < nJ && tt < kT6Stages; ++jj, ++tt)
                    g_part(tt, b, bP + ii, bQ + jj);
        }
        if (kEarly) {
            sy_pdl_wait();
            if (sa.done) sy_pdl_trigger();
        }
        tt = 0;
        for (int k = k0; k < k1; ++k) {
            int b, P, Q, nI, nJ;
            item_u(k, b, P, Q, nI, nJ);
            const int bP = blk0_u(P), bQ = blk0_u(Q);
            const double* Wb = sa.WTin + (size_t)b * nRB * (kT6 * NR);
            for (int ii = 0; ii < nI; ++ii)
                for (int jj = P == Q ? ii : 0; jj < nJ; ++jj, ++tt) {
                    const int I = bP + ii, J = bQ + jj, s = tt % kT6Stages;
                    if (tt >= kT6Stages) {
                        mbar_wait(&empty[s], ((tt / kT6Stages) - 1) & 1);
                        g_part(s, b, I, J);
                    }
                    if (sy_elect_one()) {
                        const uint32_t st = smem0 + s * (uint32_t)kStage + kT6TileBytes,
                                       fb = full0 + s * 8;
                        sy_bulk_u(st, Wb + (size_t)J * (kT6 * NR), (uint32_t)kWB, fb, pW);
                        if (I != J)
                            sy_bulk_u(st + (uint32_t)kWB, Wb + (size_t)I * (kT6 * NR), (uint32_t)kWB,
                                      fb, pW);
                    }
                    __syncwarp();
                }
        }
        return;
    }
    // ---------------------------------------------------------- DMMA warps
    const bool use2 = warp >= NC / 2;
    const int u = warp % (NC / 2);
    const int m0 = Map::m0(u), n0 = Map::n0(u);  // rows (use 1) / columns (use 2), replicas
    double racc[MT][NT][2];
    int tt = 0;
    for (int k = it0; k < it1; ++k) {
        int b, P, Q, nI, nJ;
        item(k, b, P, Q, nI, nJ);
        const bool diag = P == Q;
        const int nblk = diag ? nI : nJ;  // smem accumulator blocks of this item
        // zero this warp's rows of the accumulator blocks (use-2 warps; both
        // groups touch the same rows of a diagonal item's blocks)
        if (use2) {
            for (int kb = 0; kb < nblk; ++kb)
                for (int e = lane; e < Map::RW * NT * 8; e += 32)
                    accs[kb * kBlk + (m0 + e / (NT * 8)) * NR + n0 + e % (NT * 8)] = 0.0;
        }
        s6_bar<NC>(1);
        for (int ii = 0; ii < nI; ++ii) {
            if (!use2) s6_acc_zero<MT, NT>(racc);
            for (int jj = diag ? ii : 0; jj < nJ; ++jj, ++tt) {
                const int I = blk0(P) + ii, J = blk0(Q) + jj, s = tt % kT6Stages;
                mbar_wait(&full[s], (tt / kT6Stages) & 1);
                const double* tile = reinterpret_cast<const double*>(smem + s * kStage);
                const double* wJ = reinterpret_cast<const double*>(smem + s * kStage + kT6TileBytes);
                const double* wI = wJ + kT6 * NR;
                if (!use2) {
                    if (diag) {  // use 1 into block ii's shared accumulator
                        double acc[MT][NT][2];
                        s6_acc_ld<NR, MT, NT>(accs + ii * kBlk, m0, n0, lane, acc);
                        s6_tile_mma<NR, MT, NT, false>(tile, wJ, m0, n0, lane, acc);
                        s6_acc_st<NR, MT, NT>(accs + ii * kBlk, m0, n0, lane, acc);
                    } else {
                        s6_tile_mma<NR, MT, NT, false>(tile, wJ, m0, n0, lane, racc);
                    }
                } else if (I != J) {  // use 2 into column block jj
                    double acc[MT][NT][2];
                    s6_acc_ld<NR, MT, NT>(accs + jj * kBlk, m0, n0, lane, acc);
                    s6_tile_mma<NR, MT, NT, true>(tile, wI, m0, n0, lane, acc);
                    s6_acc_st<NR, MT, NT>(accs + jj * kBlk, m0, n0, lane, acc);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            if (diag) {
                s6_bar<NC>(1);  // use-2 of rows <= ii lands before use 1 of row ii + 1
            } else if (!use2) {  // row block I complete for this item: slot Q
                double* p = sa.part + ((((size_t)b * nRB + blk0(P) + ii) * nSB + Q) * kT6) * NR;
                s6_acc_st<NR, MT, NT>(p, m0, n0, lane, racc);
            }
        }
        // item done: shared accumulators -> partials (slot P)
        if (use2) {
            const int J0 = blk0(diag ? P : Q);
            for (int kb = 0; kb < nblk; ++kb) {
                double* p = sa.part + ((((size_t)b * nRB + J0 + kb) * nSB + P) * kT6) * NR;
                for (int e = lane; e < Map::RW * NT * 4; e += 32) {  // 2 doubles per element
                    const int r = m0 + e / (NT * 4), cc = n0 + 2 * (e % (NT * 4));
                    *reinterpret_cast<double2*>(p + r * NR + cc) =
                        *reinterpret_cast<const double2*>(accs + kb * kBlk + r * NR + cc);
                }
            }
        }
        s6_bar<NC>(1);  // accumulators free for the next item; every warp's partials are stored
        // (the barrier orders the other threads' stores before thread 0's cumulative
        // gpu-scope fence in s6_item_done: the __syncthreads / __threadfence / atomic pattern)
        if (sa.done && threadIdx.x == 0) s6_item_done(sa.done, b);
    }
    if (sa.tlog && threadIdx.x == 0) sa.tlog[blockIdx.x * 4 + 2] = sy_gtime();
}

// w tiles [nRB][64][NR] from a plain [b][i][r] W (after init / support / mask / CG)
template <int NR>
__global__ void sym64_wconvert_kernel(const double* __restrict__ W, int N, int ldN, int nRB,
                                      double* __restrict__ WT) {
    const int X = blockIdx.x, b = blockIdx.y;
    for (int e = threadIdx.x; e < kT6 * NR; e += blockDim.x) {
        const int k = e / NR, n = e % NR, j = X * kT6 + k;
        WT[((size_t)b * nRB + X) * (kT6 * NR) + s6_wofs<NR>(k, n)] =
            j < N ? W[((size_t)b * ldN + j) * NR + n] : 0.0;
    }
}

// Second pass of a step: block (b, K) of 64 rows by 64 x (NR / 4) threads,
// thread (row, g) owns replicas 4g..4g+3; sums the nSB fp64 slots in order
// ((0 + P_0) + P_1 + ...), runs the fused fp64 update (the arithmetic of
// gemv_fused_kernel<double>'s epilogue: bitwise the oracle's) and emits the w
// tile of the new w.
// ROWS = rows per CTA: 64 (a whole block), or 32 in the step modes -- a 4-warp CTA
// of 80 registers is what fits beside a resident tile CTA (its 9 warps x 144 registers
// leave 2560 registers on the SM sub-partition that holds three of them: one warp),
// and the step modes reduce across rows only through an atomicMin.
template <int NR, int MODE, int ROWS = kT6>
__global__ void __maxnreg__(80) sym64_update_kernel(Sym64Args sa) {
    constexpr int QG = NR / 4;
    constexpr int NW = (ROWS * QG + 31) / 32;
    constexpr int SPLIT = kT6 / ROWS;  // CTAs per 64-row block
    static_assert(ROWS == kT6 || MODE == EPI_STEP_BN || MODE == EPI_STEP_CN, "half blocks: step modes");
    __shared__ double s_min[NW][NR];
    __shared__ double s_sc[NW][NR][3];
    const TcArgs& a = sa.t;
    const StepScalars& sc = a.s;
    const double* __restrict__ Dp = static_cast<const double*>(a.D);
    const double* __restrict__ Hp = static_cast<const double*>(a.hz);
    const double* __restrict__ Win = static_cast<const double*>(a.Win);
    double* __restrict__ Wout = static_cast<double*>(a.Wout);
    double* __restrict__ Rp = static_cast<double*>(a.Rs);
    double* __restrict__ Cp = static_cast<double*>(a.C);
    double* __restrict__ Ep = static_cast<double*>(a.E);
    double* __restrict__ Hd = static_cast<double*>(a.Hdbg);
    const int K = blockIdx.x / SPLIT, b = blockIdx.y, nRB = a.nRB, N = a.N;
    const int t = threadIdx.x, g = t % QG, row = (blockIdx.x % SPLIT) * ROWS + t / QG;
    const int lane = t & 31, wid = t >> 5;
    const int i = K * kT6 + row, q0 = 4 * g;
    const bool valid = i < N;
    const size_t si = (size_t)b * a.ldN + i, vi0 = si * NR + q0;
    unsigned long long* tl =
        sa.tlog && t == 0 ? sa.tlog + (kTlUpd + (size_t)b * gridDim.x + blockIdx.x) * 4 : nullptr;
    if (tl) tl[0] = sy_gtime();
    if (sa.done) {  // this instance's items only: the tile grid may still be running
        if (t == 0) s6_wait_items(sa.done, sa.taken, b, sa.ipi, gridDim.x, a.err);
        __syncthreads();
    } else {
        sy_pdl_wait();
    }
    if (tl) tl[1] = sy_gtime();
    sy_pdl_trigger();  // early: dependents launch once every CTA of this grid has started
    double Rv[4] = {0, 0, 0, 0}, cv[4] = {0, 0, 0, 0}, ev[4] = {0, 0, 0, 0};
    double st_D = 0.0, st_hz = 0.0;
    if constexpr (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) {
        if (valid) {
            sy_ldg4(Rp + vi0, Rv);
            sy_ld4(Cp + vi0, cv);
            sy_ld4(Ep + vi0, ev);
            st_D = __ldg(Dp + si);
            st_hz = __ldg(Hp + si);
        }
    }
    double gw[4] = {0.0, 0.0, 0.0, 0.0};
    {
        const double* src = sa.part + (((size_t)b * nRB + K) * sa.nSB * kT6 + row) * NR + q0;
        for (int s = 0; s < sa.nSB; ++s) {
            double v[4];
            sy_ld4(src + (size_t)s * kT6 * NR, v);
#pragma unroll
            for (int u = 0; u < 4; ++u) gw[u] = gw[u] + v[u];
        }
    }
    bool fz[4];
    const int4 fg4 = *reinterpret_cast<const int4*>(a.fail_gstep + b * NR + q0);
    const int fga[4] = {fg4.x, fg4.y, fg4.z, fg4.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
        fz[u] = (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN || MODE == EPI_STEP_PP)
                    ? fga[u] < a.alt->gstep_base + a.step
                    : fga[u] != kFreeTraj;
    double wn[4] = {0.0, 0.0, 0.0, 0.0};
    bool emit = false;
    if constexpr (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) {
        emit = true;
        double lmin[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
        if (valid) {
            const double Dv = st_D, hzv = st_hz;
            const double half_rt = sc.half_rt, rt = sc.rt, dt = sc.dt;
            double wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                wv[u] = MODE == EPI_STEP_BN ? Rv[u] * (cv[u] > 0.0 ? 1.0 : 0.0)
                                            : (Rv[u] * 0.25) * (cv[u] + rt);
            const double Kj = sc.Kj, nbeta = sc.nbeta, tau = sc.tau;
            const double pd = a.pump ? a.pump[a.step] : a.p_scalar;
            const double loss = sc.minus_j != 0.0 ? (-1.0 + pd) - sc.minus_j : -1.0 + pd;
            const double thresh = a.alt->thresh;
            double cn[4], en[4], wo[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double c = cv[u], e = ev[u];
                const double Jw = Dv * wv[u] - gw[u];  // apply_coupling: gram_diag∘w - G w
                double h;
                if constexpr (MODE == EPI_STEP_BN)
                    h = half_rt * (Jw + hzv);
                else
                    h = Jw + half_rt * hzv;
                if (Hd) Hd[vi0 + u] = h;
                const double inj = (Kj * e) * (Rv[u] * h - thresh);
                cn[u] = c + dt * ((loss - c * c) * c + inj);
                en[u] = e + dt * ((nbeta * (c * c - tau)) * e);
                wo[u] = wv[u];
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
                    double w;
                    if constexpr (MODE == EPI_STEP_BN)
                        w = Rv[u] * (cn[u] > 0.0 ? 1.0 : 0.0);
                    else
                        w = (Rv[u] * 0.25) * (cn[u] + rt);
                    wo[u] = w;
                }
                wn[u] = wo[u];  // frozen / failing trajectories keep their w
            }
            sy_st4(Cp + vi0, cn);
            sy_st4(Ep + vi0, en);
            if (sa.keep_w) sy_st4(Wout + vi0, wo);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            double m = lmin[u];
#pragma unroll
            for (int off = 16; off >= QG; off >>= 1) {
                const double o = __shfl_xor_sync(0xffffffffu, m, off);
                m = o < m ? o : m;
            }
            if (lane < QG) s_min[wid][q0 + u] = m;
        }
        __syncthreads();
        if (t < NR) {
            double mn = INFINITY;
            for (int w = 0; w < NW; ++w) mn = s_min[w][t] < mn ? s_min[w][t] : mn;
            if (mn != INFINITY) atomicMin(&a.minE[b * NR + t], ord_key(mn));
        }
    } else if constexpr (MODE == EPI_STEP_PP) {
        // Positive-P step (pp_elem, kernels.cuh): the same element update as the CUDA-core
        // epilogue on this path's G w; the plain w is read and written as well as its tile
        emit = true;
        double lmin[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
        if (valid) {
            double* __restrict__ Np = static_cast<double*>(a.Pn);
            double* __restrict__ Mp = static_cast<double*>(a.Pm);
            double* __restrict__ MTp = static_cast<double*>(a.MT);
            const double pd = a.pump ? a.pump[a.step] : a.p_scalar;
            const PpConsts<double> pc(sc, *a.alt, pd);
            const double Dv = __ldg(Dp + si), hzv = __ldg(Hp + si);
            double wv[4], Rr[4], mu[4], nn[4], mm[4], ee[4], mt[4] = {0, 0, 0, 0}, z0[4], z1[4];
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
                const PpElem<double> o =
                    pp_elem(pc, wv[u], Dv, hzv, Rr[u], gw[u], mu[u], nn[u], mm[u], ee[u], z0[u]);
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
                if (fabs(o.mu) > pc.mu_abort) {  // run_pp :119-124, kind 1
                    atomicMin(&a.fail_gstep[b * NR + q0 + u], a.alt->gstep_base + a.step);
                    atomicMin(&a.fail_idx[b * NR + q0 + u], (1 << 30) + i);
                }
                wn[u] = pp_next_w(pc, Rr[u], o.mu, z1[u]);
            }
            sy_st4(Cp + vi0, mu);
            sy_st4(Np + vi0, nn);
            sy_st4(Mp + vi0, mm);
            sy_st4(Ep + vi0, ee);
            sy_st4(MTp + vi0, mt);
            sy_st4(Wout + vi0, wn);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            double m = lmin[u];
#pragma unroll
            for (int off = 16; off >= QG; off >>= 1) {
                const double o = __shfl_xor_sync(0xffffffffu, m, off);
                m = o < m ? o : m;
            }
            if (lane < QG) s_min[wid][q0 + u] = m;
        }
        __syncthreads();
        if (t < NR) {
            double mn = INFINITY;
            for (int w = 0; w < NW; ++w) mn = s_min[w][t] < mn ? s_min[w][t] : mn;
            if (mn != INFINITY) atomicMin(&a.minE[b * NR + t], ord_key(mn));
        }
    } else if constexpr (MODE == EPI_JACOBI) {
        emit = true;
        if (valid) {
            const double Dv = __ldg(Dp + si), bv = __ldg(Hp + si);
            const double omd = sc.one_minus_dtc, dtc = sc.dt_c;
            double Rj[4], wo[4];
            sy_ld4(Rp + vi0, Rj);
            sy_ld4(Win + vi0, wo);
            const char4 s4 = *reinterpret_cast<const char4*>(a.sigma + vi0);
            const bool on4[4] = {s4.x != 0, s4.y != 0, s4.z != 0, s4.w != 0};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (fz[u]) continue;
                const bool on = on4[u];
                double rn = Rj[u];
                if (on) {
                    if (Dv == 0.0) {
                        atomicMin(a.err, sa.rowmap ? sa.rowmap[(size_t)b * a.ldN + i] : i);
                        continue;
                    }
                    const double off = gw[u] - Dv * Rj[u];
                    rn = omd * Rj[u] + dtc * ((bv - off) / Dv);
                    Rj[u] = rn;
                }
                wo[u] = rn * (on ? 1.0 : 0.0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) wn[u] = wo[u];
            sy_st4(Rp + vi0, Rj);
            sy_st4(Wout + vi0, wo);
        }
    } else if constexpr (MODE == EPI_MATVEC) {
        if (valid) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (!fz[u]) a.Mv[vi0 + u] = gw[u];
        }
    } else {  // EPI_SCORE
        double pa[4], pb[4], pc[4];
        double wv4[4] = {0.0, 0.0, 0.0, 0.0};
        if (valid) sy_ld4(Win + vi0, wv4);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pa[u] = pb[u] = pc[u] = 0.0;
            if (valid && !fz[u]) {
                const double wv = wv4[u];
                pa[u] = wv * gw[u];
                pb[u] = Hp[si] * wv;
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
        if (t < NR) {
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
    if (emit && sa.WTout) {  // the w tile of the next contraction (4 consecutive doubles)
        double* wt = sa.WTout + ((size_t)b * nRB + K) * (kT6 * NR);
        sy_st4(wt + s6_wofs<NR>(row, q0), wn);
    }
    sy_pdl_trigger();
    if (tl) tl[2] = sy_gtime();
}

}  // namespace cimcs
