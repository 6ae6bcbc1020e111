// dct_kernels.cuh -- matrix-free coupling of BASELINE config 3 (DCT o Haar^-1).
//
// Config 3's sensing matrix is A = S C2 Psi^-1: Psi = the L-level orthonormal
// Mallat 2-D Haar transform of a 128 x 128 image (the reference's average /
// difference split, mri.cpp:30-48 / 122-165, stopped after L levels), C2 = the
// orthonormal 2-D DCT-II (X -> C X C^T, C the 128 x 128 DCT matrix) and S the
// selection of M frequencies.  The dense path stores G = A^T A (16384^2, 537 MB
// of fp16 hi/lo tiles per step); the chain applies it instead:
//     G w = Psi C^T (mask o (C (Psi^-1 w) C^T)) C,
// four 128-point matrix products and two Haar transforms per vector.  One
// thread-block cluster of 8 CTAs owns one vector; CTA k owns image rows
// [16k, 16k + 16) in the row phases and image columns [16k, 16k + 16) in the
// column phases, so every product is a 16 x 128 x 128 (or 128 x 16 x 128)
// slab GEMM on mma.sync m16n8k8 TF32 in the 3xTF32 split (a_hi b_hi + a_hi b_lo
// + a_lo b_hi: fp32-level accuracy), one m16 x n16 block per warp:
//   1. X   = Psi^-1 w, own rows (each pixel evaluated directly from its 3L + 1
//            coefficients: an L <= 3 level Haar block is 8 x 8, inside the slab);
//   2. Z   = X C^T, own rows; block (own rows, columns of CTA p) -> CTA p (DSMEM);
//   3. Y   = C Z, own columns, masked                  (cluster barrier before);
//   4. U   = C^T Y, own columns; block (rows of CTA p, own columns) -> CTA p;
//   5. X'  = U C, own rows                             (cluster barrier before);
//   6. G w = Psi X' of the own rows' coefficients (signed sums over their
//            2^l x 2^l supports in the slab).
// Only two 8 KB block all-to-alls cross the cluster.  C is stored pre-swizzled
// in global memory and lands in shared memory with one bulk copy that overlaps
// phase 1; shared memory is 104 KB, so two clusters share an SM and the 16
// replicas of config 3 run in one wave on 64 SMs.  Row-major 128-float
// matrices have their columns XOR-swizzled by dsw(row) (all fragment patterns
// conflict-free); the column slabs use a 24-float row stride.  G w lands in the
// transform-chain slot buffer ([N][NR]) and sym_update_kernel runs the fused
// epilogue, as for the DFT chain (mri_kernels.cuh) -- including the damped
// Jacobi refit, which the dense config-3 problem uses (D = diag G from the
// chain on basis vectors).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace cimcs {

constexpr int kDctN = 128;                 // image edge
constexpr int kDctCS = 8;                  // CTAs per cluster (one vector per cluster)
constexpr int kDctRH = kDctN / kDctCS;     // rows (columns) of a slab = one m16 tile
constexpr int kDctThreads = 256;           // 8 warps: warp w <-> slab block / peer w
constexpr int kDctMaxLevels = 3;           // Haar block 8 x 8 <= kDctRH
constexpr int kDctCStr = 24;               // column-slab row stride (conflict-free B reads)

enum { DCT_APPLY = 0, DCT_HZ = 1, DCT_DIAG = 2, DCT_COLS = 3 };

struct DctArgs {
    int NR;                       // APPLY: slots of w / out ([N][NR])
    const float* C;               // [128][128] orthonormal DCT-II, PRE-SWIZZLED (dofs)
    const unsigned char* mask;    // [128 * 128] frequency (u, v) sampled
    const float* in;              // APPLY: w [N][NR]; HZ: y scattered on the frequency grid
    float* out;                   // APPLY: G w [N][NR]; HZ: hz [N]; DIAG: D [N]; COLS: rows of G
    int r0;                       // DIAG / COLS: first basis vector of this launch
};

constexpr size_t kDctMat = (size_t)kDctN * kDctN;  // floats per 128 x 128 matrix
constexpr size_t kDctSlab = (size_t)kDctRH * kDctN;
constexpr size_t kDctCSlab = (size_t)kDctN * kDctCStr;
inline constexpr size_t dct_smem_bytes() { return (kDctMat + 2 * kDctSlab + 2 * kDctCSlab) * 4 + 16; }

// column swizzle of row i: conflict-free for (8 rows x 4 columns) and
// (4 rows x 8 columns) fragment patterns; a multiple of 4 (float4 groups stay whole)
__host__ __device__ __forceinline__ int dsw(int i) { return ((i & 3) << 3) | (((i >> 2) & 1) << 2); }
__host__ __device__ __forceinline__ int dofs(int i, int j) { return i * kDctN + (j ^ dsw(i)); }

// 3xTF32 operand split: hi = x truncated to TF32 (sign, exponent, 10 mantissa
// bits), lo = x - hi (exact in fp32; the MMA reads its top 19 bits)
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(x) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// One warp's 16 x 16 output block: d[t][.] = sum_k A(m, k) B(k, 8 t + n) over
// k < 128, A / B read through the functors (block-relative m, n), 3xTF32
template <typename FA, typename FB>
__device__ __forceinline__ void dct_block_mm(float (&d)[2][4], FA fa, FB fb) {
    const int lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) d[t][e] = 0.f;
#pragma unroll 4
    for (int k0 = 0; k0 < kDctN; k0 += 8) {
        uint32_t ah[4], al[4];
        tf32_split(fa(gid, k0 + t4), ah[0], al[0]);
        tf32_split(fa(gid + 8, k0 + t4), ah[1], al[1]);
        tf32_split(fa(gid, k0 + t4 + 4), ah[2], al[2]);
        tf32_split(fa(gid + 8, k0 + t4 + 4), ah[3], al[3]);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            uint32_t bh0, bl0, bh1, bl1;
            tf32_split(fb(k0 + t4, 8 * t + gid), bh0, bl0);
            tf32_split(fb(k0 + t4 + 4, 8 * t + gid), bh1, bl1);
            mma_tf32(d[t], al[0], al[1], al[2], al[3], bh0, bh1);  // small terms first
            mma_tf32(d[t], ah[0], ah[1], ah[2], ah[3], bl0, bl1);
            mma_tf32(d[t], ah[0], ah[1], ah[2], ah[3], bh0, bh1);
        }
    }
}

// accumulator pair h (elements 2h, 2h + 1) of tile t: block-relative row, column
__device__ __forceinline__ int dct_acc_row(int h) { return ((threadIdx.x & 31) >> 2) + 8 * h; }
__device__ __forceinline__ int dct_acc_col(int t) { return 8 * t + 2 * (threadIdx.x & 3); }

// the t-th of the 2048 Haar coefficients whose support lies in the slab of
// cluster rank kc: (row, column) in the Mallat layout, level l, sub-band sb
// (0 LL_L, 1 column detail at (a, s + b), 2 row detail at (s + a, b), 3 both)
struct DctCoef {
    int row, col, l, sb, a, b;
};
template <int L>
__device__ __forceinline__ DctCoef dct_coef(int t, int kc) {
#pragma unroll
    for (int l = 1; l <= L; ++l) {
        constexpr int kRH = kDctRH;
        const int ra = kRH >> l, s = kDctN >> l, cnt = 3 * ra * s;
        if (t < cnt) {
            const int sb = 1 + t / (ra * s), u = t % (ra * s);
            const int a = ((kc * kRH) >> l) + u / s, b = u % s;
            return {sb == 1 ? a : s + a, sb == 2 ? b : s + b, l, sb, a, b};
        }
        t -= cnt;
    }
    const int s = kDctN >> L;
    const int a = ((kc * kDctRH) >> L) + t / s, b = t % s;
    return {a, b, L, 0, a, b};
}

template <int L>
__global__ void __launch_bounds__(kDctThreads, 2) dct_cluster_kernel(DctArgs a, int mode) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(128) float dsm[];
    float* Cm = dsm;                  // C (swizzled)
    float* RS = Cm + kDctMat;         // row slab: X, later X'
    float* RS2 = RS + kDctSlab;       // row slab: U (filled by the peers)
    float* CS = RS2 + kDctSlab;       // column slab: Z (filled by the peers)
    float* CS2 = CS + kDctCSlab;      // column slab: masked Y
    uint64_t* bar = reinterpret_cast<uint64_t*>(CS2 + kDctCSlab);
    const int kc = (int)cl.block_rank(), q = blockIdx.x / kDctCS;
    const int row0 = kc * kDctRH;
    const int tid = threadIdx.x, w = tid >> 5;
    if (tid == 0) {  // C: one bulk copy, overlapping phase 1
        mbar_init(bar, 1);
        mbar_fence_init();
        mbar_arrive_expect_tx(bar, (uint32_t)(kDctMat * 4));
        sy_bulk_g2s(Cm, a.C, (uint32_t)(kDctMat * 4), bar, sy_policy_last());
    }
    cl.sync();  // every CTA of the cluster is resident before any DSMEM store
    // programmatic dependent launch: the update kernel may be scheduled now; the
    // reads of w wait for the previous step's update kernel
    sy_pdl_trigger();
    sy_pdl_wait();
    float d[2][4];
    if (mode != DCT_HZ) {
        // 1. X = Psi^-1 w, own rows: the slab's 2048 coefficients staged (one
        //    load each, in dct_coef order), then L inverse levels coarsest first
        //    (column merge, then row merge: mri.cpp:143-165)
        const int rb = mode == DCT_APPLY ? -1 : a.r0 + q;  // basis vector of DIAG / COLS
        float* stg = CS2;                   // [2048] staged coefficients
        float* llb[2] = {CS2 + kDctSlab, CS2 + kDctSlab + 512};
#pragma unroll
        for (int u = 0; u < (int)kDctSlab / kDctThreads; ++u) {
            const int t = tid + u * kDctThreads;
            const DctCoef cf = dct_coef<L>(t, kc);
            const int idx = cf.row * kDctN + cf.col;
            stg[t] = rb < 0 ? __ldg(a.in + (size_t)idx * a.NR + q) : (idx == rb ? 1.f : 0.f);
        }
        __syncthreads();
        {
            const float sq = 0.70710678118654752440f;
            int off = 0;  // detail offset of level l in the staged order
#pragma unroll
            for (int l = 1; l <= L; ++l) off += 3 * (kDctRH >> l) * (kDctN >> l);
            const float* cur = stg + off;  // LL_L
#pragma unroll
            for (int l = L; l >= 1; --l) {
                const int ra = kDctRH >> l, sl = kDctN >> l;
                off -= 3 * ra * sl;
                float* nxt = llb[l & 1];
                for (int e = tid; e < ra * sl; e += kDctThreads) {
                    const int al = e / sl, bb = e % sl;
                    const float LL = cur[e], HL = stg[off + e], LH = stg[off + ra * sl + e],
                                HH = stg[off + 2 * ra * sl + e];
                    const float c00 = (LL + LH) * sq, c10 = (LL - LH) * sq;
                    const float c01 = (HL + HH) * sq, c11 = (HL - HH) * sq;
                    const float x00 = (c00 + c01) * sq, x01 = (c00 - c01) * sq;
                    const float x10 = (c10 + c11) * sq, x11 = (c10 - c11) * sq;
                    if (l == 1) {
                        *reinterpret_cast<float2*>(RS + dofs(2 * al, 2 * bb)) = make_float2(x00, x01);
                        *reinterpret_cast<float2*>(RS + dofs(2 * al + 1, 2 * bb)) = make_float2(x10, x11);
                    } else {
                        *reinterpret_cast<float2*>(nxt + (2 * al) * (2 * sl) + 2 * bb) = make_float2(x00, x01);
                        *reinterpret_cast<float2*>(nxt + (2 * al + 1) * (2 * sl) + 2 * bb) =
                            make_float2(x10, x11);
                    }
                }
                __syncthreads();
                cur = nxt;
            }
        }
        mbar_wait(bar, 0);
        // 2. Z = X C^T, own rows; warp w's 16 columns go to CTA w's column slab
        dct_block_mm(d, [&](int m, int k) { return RS[dofs(m, k)]; },
                     [&](int k, int n) { return Cm[dofs(16 * w + n, k)]; });
        {
            float* dst = cl.map_shared_rank(CS, w);
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    *reinterpret_cast<float2*>(dst + (row0 + dct_acc_row(h)) * kDctCStr +
                                               dct_acc_col(t)) =
                        make_float2(d[t][2 * h], d[t][2 * h + 1]);
        }
        cl.sync();
        // 3. Y = C Z, own columns (warp w: frequency rows 16 w ..), masked
        dct_block_mm(d, [&](int m, int k) { return Cm[dofs(16 * w + m, k)]; },
                     [&](int k, int n) { return CS[k * kDctCStr + n]; });
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int r = 16 * w + dct_acc_row(e >> 1), c = dct_acc_col(t) + (e & 1);
                CS2[r * kDctCStr + c] = __ldg(a.mask + r * kDctN + row0 + c) ? d[t][e] : 0.f;
            }
    } else {
        // hz = Psi C^T Y C with Y = the observations on the frequency grid
        for (int p = tid; p < kDctN * kDctRH; p += kDctThreads) {
            const int r = p >> 4, c = p & (kDctRH - 1);
            CS2[r * kDctCStr + c] = __ldg(a.in + (size_t)r * kDctN + row0 + c);
        }
        mbar_wait(bar, 0);
    }
    __syncthreads();
    // 4. U = C^T Y, own columns (warp w: image rows 16 w .., owned by CTA w)
    dct_block_mm(d, [&](int m, int k) { return Cm[dofs(k, 16 * w + m)]; },
                 [&](int k, int n) { return CS2[k * kDctCStr + n]; });
    {
        float* dst = cl.map_shared_rank(RS2, w);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                *reinterpret_cast<float2*>(dst + dofs(dct_acc_row(h), row0 + dct_acc_col(t))) =
                    make_float2(d[t][2 * h], d[t][2 * h + 1]);
    }
    cl.sync();
    // 5. X' = U C, own rows (warp w: columns 16 w ..)
    dct_block_mm(d, [&](int m, int k) { return RS2[dofs(m, k)]; },
                 [&](int k, int n) { return Cm[dofs(k, 16 * w + n)]; });
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h)
            *reinterpret_cast<float2*>(RS + dofs(dct_acc_row(h), 16 * w + dct_acc_col(t))) =
                make_float2(d[t][2 * h], d[t][2 * h + 1]);
    __syncthreads();
    // 6. forward Haar of the own rows, level by level (row split, then column
    //    split: mri.cpp:122-141); details go straight to their Mallat positions
    {
        const int rb = a.r0 + q;
        auto emit = [&](int idx, float v) {
            if (mode == DCT_APPLY)
                a.out[(size_t)idx * a.NR + q] = v;
            else if (mode == DCT_HZ)
                a.out[idx] = v;
            else if (mode == DCT_DIAG) {
                if (idx == rb) a.out[idx] = v;
            } else {
                a.out[(size_t)rb * kDctMat + idx] = v;
            }
        };
        const float sq = 0.70710678118654752440f;
        float* llb[2] = {CS, CS + 512};
        const float* in = RS;
#pragma unroll
        for (int l = 1; l <= L; ++l) {
            const int ra = kDctRH >> l, sl = kDctN >> l, a0 = row0 >> l;
            float* nxt = llb[l & 1];
            for (int e = tid; e < ra * sl; e += kDctThreads) {
                const int al = e / sl, bb = e % sl;
                float x00, x01, x10, x11;
                if (l == 1) {
                    const float2 r0v = *reinterpret_cast<const float2*>(RS + dofs(2 * al, 2 * bb));
                    const float2 r1v = *reinterpret_cast<const float2*>(RS + dofs(2 * al + 1, 2 * bb));
                    x00 = r0v.x; x01 = r0v.y; x10 = r1v.x; x11 = r1v.y;
                } else {
                    const float2 r0v = *reinterpret_cast<const float2*>(in + (2 * al) * (2 * sl) + 2 * bb);
                    const float2 r1v =
                        *reinterpret_cast<const float2*>(in + (2 * al + 1) * (2 * sl) + 2 * bb);
                    x00 = r0v.x; x01 = r0v.y; x10 = r1v.x; x11 = r1v.y;
                }
                const float p0 = (x00 + x01) * sq, p1 = (x00 - x01) * sq;
                const float q0 = (x10 + x11) * sq, q1 = (x10 - x11) * sq;
                const int ga = a0 + al;
                emit(ga * kDctN + sl + bb, (p1 + q1) * sq);           // column detail
                emit((sl + ga) * kDctN + bb, (p0 - q0) * sq);         // row detail
                emit((sl + ga) * kDctN + sl + bb, (p1 - q1) * sq);    // both
                const float LLv = (p0 + q0) * sq;
                if (l == L)
                    emit(ga * kDctN + bb, LLv);
                else
                    nxt[e] = LLv;
            }
            if (l < L) __syncthreads();
            in = nxt;
        }
    }
}

}  // namespace cimcs
