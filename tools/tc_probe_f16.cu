// tc_probe_f16.cu -- can one shared-memory tile of G serve both G*W and G^T*W
// on tcgen05 kind::f16?  The tile is stored K-major (canonical, no swizzle) for
// the first product; the second reads the SAME bytes as an MN-major operand.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tc_probe_f16 tools/tc_probe_f16.cu
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define T 128   // tile edge (i and j)
#define NN 16   // replicas (MMA N)

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major canonical (no swizzle) for an (MN x K) fp16 operand: core = 8 MN rows x 8 K
// (16 B) ; rows 16 B apart; MN core groups at SBO, K core groups at LBO.
__host__ __device__ inline int offK(int mn, int k, int MN) {
    return (k / 8) * (MN / 8) * 128 + (mn / 8) * 128 + (mn % 8) * 16 + (k % 8) * 2;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// use = 0: D = A * B   (A = tile, M = i, K = j, K-major)
// use = 1: D = A^T * B (A' = tile^T, M = j, K = i, MN-major view of the same bytes)
__global__ void probe(const half* G, const half* W, float* D, int use, int variant) {
    __shared__ __align__(1024) unsigned char sA[T * T * 2];
    __shared__ __align__(1024) unsigned char sB[T * NN * 2];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x;
    for (int e = t; e < T * T; e += blockDim.x) {
        const int i = e / T, j = e % T;  // G[i][j] row-major in global
        *reinterpret_cast<half*>(sA + offK(i, j, T)) = G[e];
    }
    for (int e = t; e < T * NN; e += blockDim.x) {
        const int k = e / NN, n = e % NN;  // W[k][n]
        *reinterpret_cast<half*>(sB + offK(n, k, NN)) = W[e];
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tbase;
    const uint32_t amn = use;  // transpose-A bit
    const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | (amn << 15) | (0u << 16) |
                           ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(T >> 4) << 24);
    if (t == 0) {
        for (int kb = 0; kb < T / 16; ++kb) {
            uint64_t da;
            const uint32_t kstride = (T / 8) * 128;  // stored LBO (j groups) ; SBO = 128 (i groups)
            if (use == 0) {
                da = sdesc(su32(sA) + kb * 2 * kstride, kstride, 128);
            } else {
                // A' = tile^T: MN' = j (stored K dir, group stride kstride), K' = i (stored MN
                // dir, group stride 128).  K' step of 16 = 2 i-groups = 256 B.
                uint32_t lbo = kstride, sbo = 128;
                if (variant & 1) { uint32_t x = lbo; lbo = sbo; sbo = x; }
                da = sdesc(su32(sA) + kb * 256, lbo, sbo);
            }
            const uint64_t db = sdesc(su32(sB) + kb * 2 * (NN / 8) * 128, (NN / 8) * 128, 128);
            const uint32_t acc = kb ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int w = t / 32, lane = t % 32;
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
                   "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(32 * w) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int n = 0; n < 16; ++n) D[(32 * w + lane) * NN + n] = __uint_as_float(r[n]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
    std::vector<half> G(T * T), W(T * NN);
    std::vector<float> Gf(T * T), Wf(T * NN), D(T * NN);
    srand(3);
    for (int e = 0; e < T * T; ++e) { G[e] = __float2half((float)rand() / RAND_MAX - 0.5f); Gf[e] = __half2float(G[e]); }
    for (int e = 0; e < T * NN; ++e) { W[e] = __float2half((float)rand() / RAND_MAX - 0.5f); Wf[e] = __half2float(W[e]); }
    half *dG, *dW;
    float* dD;
    cudaMalloc(&dG, G.size() * 2);
    cudaMalloc(&dW, W.size() * 2);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dG, G.data(), G.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 2, cudaMemcpyHostToDevice);
    for (int use = 0; use < 2; ++use)
        for (int variant = 0; variant < (use ? 2 : 1); ++variant) {
            cudaMemset(dD, 0, D.size() * 4);
            probe<<<1, 128>>>(dG, dW, dD, use, variant);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0, maxref = 0;
            for (int m = 0; m < T; ++m)
                for (int n = 0; n < NN; ++n) {
                    double s = 0;
                    for (int k = 0; k < T; ++k)
                        s += (double)(use ? Gf[k * T + m] : Gf[m * T + k]) * Wf[k * NN + n];
                    maxerr = fmax(maxerr, fabs(s - D[m * NN + n]));
                    maxref = fmax(maxref, fabs(s));
                }
            printf("use %d (%s) variant %d: max err %.3e (max |ref| %.3f) D[0]=%f\n", use,
                   use ? "A^T, MN-major view" : "A, K-major", variant, maxerr, maxref, D[0]);
        }
    return 0;
}
