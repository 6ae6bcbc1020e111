// tc_probe.cu -- standalone check of the tcgen05 kind::tf32 encodings used by the
// fp32 tensor-core step (canonical no-swizzle MN-major smem operands, F32
// accumulator in TMEM), plus how fp32 inputs are converted to tf32.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tc_probe tools/tc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#define M 128
#define N 16
#define K 32  // 4 MMAs of K=8

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// A (M x K) element (m,k): (k/8)*LBO_A + (m/4)*128 + (k%8)*16 + (m%4)*4
__device__ int g_kmajor = 0;
// MN-major interleave: core matrix = 4 MN x 8 K (K rows 16 B apart)
// K-major interleave:  core matrix = 8 MN x 4 K (MN rows 16 B apart)
__host__ __device__ inline int offA(int m, int k, int km) {
    return km ? (k / 4) * (M / 8) * 128 + (m / 8) * 128 + (m % 8) * 16 + (k % 4) * 4
              : (k / 8) * (M / 4) * 128 + (m / 4) * 128 + (k % 8) * 16 + (m % 4) * 4;
}
__host__ __device__ inline int offB(int k, int n, int km) {
    return km ? (k / 4) * (N / 8) * 128 + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4
              : (k / 8) * (N / 4) * 128 + (n / 4) * 128 + (k % 8) * 16 + (n % 4) * 4;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm100)
    // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
    return d;
}

__global__ void probe(const float* A, const float* B, float* D, int passes, int km, int sanity, int amn, int bmn, int swap) {
    __shared__ __align__(1024) unsigned char sA[M * K * 4];
    __shared__ __align__(1024) unsigned char sB[K * N * 4];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x;
    for (int e = t; e < M * K; e += blockDim.x) {
        const int m = e / K, k = e % K;
        *reinterpret_cast<float*>(sA + offA(m, k, amn ? 0 : 1)) = A[m * K + k];
    }
    for (int e = t; e < K * N; e += blockDim.x) {
        const int k = e / N, n = e % N;
        *reinterpret_cast<float*>(sB + offB(k, n, bmn ? 0 : 1)) = B[k * N + n];
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
    // idesc: F32 accum, A/B TF32, both MN-major, N>>3, M>>4
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (sanity) {
        const int w = t / 32;
        uint32_t v[16];
        for (int n = 0; n < 16; ++n) v[n] = __float_as_uint((float)(1000 * t + n));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     :: "r"(tmem + ((uint32_t)(32 * w) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                     "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (t == 0 && !sanity) {
        for (int p = 0; p < passes; ++p)
            for (int kb = 0; kb < K / 8; ++kb) {
                // MN-major: SBO = MN-group stride (128), LBO = K-group stride
                // K-major : SBO = MN 8-row group stride (128), LBO = K 4-col group stride
                uint32_t la = amn ? (M / 4) * 128 : (M / 8) * 128, sa = 128;
                uint32_t lb = bmn ? (N / 4) * 128 : (N / 8) * 128, sb = 128;
                if (swap & 1) { uint32_t t = la; la = sa; sa = t; }
                if (swap & 2) { uint32_t t = lb; lb = sb; sb = t; }
                const uint64_t da = amn ? sdesc(su32(sA) + kb * (M / 4) * 128, la, sa)
                                        : sdesc(su32(sA) + kb * 2 * (M / 8) * 128, la, sa);
                const uint64_t db = bmn ? sdesc(su32(sB) + kb * (N / 4) * 128, lb, sb)
                                        : sdesc(su32(sB) + kb * 2 * (N / 8) * 128, lb, sb);
                const uint32_t acc = (p | kb) ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
    }
    if (t == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    // wait for the MMAs
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int w = t / 32, lane = t % 32;
    const uint32_t taddr = tmem + ((uint32_t)(32 * w) << 16);
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
                   "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = 32 * w + lane;
    for (int n = 0; n < 16; ++n) D[m * N + n] = __uint_as_float(r[n]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

static float trunc_tf32(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    memcpy(&x, &u, 4);
    return x;
}

static double run(float* dA, float* dB, float* dD, std::vector<float>& A, std::vector<float>& B,
                  std::vector<float>& D, int amn, int bmn, int swap, int sanity) {
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128>>>(dA, dB, dD, 1, 0, sanity, amn, bmn, swap);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            if (sanity) s = 1000.0 * m + n;
            else for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[k * N + n];
            maxerr = fmax(maxerr, fabs(s - D[m * N + n]));
        }
    return maxerr;
}

int main(int argc, char** argv) {
    const int amn = argc > 1 ? atoi(argv[1]) : 0, bmn = argc > 2 ? atoi(argv[2]) : 0,
              swap = argc > 3 ? atoi(argv[3]) : 0;
    std::vector<float> A(M * K), B(K * N), D(M * N);
    srand(1);
    for (auto& v : A) v = trunc_tf32((float)rand() / RAND_MAX - 0.5f);
    for (auto& v : B) v = trunc_tf32((float)rand() / RAND_MAX - 0.5f);
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    double e = run(dA, dB, dD, A, B, D, amn, bmn, swap, 0);
    printf("A %s B %s swap %d : err %.3e  D[1]=%f\n", amn ? "MN" : "K ", bmn ? "MN" : "K ", swap, e, D[1]);
    return 0;
}
