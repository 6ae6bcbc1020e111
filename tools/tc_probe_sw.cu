// tc_probe_sw.cu -- does tcgen05 kind::tf32 accept SWIZZLE_128B K-major and
// MN-major A operands (the latter = the transpose of the former)?
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#define M 128
#define N 16
#define K 32
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// A K-major SW128: rows of 32 k (128 B), 8-row atoms (1 KB), chunk (k/4) xor (m%8)
__host__ __device__ inline int offAK(int m, int k) { return (m / 8) * 1024 + (m % 8) * 128 + (((k / 4) ^ (m % 8)) * 16) + (k % 4) * 4; }
// A MN-major SW128: 32 m per 128 B row, 8 k-rows per atom; m-atoms at LBO=1024 (K=8 only)
__host__ __device__ inline int offAMN(int m, int k) { return (k / 8) * 4096 + (m / 32) * 1024 + (k % 8) * 128 + ((((m % 32) / 4) ^ (k % 8)) * 16) + (m % 4) * 4; }
// B K-major no swizzle (known good)
__host__ __device__ inline int offB(int k, int n) { return (k / 4) * (N / 8) * 128 + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4; }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__global__ void probe(const float* A, const float* B, float* D, int mode) {
    __shared__ __align__(1024) unsigned char sA[M * K * 4 + 4096];
    __shared__ __align__(1024) unsigned char sB[K * N * 4];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x;
    for (int e = t; e < M * K; e += blockDim.x) {
        const int m = e / K, k = e % K;
        *reinterpret_cast<float*>(sA + (mode ? offAMN(m, k) : offAK(m, k))) = A[m * K + k];
    }
    for (int e = t; e < K * N; e += blockDim.x) {
        const int k = e / N, n = e % N;
        *reinterpret_cast<float*>(sB + offB(k, n)) = B[k * N + n];
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(mode ? 1 : 0) << 15) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (t == 0) {
        for (int kb = 0; kb < K / 8; ++kb) {
            uint64_t da;
            if (mode == 0) da = sdesc(su32(sA) + kb * 32, 16, 1024, 2);        // K-major SW128: advance 32 B per k-block
            else da = sdesc(su32(sA) + kb * 4096, 1024, 4096, 2);              // MN-major SW128: LBO = m-atom stride
            const uint64_t db = sdesc(su32(sB) + kb * 2 * (N / 8) * 128, (N / 8) * 128, 128, 0);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(kb ? 1u : 0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int w = t / 32, lane = t % 32;
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(32 * w) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int n = 0; n < 16; ++n) D[(32 * w + lane) * N + n] = __uint_as_float(r[n]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}
static float tr(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x; }
int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    std::vector<float> A(M * K), B(K * N), D(M * N);
    srand(3);
    for (auto& v : A) v = tr((float)rand() / RAND_MAX - 0.5f);
    for (auto& v : B) v = tr((float)rand() / RAND_MAX - 0.5f);
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d CUDA error %s\n", mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double s = 0; for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[k * N + n];
        maxerr = fmax(maxerr, fabs(s - D[m * N + n]));
    }
    printf("mode %d (%s SW128 A): err %.3e D[1]=%f\n", mode, mode ? "MN-major" : "K-major", maxerr, D[1]);
    return 0;
}
