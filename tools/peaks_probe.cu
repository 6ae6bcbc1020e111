// Peak probes for the roofline denominators SURVEY 8(d) asks for, measured on
// the box: L2 read bandwidth (working sets 8..96 MB), HBM read bandwidth (2 GB),
// FP64 DFMA, FP64 DMMA (mma.sync m8n8k4 f64) and FP32 FFMA throughput; and the
// rounding semantics of the f64 DMMA (is it an fma chain over k?).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/peaks_probe tools/peaks_probe.cu
//   tools/peaks_probe [out.json] [dmma_vectors.bin]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

__global__ void read_kernel(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
            float4 v;
            asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "l"(p + i));
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 12345.f) *sink = acc;
}

__global__ void dfma_kernel(double* out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4,
           a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 1.2345) out[0] = s;
}

__global__ void ffma_kernel(float* out, int iters) {
    float a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-3f + k;
    const float b = 0.9999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < 16; ++k) a[k] = fmaf(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    if (s == 1.2345f) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0,
                                     double c1) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d0), "=d"(d1)
                 : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

__global__ void dmma_kernel(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
    double c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            dmma(c[0], c[1], a, b, c[0], c[1]);
            dmma(c[2], c[3], a, b, c[2], c[3]);
            dmma(c[4], c[5], a, b, c[4], c[5]);
            dmma(c[6], c[7], a, b, c[6], c[7]);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k];
    if (s == 1.2345) out[0] = s;
}

// one m8n8k4 per warp on given A (8x4 row-major), B (4x8: B[k][n]), C (8x8)
__global__ void dmma_semantics(const double* A, const double* B, const double* C, double* D,
                               int ncase) {
    const int lane = threadIdx.x & 31, w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= ncase) return;
    const double* a = A + (size_t)w * 32;
    const double* b = B + (size_t)w * 32;
    const double* c = C + (size_t)w * 64;
    const int g = lane >> 2, t = lane & 3;
    double d0, d1;
    dmma(d0, d1, a[g * 4 + t], b[t * 8 + g], c[g * 8 + 2 * t], c[g * 8 + 2 * t + 1]);
    D[(size_t)w * 64 + g * 8 + 2 * t] = d0;
    D[(size_t)w * 64 + g * 8 + 2 * t + 1] = d1;
}

template <class F>
float time_ms(F&& f, int reps) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    f();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0));
        f();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    return best;
}

int main(int argc, char** argv) {
    const char* outp = argc > 1 ? argv[1] : "peaks.json";
    const char* vecp = argc > 2 ? argv[2] : nullptr;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    FILE* fo = fopen(outp, "w");
    fprintf(fo, "{\n \"sms\": %d,\n", sms);
    float* sink;
    CK(cudaMalloc(&sink, 64));
    // --- L2 / HBM read bandwidth
    const size_t big = (size_t)2 << 30;
    float4* buf;
    CK(cudaMalloc(&buf, big));
    CK(cudaMemset(buf, 0, big));
    fprintf(fo, " \"read_gbs\": {");
    const size_t sizes_mb[] = {8, 16, 24, 32, 48, 64, 80, 96, 2048};
    for (int s = 0; s < 9; ++s) {
        const size_t bytes = sizes_mb[s] << 20;
        const size_t n4 = bytes / 16;
        const int reps = sizes_mb[s] >= 2048 ? 1 : (int)(4096 / sizes_mb[s]);
        float ms = time_ms([&] { read_kernel<<<sms * 4, 512>>>(buf, n4, reps, sink); }, 5);
        double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
        fprintf(fo, "%s\"%zu_MB\": %.1f", s ? ", " : "", sizes_mb[s], gbs);
        printf("read %5zu MB x %4d: %.1f GB/s\n", sizes_mb[s], reps, gbs);
    }
    fprintf(fo, "},\n");
    // --- FP64 DFMA
    {
        const int iters = 4096;
        double* o;
        CK(cudaMalloc(&o, 64));
        float ms = time_ms([&] { dfma_kernel<<<sms * 8, 256>>>(o, iters); }, 3);
        double fl = 2.0 * 8 * 8 * (double)iters * sms * 8 * 256;
        fprintf(fo, " \"dfma_tflops\": %.2f,\n", fl / (ms * 1e-3) / 1e12);
        printf("DFMA %.2f TFLOP/s\n", fl / (ms * 1e-3) / 1e12);
        ms = time_ms([&] { dmma_kernel<<<sms * 8, 256>>>(o, iters); }, 3);
        fl = 2.0 * 256 * 32 * (double)iters * sms * 8 * 256 / 32;  // per warp: 32 mma x 256 FMA
        fprintf(fo, " \"dmma_tflops\": %.2f,\n", fl / (ms * 1e-3) / 1e12);
        printf("DMMA %.2f TFLOP/s\n", fl / (ms * 1e-3) / 1e12);
        float* of;
        CK(cudaMalloc(&of, 64));
        ms = time_ms([&] { ffma_kernel<<<sms * 8, 256>>>(of, iters); }, 3);
        fl = 2.0 * 8 * 16 * (double)iters * sms * 8 * 256;
        fprintf(fo, " \"ffma_tflops\": %.2f,\n", fl / (ms * 1e-3) / 1e12);
        printf("FFMA %.2f TFLOP/s\n", fl / (ms * 1e-3) / 1e12);
    }
    // --- DMMA rounding semantics: random cases, dumped for an exact host check
    {
        const int ncase = 4096;
        std::mt19937_64 g(12345);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        std::uniform_int_distribution<int> ex(-30, 30);
        std::vector<double> A(ncase * 32), B(ncase * 32), C(ncase * 64), D(ncase * 64);
        for (auto& v : A) v = std::ldexp(u(g), ex(g));
        for (auto& v : B) v = std::ldexp(u(g), ex(g));
        for (auto& v : C) v = std::ldexp(u(g), ex(g));
        double *dA, *dB, *dC, *dD;
        CK(cudaMalloc(&dA, A.size() * 8));
        CK(cudaMalloc(&dB, B.size() * 8));
        CK(cudaMalloc(&dC, C.size() * 8));
        CK(cudaMalloc(&dD, D.size() * 8));
        CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
        dmma_semantics<<<ncase / 4, 128>>>(dA, dB, dC, dD, ncase);
        CK(cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost));
        int chain = 0, chain_rev = 0;
        for (int w = 0; w < ncase; ++w)
            for (int m = 0; m < 8; ++m)
                for (int n = 0; n < 8; ++n) {
                    double acc = C[w * 64 + m * 8 + n];
                    for (int k = 0; k < 4; ++k)
                        acc = std::fma(A[w * 32 + m * 4 + k], B[w * 32 + k * 8 + n], acc);
                    double acc2 = C[w * 64 + m * 8 + n];
                    for (int k = 3; k >= 0; --k)
                        acc2 = std::fma(A[w * 32 + m * 4 + k], B[w * 32 + k * 8 + n], acc2);
                    chain += acc == D[w * 64 + m * 8 + n];
                    chain_rev += acc2 == D[w * 64 + m * 8 + n];
                }
        fprintf(fo, " \"dmma_equals_fma_chain_k0123\": %d,\n \"dmma_equals_fma_chain_k3210\": %d,\n"
                    " \"dmma_cases\": %d\n}\n", chain, chain_rev, ncase * 64);
        printf("DMMA == fma chain k0..3: %d / %d; k3..0: %d\n", chain, ncase * 64, chain_rev);
        if (vecp) {
            FILE* fv = fopen(vecp, "wb");
            fwrite(A.data(), 8, A.size(), fv);
            fwrite(B.data(), 8, B.size(), fv);
            fwrite(C.data(), 8, C.size(), fv);
            fwrite(D.data(), 8, D.size(), fv);
            fclose(fv);
        }
    }
    fclose(fo);
    return 0;
}
