// What does ONE SM ingest with cp.async.bulk (global -> shared) as a function of the
// bytes it keeps in flight, and does it depend on how many SMs stream?  One CTA per
// SM, one thread issuing `chunk`-byte bulk copies into a ring of `stages` slots
// (slot s is re-issued as soon as its mbarrier completes: no compute), each CTA
// walking its own contiguous region of a 2 GB buffer (HBM-resident stream).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/bulk_probe tools/bulk_probe.cu
//   /tmp/bulk_probe [out.json]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                             \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                          \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));    \
            exit(1);                                                                      \
        }                                                                                 \
    } while (0)

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) bulk_kernel(const unsigned char* __restrict__ src, size_t per_cta,
                                                     int chunk, int stages, int n_chunks) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const unsigned char* p = src + (size_t)blockIdx.x * per_cta;
    auto issue = [&](int i) {
        const int s = i % stages;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(chunk)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                s32(smem + (size_t)s * chunk)),
            "l"(p + (size_t)i * chunk), "r"(chunk), "r"(s32(&bar[s]))
            : "memory");
    };
    for (int i = 0; i < stages && i < n_chunks; ++i) issue(i);
    for (int i = 0; i < n_chunks; ++i) {
        const int s = i % stages;
        const uint32_t ph = (i / stages) & 1;
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(ok)
                : "r"(s32(&bar[s])), "r"(ph)
                : "memory");
        if (i + stages < n_chunks) issue(i + stages);
    }
}

int main(int argc, char** argv) {
    const size_t total = (size_t)2 << 30;
    unsigned char* d;
    CK(cudaMalloc(&d, total));
    CK(cudaMemset(d, 1, total));
    CK(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    FILE* f = argc > 1 ? fopen(argv[1], "w") : nullptr;
    if (f) fprintf(f, "[\n");
    bool first = true;
    const int grids[] = {148, 111, 74, 37};
    const int chunks[] = {32768, 16384, 65536};
    for (int chunk : chunks)
        for (int grid : grids)
            for (int inflight_kb : {64, 128, 160, 192, 224}) {
                const int stages = inflight_kb * 1024 / chunk;
                if (stages < 1 || stages > 16) continue;
                const size_t per_cta = (total / 148) / chunk * chunk;
                const int n_chunks = (int)(per_cta / chunk);
                float best = 1e30f;
                for (int rep = 0; rep < 3; ++rep) {
                    CK(cudaEventRecord(e0));
                    bulk_kernel<<<grid, 32, (size_t)stages * chunk>>>(d, per_cta, chunk, stages, n_chunks);
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0, e1));
                    if (ms < best) best = ms;
                }
                CK(cudaGetLastError());
                const double bytes = (double)grid * n_chunks * chunk;
                const double tbs = bytes / (best * 1e-3) / 1e12;
                printf("chunk %6d  CTAs %3d  in flight %3d KB (%2d stages): %6.3f TB/s total, %6.1f GB/s per SM\n",
                       chunk, grid, inflight_kb, stages, tbs, 1e3 * tbs / grid);
                if (f) {
                    fprintf(f, "%s {\"chunk\": %d, \"ctas\": %d, \"in_flight_kb\": %d, \"tb_s\": %.4f, \"gb_s_per_sm\": %.2f}",
                            first ? "" : ",\n", chunk, grid, inflight_kb, tbs, 1e3 * tbs / grid);
                    first = false;
                }
            }
    if (f) {
        fprintf(f, "\n]\n");
        fclose(f);
    }
    return 0;
}
