// cluster_kernels.cuh -- whole CIM call / whole Jacobi refit in ONE launch for
// small instances (N <= 512): BASELINE config 0 and other latency-bound sizes.
//
// The grid kernels (kernels.cuh / tc_kernels.cuh) stream G from HBM once per
// Euler step; at N = 500 a step moves 2 MB and is bound by launch + grid
// synchronisation latency (~4 us/step), not by bytes.  Here one thread-block
// cluster (one CTA per 32 spin rows, <= 16 CTAs, non-portable size) owns one
// instance for the whole call:
//
//  * thread (row, seg) holds its canonical-order slice of G in REGISTERS for
//    all steps: row i, granules g = seg + 8m (m < 8), i.e. the exact fma chain
//    "segment seg" of the documented G*v order (8 segments of 8-wide
//    granules), so the result is bitwise the grid kernel's;
//  * the contraction input w (N x NR) lives in every CTA's shared memory,
//    double-buffered.  After its Euler update a CTA pushes its 32-row slice
//    of the next w (plus one failure flag per replica) into every CTA of the
//    cluster with st.async (16-byte DSMEM stores that complete_tx on the
//    receiver's mbarrier).  A CTA starts step k+1 as soon as its own
//    mbarrier says all of w_{k+1} has landed -- no cluster-wide barrier, no
//    fence, no L1 invalidation per step;
//  * c, e (or R for Jacobi), D, hz stay in registers and the pump table in
//    shared memory; HBM is touched only at the start and end of the call.
//
// Buffer reuse is safe without a barrier: a CTA overwrites a peer's buffer
// (k & 1) with w_{k+2} only after it has received w_{k+1} from that peer,
// which the peer pushes after its step-k contraction has finished reading
// buffer (k & 1).  Per step the bound is the 63-deep dependent FMA chain +
// one DSMEM round trip.
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"
#include "tc_kernels.cuh"

namespace cimcs {

namespace cgx = cooperative_groups;

constexpr int kClRows = 32;                  // spin rows per CTA
constexpr int kClThreads = kClRows * kSeg;   // one thread per (row, segment)
constexpr int kClMaxN = 512;
constexpr int kClMaxCta = 16;                // non-portable cluster size
constexpr int kClKG = kClMaxN / (kSeg * kGran);  // granules per segment = 8
constexpr int kClPump = 2048;                // pump entries staged in smem

// w buffers are stored by 8-row granule with a 16-byte pad after each granule:
// the 8 threads of a quarter-warp read the same chunk of 8 different granules
// (g = seg + 8m), and an odd granule stride in 16-byte units puts those 8
// chunks in 8 different bank groups (no shared-memory conflict).
template <typename T, int NR>
struct ClW {
    static constexpr int gran = kGran * NR;                 // elements per granule
    static constexpr int stride = gran + 16 / (int)sizeof(T);  // padded
    static constexpr int buf = (kClMaxN / kGran) * stride;  // elements per buffer
    __device__ static constexpr int at(int j, int q) { return (j / kGran) * stride + (j % kGran) * NR + q; }
};

// dynamic smem: W[2][padded] | stage[kClRows][NR] | flags[2][kClMaxCta][NR] int
//               | pump[kClPump] double | mbar[2]
template <typename T, int NR>
struct ClSmem {
    static constexpr size_t w = 0;
    static constexpr size_t stage = w + 2 * (size_t)ClW<T, NR>::buf * sizeof(T);
    static constexpr size_t flags = stage + (size_t)kClRows * NR * sizeof(T);
    static constexpr size_t pump = (flags + 2 * (size_t)kClMaxCta * NR * 4 + 15) / 16 * 16;
    static constexpr size_t mbar = pump + (size_t)kClPump * 8;
    static constexpr size_t bytes = mbar + 2 * 8;
};

template <typename T, int NR>
__host__ __device__ constexpr size_t cluster_smem_bytes() {
    return ClSmem<T, NR>::bytes;
}

__device__ __forceinline__ uint32_t cl_mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_st_async16(uint32_t raddr, uint64_t lo, uint64_t hi,
                                              uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(
            raddr),
        "l"(lo), "l"(hi), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void cl_st_async8(uint32_t raddr, uint64_t v, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
        "l"(v), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void cl_st_async4(uint32_t raddr, uint32_t v, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
        "r"(v), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void cl_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "CLW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra CLW_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// MODE: EPI_STEP_BN / EPI_STEP_CN (n_iters Euler steps, a.step = first step)
//       EPI_JACOBI (n_iters damped Jacobi sweeps on the support a.sigma)
template <typename T, int NR, int MODE>
__global__ void __launch_bounds__(kClThreads, 1)
    cluster_loop_kernel(GemvArgs a, int nRB, int nch, int n_iters) {
    using L = ClSmem<T, NR>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using WL = ClW<T, NR>;
    T* sW = reinterpret_cast<T*>(smem_raw + L::w);              // [2][WL::buf]
    T* sStage = reinterpret_cast<T*>(smem_raw + L::stage);      // [kClRows][NR]
    int* sFlags = reinterpret_cast<int*>(smem_raw + L::flags);  // [2][kClMaxCta][NR]
    double* sPump = reinterpret_cast<double*>(smem_raw + L::pump);
    uint64_t* sBar = reinterpret_cast<uint64_t*>(smem_raw + L::mbar);
    __shared__ int s_failed[2][NR];  // this CTA's failures, by step parity

    cgx::cluster_group cluster = cgx::this_cluster();
    const int cs = (int)cluster.num_blocks();
    const int cr = (int)cluster.block_rank();
    const int b = blockIdx.x / cs;
    const int N = a.N, ldN = a.ldN;
    const int lane = threadIdx.x & 31;
    const int row_l = threadIdx.x >> 3, seg = threadIdx.x & 7;
    const int i = cr * kClRows + row_l;  // global spin row of this thread
    const bool row_ok = i < N;
    constexpr int kRB = row_block<T>();
    constexpr uint32_t kSlice = kClRows * NR * sizeof(T);  // bytes pushed per CTA
    const uint32_t fill_bytes = (uint32_t)cs * (kSlice + NR * 4);

    // ---- G slice -> registers (panels [B][nRB][ldJ][RB]), column j of row i
    T gv[kClKG][kGran];
    {
        const T* G = static_cast<const T*>(a.G);
        const size_t pan = ((size_t)b * nRB + i / kRB) * (size_t)a.ldJ * kRB + (i % kRB);
#pragma unroll
        for (int m = 0; m < kClKG; ++m)
#pragma unroll
            for (int jj = 0; jj < kGran; ++jj) {
                const int j = (seg + kSeg * m) * kGran + jj;
                T v = T(0);
                if (row_ok && j < N)
                    v = G[pan + (size_t)j * kRB];
                gv[m][jj] = v;
            }
    }
    // ---- w_0 -> buffer 0; buffer 1 zero; flags zero; pump table
    const T* Win = static_cast<const T*>(a.Win);
    for (int k = threadIdx.x; k < 2 * WL::buf; k += kClThreads) sW[k] = T(0);
    __syncthreads();
    for (int k = threadIdx.x; k < N * NR; k += kClThreads) {
        const int j = k / NR, q = k % NR;
        sW[WL::at(j, q)] = Win[((size_t)b * ldN + j) * NR + q];
    }
    for (int k = threadIdx.x; k < 2 * kClMaxCta * NR; k += kClThreads) sFlags[k] = 0;
    if constexpr (MODE != EPI_JACOBI) {
        const int np = n_iters < kClPump ? n_iters : kClPump;
        for (int k = threadIdx.x; k < np; k += kClThreads)
            sPump[k] = a.pump ? a.pump[a.step + k] : a.p_scalar;
    }
    if (threadIdx.x < 2 * NR) (&s_failed[0][0])[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&sBar[0], 1);
        mbar_init(&sBar[1], 1);
        mbar_fence_init();
        if (n_iters >= 1) mbar_arrive_expect_tx(&sBar[1], fill_bytes);  // w_1
        if (n_iters >= 2) mbar_arrive_expect_tx(&sBar[0], fill_bytes);  // w_2
    }

    // ---- per-(row, replica) state in registers: lane seg owns replicas q = seg (+8)
    constexpr int QPL = NR > kSeg ? NR / kSeg : 1;  // replicas per lane
    const bool q_lane = seg < NR;
    T st_c[QPL], st_e[QPL], st_R[QPL];
    bool st_on[QPL];
    T Dv = T(0), hzv = T(0);
    if (row_ok) {
        Dv = static_cast<const T*>(a.D)[(size_t)b * ldN + i];
        hzv = static_cast<const T*>(a.hz)[(size_t)b * ldN + i];
    }
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
        const int q = seg + kSeg * u;
        const size_t vi = ((size_t)b * ldN + i) * NR + q;
        st_c[u] = st_e[u] = st_R[u] = T(0);
        st_on[u] = false;
        if (row_ok && q_lane) {
            st_R[u] = static_cast<const T*>(a.Rs)[vi];
            if constexpr (MODE == EPI_JACOBI) {
                st_on[u] = a.sigma[vi] != 0;
            } else {
                st_c[u] = static_cast<const T*>(a.C)[vi];
                st_e[u] = static_cast<const T*>(a.E)[vi];
            }
        }
    }
    bool frozen[QPL];
    T lmin[QPL];
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
        const int q = seg + kSeg * u;
        lmin[u] = T(INFINITY);
        frozen[u] = true;
        if (q_lane) {
            const int g = a.fail_gstep[b * NR + q];
            if constexpr (MODE == EPI_JACOBI)
                frozen[u] = g != kFreeTraj;
            else
                frozen[u] = g < a.alt->gstep_base + a.step;
        }
    }
    const StepScalars& sc = a.s;
    const T half_rt = (T)sc.half_rt, rt = (T)sc.rt, dt = (T)sc.dt, Kj = (T)sc.Kj;
    const T nbeta = (T)sc.nbeta, tau = (T)sc.tau;
    const T thresh = (MODE == EPI_JACOBI) ? T(0) : (T)a.alt->thresh;
    const T omd = (T)sc.one_minus_dtc, dtc = (T)sc.dt_c;
    const int gstep0 = (MODE == EPI_JACOBI) ? 0 : a.alt->gstep_base + a.step;
    const uint32_t w_base = smem_u32(sW), f_base = smem_u32(sFlags), bar_base = smem_u32(sBar);
    cluster.sync();  // mbarriers initialised and armed everywhere before any push

    for (int it = 0; it < n_iters; ++it) {
        const int cur = it & 1, nxt = cur ^ 1;
        if (it > 0) {
            cl_wait(&sBar[cur], ((it - 1) >> 1) & 1);  // w_it and its flags have landed
            if (threadIdx.x == 0 && it + 2 <= n_iters)
                mbar_arrive_expect_tx(&sBar[cur], fill_bytes);  // w_{it+2}
            if (q_lane) {  // replicas that failed anywhere in the previous step freeze now
#pragma unroll
                for (int u = 0; u < QPL; ++u) {
                    const int q = seg + kSeg * u;
                    int f = 0;
                    for (int r = 0; r < cs; ++r) f |= sFlags[(cur * kClMaxCta + r) * NR + q];
                    frozen[u] |= f != 0;
                }
            }
        }
        const T* Wc = sW + (size_t)cur * WL::buf;
        // ---- segment chain: acc[q] = fma(G[i][j], w[j][q], acc[q]); the w granule
        // of step m+1 is loaded while m's fmas issue.  Past N both G and w are 0
        // and fma(0, 0, acc) == acc exactly (acc is never -0), so the chain is
        // the grid kernel's.
        T acc[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) acc[q] = T(0);
        T wv[kGran][NR], wx[kGran][NR];
#pragma unroll
        for (int jj = 0; jj < kGran; ++jj)
#pragma unroll
            for (int q = 0; q < NR; ++q) wv[jj][q] = Wc[WL::at(seg * kGran + jj, q)];
#pragma unroll
        for (int m = 0; m < kClKG; ++m) {
            if (m * kSeg * kGran >= N) break;  // warp-uniform
            if (m + 1 < kClKG) {
#pragma unroll
                for (int jj = 0; jj < kGran; ++jj)
#pragma unroll
                    for (int q = 0; q < NR; ++q)
                        wx[jj][q] = Wc[WL::at((seg + kSeg * (m + 1)) * kGran + jj, q)];
            }
#pragma unroll
            for (int jj = 0; jj < kGran; ++jj)
#pragma unroll
                for (int q = 0; q < NR; ++q) acc[q] = fma_<T>(gv[m][jj], wv[jj][q], acc[q]);
#pragma unroll
            for (int jj = 0; jj < kGran; ++jj)
#pragma unroll
                for (int q = 0; q < NR; ++q) wv[jj][q] = wx[jj][q];
        }
        // ---- segment partials added left to right (every lane of the row group)
        T gw[NR];
        const int base = lane & ~7;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
            T p[kSeg];
#pragma unroll
            for (int w = 0; w < kSeg; ++w) p[w] = __shfl_sync(0xffffffffu, acc[q], base + w);
            T s = p[0];
#pragma unroll
            for (int w = 1; w < kSeg; ++w) s = s + p[w];
            gw[q] = s;
        }

        // ---- fused update of (row i, replicas owned by this lane) -> stage
#pragma unroll
        for (int u = 0; u < QPL; ++u) {
            const int q = seg + kSeg * u;
            if (!q_lane) continue;
            const T wold = row_ok ? Wc[WL::at(i, q)] : T(0);
            T wn = wold;  // frozen / failed entries keep the previous value
            if (row_ok && !frozen[u]) {
                T g_q = gw[0];
#pragma unroll
                for (int qq = 1; qq < NR; ++qq)
                    if (qq == q) g_q = gw[qq];
                if constexpr (MODE == EPI_JACOBI) {
                    T rn = st_R[u];
                    bool okd = true;
                    if (st_on[u]) {
                        if (Dv == T(0)) {
                            atomicMin(a.err, i);
                            okd = false;
                        } else {
                            const T off = g_q - Dv * st_R[u];
                            rn = omd * st_R[u] + dtc * ((hzv - off) / Dv);
                            st_R[u] = rn;
                        }
                    }
                    if (okd) wn = rn * (st_on[u] ? T(1) : T(0));
                } else {
                    const double pd = it < kClPump ? sPump[it]
                                                   : (a.pump ? a.pump[a.step + it] : a.p_scalar);
                    const T loss =
                        sc.minus_j != 0.0 ? (T)((-1.0 + pd) - sc.minus_j) : (T)(-1.0 + pd);
                    const T c = st_c[u], e = st_e[u];
                    const T Jw = Dv * wold - g_q;  // apply_coupling: gram_diag∘w - G w
                    T h;
                    if constexpr (MODE == EPI_STEP_BN)
                        h = half_rt * (Jw + hzv);
                    else
                        h = Jw + half_rt * hzv;
                    const T inj = (Kj * e) * (st_R[u] * h - thresh);
                    const T cn = c + dt * ((loss - c * c) * c + inj);
                    const T en = e + dt * ((nbeta * (c * c - tau)) * e);
                    if (!finite_(cn) || !finite_(en)) {
                        const int traj = b * NR + q;
                        atomicMin(&a.fail_gstep[traj], gstep0 + it);
                        atomicMin(&a.fail_idx[traj], i);
                        s_failed[cur][q] = 1;
                    } else {
                        st_c[u] = cn;
                        st_e[u] = en;
                        if constexpr (MODE == EPI_STEP_BN)
                            wn = st_R[u] * (cn > T(0) ? T(1) : T(0));
                        else
                            wn = (st_R[u] * T(0.25)) * (cn + rt);
                        lmin[u] = en < lmin[u] ? en : lmin[u];
                    }
                }
            }
            sStage[row_l * NR + q] = wn;
        }
        __syncthreads();  // slice + failure flags staged
        // flags of the previous step were pushed before its closing barrier
        if (threadIdx.x < NR) s_failed[nxt][threadIdx.x] = 0;

        // ---- push w_{it+1} slice (16-byte st.async) and flags to every CTA
        {
            constexpr int nch16 = (int)(kSlice / 16);
            constexpr int cpg = WL::gran * (int)sizeof(T) / 16;  // 16-byte chunks per granule
            const uint32_t wdst = w_base + (uint32_t)((nxt * WL::buf +
                                                       cr * (kClRows / kGran) * WL::stride) *
                                                      sizeof(T));
            const uint32_t fdst = f_base + (uint32_t)((nxt * kClMaxCta + cr) * NR * 4);
            const uint32_t bar = bar_base + nxt * 8;
            for (int k = threadIdx.x; k < cs * nch16; k += kClThreads) {
                const int r = k / nch16, ch = k % nch16;
                const uint64_t* src = reinterpret_cast<const uint64_t*>(sStage) + 2 * ch;
                const uint32_t off = (uint32_t)((ch / cpg) * WL::stride * sizeof(T) + (ch % cpg) * 16);
                cl_st_async16(cl_mapa(wdst + off, r), src[0], src[1], cl_mapa(bar, r));
            }
            for (int k = threadIdx.x; k < cs * NR; k += kClThreads) {
                const int r = k / NR, q = k % NR;
                cl_st_async4(cl_mapa(fdst + q * 4, r), (uint32_t)s_failed[cur][q], cl_mapa(bar, r));
            }
        }
        __syncthreads();  // stage / flags consumed before the next step rewrites them
    }
    if (n_iters > 0) cl_wait(&sBar[n_iters & 1], ((n_iters - 1) >> 1) & 1);

    // ---- write back state, final w and the min of e
    const T* Wf = sW + (size_t)(n_iters & 1) * WL::buf;
    T* Wout = static_cast<T*>(a.Wout);
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
        const int q = seg + kSeg * u;
        if (!row_ok || !q_lane) continue;
        const size_t vi = ((size_t)b * ldN + i) * NR + q;
        if constexpr (MODE == EPI_JACOBI) {
            static_cast<T*>(a.Rs)[vi] = st_R[u];
        } else {
            static_cast<T*>(a.C)[vi] = st_c[u];
            static_cast<T*>(a.E)[vi] = st_e[u];
            if (lmin[u] != T(INFINITY)) atomicMin(&a.minE[b * NR + q], ord_key(lmin[u]));
        }
        const T v = Wf[WL::at(i, q)];
        Wout[vi] = v;
    }
    cluster.sync();  // no CTA leaves while a peer may still address its shared memory
}

}  // namespace cimcs
