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
//    double-buffered; after its Euler update a CTA pushes its 32 new w rows
//    into all peers' next buffer through distributed shared memory
//    (st.shared::cluster), and one cluster barrier per step publishes them;
//  * c, e (or R for Jacobi), D, hz and the replica's state stay in registers;
//    HBM is touched only at the start and end of the call.
//
// Per step the bound is the 63-deep dependent DFMA/FFMA chain + one cluster
// barrier.
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

template <typename T, int NR>
__host__ __device__ constexpr size_t cluster_smem_bytes() {
    return 2 * (size_t)kClMaxN * NR * sizeof(T);
}

// MODE: EPI_STEP_BN / EPI_STEP_CN (n_iters Euler steps, a.step = first step)
//       EPI_JACOBI (n_iters damped Jacobi sweeps on the support a.sigma)
template <typename T, int NR, int MODE>
__global__ void __launch_bounds__(kClThreads, 1)
    cluster_loop_kernel(GemvArgs a, int nRB, int nch, int n_iters) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sW = reinterpret_cast<T*>(smem_raw);  // [2][kClMaxN][NR]
    __shared__ int s_fail[2][NR];

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

    // ---- G slice -> registers (panels [B][nRB][ldJ][RB], or the tcgen05
    // canonical tiles of an fp32 tensor-core context), column j of row i
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
                    v = a.tc_in ? G[tc_gofs(nRB, nch, b, i, j)] : G[pan + (size_t)j * kRB];
                gv[m][jj] = v;
            }
    }
    // ---- w_0 -> buffer 0; buffer 1 zero (entries beyond N stay zero)
    const T* Win = static_cast<const T*>(a.Win);
    for (int k = threadIdx.x; k < 2 * kClMaxN * NR; k += kClThreads) {
        const int j = k / NR, q = k % NR;  // j >= kClMaxN: buffer 1
        T v = T(0);
        if (j < N)
            v = a.tc_in ? Win[tc_wofs(a.ldJ, NR, b, j, q)] : Win[((size_t)b * ldN + j) * NR + q];
        sW[k] = v;
    }
    if (threadIdx.x < 2 * NR) (&s_fail[0][0])[threadIdx.x] = 0;

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
    cluster.sync();  // every CTA initialised before any remote store

    for (int it = 0; it < n_iters; ++it) {
        const int cur = it & 1;
        const T* Wc = sW + (size_t)cur * kClMaxN * NR;
        // frozen flags raised by any CTA during the previous step
        if (q_lane) {
#pragma unroll
            for (int u = 0; u < QPL; ++u) frozen[u] |= s_fail[cur][seg + kSeg * u] != 0;
        }
        // ---- segment chain: acc[q] = fma(G[i][j], w[j][q], acc[q]) over this segment
        T acc[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) acc[q] = T(0);
#pragma unroll
        for (int m = 0; m < kClKG; ++m) {
            const int j0 = (seg + kSeg * m) * kGran;
            if (j0 < N) {
#pragma unroll
                for (int jj = 0; jj < kGran; ++jj) {
                    const T* wp = Wc + (size_t)(j0 + jj) * NR;
#pragma unroll
                    for (int q = 0; q < NR; ++q) acc[q] = fma_<T>(gv[m][jj], wp[q], acc[q]);
                }
            }
        }
        // ---- segment partials added left to right (every lane of the row group)
        T gw[NR];
        const int base = lane & ~7;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
            T s = __shfl_sync(0xffffffffu, acc[q], base);
#pragma unroll
            for (int w = 1; w < kSeg; ++w) s = s + __shfl_sync(0xffffffffu, acc[q], base + w);
            gw[q] = s;
        }
        __syncthreads();  // flags of `cur` read by everyone before they are cleared
        if (threadIdx.x < NR) s_fail[cur][threadIdx.x] = 0;

        // ---- fused update of (row i, replicas owned by this lane)
        T wn[QPL];
        bool wr[QPL];
#pragma unroll
        for (int u = 0; u < QPL; ++u) {
            wr[u] = false;
            const int q = seg + kSeg * u;
            if (!row_ok || !q_lane || frozen[u]) continue;
            T g_q = gw[0];
#pragma unroll
            for (int qq = 1; qq < NR; ++qq)
                if (qq == q) g_q = gw[qq];
            if constexpr (MODE == EPI_JACOBI) {
                T rn = st_R[u];
                if (st_on[u]) {
                    if (Dv == T(0)) {
                        atomicMin(a.err, i);
                        continue;
                    }
                    const T off = g_q - Dv * st_R[u];
                    rn = omd * st_R[u] + dtc * ((hzv - off) / Dv);
                    st_R[u] = rn;
                }
                wn[u] = rn * (st_on[u] ? T(1) : T(0));
                wr[u] = true;
            } else {
                const double pd = a.pump ? a.pump[a.step + it] : a.p_scalar;
                const T loss = sc.minus_j != 0.0 ? (T)((-1.0 + pd) - sc.minus_j) : (T)(-1.0 + pd);
                const T c = st_c[u], e = st_e[u];
                const T wv = Wc[(size_t)i * NR + q];
                const T Jw = Dv * wv - g_q;  // apply_coupling: gram_diag∘w - G w
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
                    atomicMin(&a.fail_gstep[traj], a.alt->gstep_base + a.step + it);
                    atomicMin(&a.fail_idx[traj], i);
                    // freeze this replica in every CTA from the next step on
                    for (int r = 0; r < cs; ++r)
                        *cluster.map_shared_rank(&s_fail[cur ^ 1][q], r) = 1;
                    continue;
                }
                st_c[u] = cn;
                st_e[u] = en;
                if constexpr (MODE == EPI_STEP_BN)
                    wn[u] = st_R[u] * (cn > T(0) ? T(1) : T(0));
                else
                    wn[u] = (st_R[u] * T(0.25)) * (cn + rt);
                wr[u] = true;
                lmin[u] = en < lmin[u] ? en : lmin[u];
            }
        }
        // ---- publish w_{it+1}: own rows into every CTA's next buffer
        T* Wn = sW + (size_t)(cur ^ 1) * kClMaxN * NR;
#pragma unroll
        for (int u = 0; u < QPL; ++u) {
            const int q = seg + kSeg * u;
            if (!row_ok || !q_lane) continue;
            // frozen / failed entries keep the buffer's previous-step value
            const T v = wr[u] ? wn[u] : Wc[(size_t)i * NR + q];
            for (int r = 0; r < cs; ++r) *cluster.map_shared_rank(&Wn[(size_t)i * NR + q], r) = v;
        }
        cluster.sync();
    }

    // ---- write back state, final w and the min of e
    const T* Wf = sW + (size_t)(n_iters & 1) * kClMaxN * NR;
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
        const T v = Wf[(size_t)i * NR + q];
        if (a.tc_in) {
            Wout[tc_wofs(a.ldJ, NR, b, i, q)] = v;
            Wout[tc_wofs(a.ldJ, NR, b, i, NR + q)] = (T)((float)v - trunc_tf32((float)v));
        } else {
            Wout[vi] = v;
        }
    }
}

}  // namespace cimcs
