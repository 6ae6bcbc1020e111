// cg_kernels.cuh -- masked conjugate-gradient refit on the GPU
// (cg_solve_operator / cg_solve, cdp.cpp:66-105; gather/scatter and
// cdp_minimize, cdp.cpp:109-139).
//
// Every trajectory (b, q) solves G_act x = b_act on its own support.  The
// contraction G*p is the shared EPI_MATVEC launch of the step kernels (one
// pass over each instance's gram serves all NR replicas; p is zero off the
// support, so the canonical order gives the oracle's sub_apply bitwise).
// The per-trajectory vector work and the two dot products run in one CTA per
// trajectory.  Dot products are summed strictly left to right over the
// active indices (the oracle's seq_dot restatement of Eigen's dot): the
// products are staged in shared memory by the CTA and one thread adds them.
//
// The CG state (x, r, p, Gp) is fp64 in both context precisions: the fp32
// path computes G*p on the tensor cores and keeps the recursion in fp64.
#pragma once

#include "kernels.cuh"

namespace cimcs {

struct CgTraj {
    double rs, stop;
    int it, done, k, breakdown;
};

constexpr int kCgThreads = 256;
constexpr int kCgChunk = 2048;  // staged products per sequential pass

// s = 0; s = s + prod(c) for c = 0 .. k-1, in order; result in every thread.
template <typename F>
__device__ double cg_seq_dot(int k, F prod, double* stage) {
    __shared__ double s_res;
    double s = 0.0;
    for (int c0 = 0; c0 < k; c0 += kCgChunk) {
        const int n = min(kCgChunk, k - c0);
        for (int t = threadIdx.x; t < n; t += blockDim.x) stage[t] = prod(c0 + t);
        __syncthreads();
        if (threadIdx.x == 0)
            for (int t = 0; t < n; ++t) s = s + stage[t];
        __syncthreads();
    }
    if (threadIdx.x == 0) s_res = s;
    __syncthreads();
    const double r = s_res;
    __syncthreads();
    return r;
}

// Ordered compaction of the active indices of trajectory (b, q) into act[0..k).
template <int NR>
__device__ int cg_active_list(const int8_t* sig, int b, int q, int N, int ldN, int* act) {
    __shared__ int s_warp[kCgThreads / 32];
    __shared__ int s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int base = 0; base < N; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const bool on = i < N && sig[((size_t)b * ldN + i) * NR + q] != 0;
        const unsigned m = __ballot_sync(0xffffffffu, on);
        if (lane == 0) s_warp[warp] = __popc(m);
        __syncthreads();
        int off = s_base;
        for (int w = 0; w < warp; ++w) off += s_warp[w];
        if (on) act[off + __popc(m & ((1u << lane) - 1u))] = i;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < kCgThreads / 32; ++w) tot += s_warp[w];
            s_base += tot;
        }
        __syncthreads();
    }
    return s_base;
}

struct CgArgs {
    const void* Rs;         // [B][ldN][NR] context precision
    const int8_t* sig;
    const void* hz;         // [B][ldN]
    double* X;              // [B][ldN][NR]
    double* Rr;
    double* P;
    double* Gp;             // EPI_MATVEC output
    int* act;               // [B*NR][ldN]
    CgTraj* st;             // [B*NR]
    const int* fail_gstep;  // frozen (diverged) trajectories are skipped
    void* W;                // contraction input (tc layout when tc)
    int* n_live;            // trajectories still iterating after this launch
    int tc, ldJ, N, ldN, max_iters;
    double tol;
};

// r = b - G x0 (Gp holds G x0), p = r, rs = |r|^2, stop = tol*|b| (or tol).
template <typename T, int NR>
__global__ void __launch_bounds__(kCgThreads) cg_init_kernel(CgArgs a) {
    __shared__ double stage[kCgChunk];
    const int traj = blockIdx.x, b = traj / NR, q = traj % NR;
    int* act = a.act + (size_t)traj * a.ldN;
    const int k = cg_active_list<NR>(a.sig, b, q, a.N, a.ldN, act);
    const T* Rs = static_cast<const T*>(a.Rs);
    const T* hz = static_cast<const T*>(a.hz);
    auto vi = [&](int c) { return ((size_t)b * a.ldN + act[c]) * NR + q; };
    auto bv = [&](int c) { return (double)hz[(size_t)b * a.ldN + act[c]]; };
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const size_t v = vi(c);
        a.X[v] = (double)Rs[v];
        const double r = bv(c) - a.Gp[v];
        a.Rr[v] = r;
        a.P[v] = r;
        put_w<T>(static_cast<T*>(a.W), a.tc, a.ldN, a.ldJ, NR, b, act[c], q, (T)r);
    }
    __syncthreads();
    const double rs = cg_seq_dot(k, [&](int c) { const double r = a.Rr[vi(c)]; return r * r; },
                                 stage);
    const double bb = cg_seq_dot(k, [&](int c) { const double x = bv(c); return x * x; }, stage);
    if (threadIdx.x == 0) {
        const double bnorm = sqrt(bb);
        const double stop = a.tol * (bnorm > 0.0 ? bnorm : 1.0);
        const bool frozen = a.fail_gstep[traj] != kFreeTraj;
        const int done = frozen || k == 0 || !(0 < a.max_iters && sqrt(rs) > stop);
        a.st[traj] = CgTraj{rs, stop, 0, done, frozen ? 0 : k, 0};
        if (!done) atomicAdd(a.n_live, 1);
    }
}

// One CG iteration of every live trajectory (Gp = G p from EPI_MATVEC).
template <typename T, int NR>
__global__ void __launch_bounds__(kCgThreads) cg_iter_kernel(CgArgs a) {
    __shared__ double stage[kCgChunk];
    const int traj = blockIdx.x, b = traj / NR, q = traj % NR;
    const CgTraj s = a.st[traj];
    if (s.done) return;
    const int k = s.k;
    const int* act = a.act + (size_t)traj * a.ldN;
    auto vi = [&](int c) { return ((size_t)b * a.ldN + act[c]) * NR + q; };
    const double curv =
        cg_seq_dot(k, [&](int c) { const size_t v = vi(c); return a.P[v] * a.Gp[v]; }, stage);
    if (!(curv > 0.0)) {
        if (threadIdx.x == 0) {
            a.st[traj].done = 1;
            a.st[traj].breakdown = 1;
        }
        return;
    }
    const double alpha = s.rs / curv;
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const size_t v = vi(c);
        a.X[v] = a.X[v] + alpha * a.P[v];
        a.Rr[v] = a.Rr[v] - alpha * a.Gp[v];
    }
    __syncthreads();
    const double rs_new =
        cg_seq_dot(k, [&](int c) { const double r = a.Rr[vi(c)]; return r * r; }, stage);
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const size_t v = vi(c);
        const double p = a.Rr[v] + (rs_new / s.rs) * a.P[v];
        a.P[v] = p;
        put_w<T>(static_cast<T*>(a.W), a.tc, a.ldN, a.ldJ, NR, b, act[c], q, (T)p);
    }
    if (threadIdx.x == 0) {
        const int it = s.it + 1;
        const int done = !(it < a.max_iters && sqrt(rs_new) > s.stop);
        a.st[traj] = CgTraj{rs_new, s.stop, it, done, k, 0};
        if (!done) atomicAdd(a.n_live, 1);
    }
}

// Loop condition: continue while any trajectory is live.
__global__ void cg_cond_kernel(int* n_live, int* live_out, cudaGraphConditionalHandle h,
                               int use_handle) {
    const int v = *n_live;
    *live_out = v;
    *n_live = 0;
    if (use_handle) cudaGraphSetConditional(h, v > 0 ? 1u : 0u);
}

// scatter_solution (cdp.cpp:109-114): R[active] = x; inactive entries untouched.
template <typename T, int NR>
__global__ void __launch_bounds__(kCgThreads) cg_final_kernel(CgArgs a) {
    const int traj = blockIdx.x, b = traj / NR, q = traj % NR;
    const int k = a.st[traj].k;
    const int* act = a.act + (size_t)traj * a.ldN;
    T* Rs = static_cast<T*>(const_cast<void*>(a.Rs));
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const size_t v = ((size_t)b * a.ldN + act[c]) * NR + q;
        Rs[v] = (T)a.X[v];
    }
}

}  // namespace cimcs
