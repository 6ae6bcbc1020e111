// rt_aux_kernels.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): small kernels of the host runtime: trajectory layout conversion,
// score finalisation, median e, best-state tracking.
#pragma once

namespace {

thread_local std::string g_err;

struct Status {
    int code;
};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            return fail(CIMCS_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int pow2_slots(int R) {
    int n = 1;
    while (n < R) n <<= 1;
    return n;
}

// ------------------------------------------------------------- aux kernels
template <typename T, int NR>
__global__ void traj_to_dev(const double* __restrict__ h, T* __restrict__ d, int Rreal, int N,
                            int ldN, int B, T pad) {
    const size_t total = (size_t)B * ldN * NR;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const int q = k % NR;
        const size_t bi = k / NR;
        const int i = bi % ldN;
        const int b = bi / ldN;
        d[k] = (i < N && q < Rreal) ? (T)h[((size_t)b * Rreal + q) * N + i] : pad;
    }
}

template <typename T, int NR>
__global__ void dev_to_traj(const T* __restrict__ d, double* __restrict__ h, int Rreal, int N,
                            int ldN, int B) {
    const size_t total = (size_t)B * Rreal * N;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const int i = k % N;
        const size_t bq = k / N;
        const int q = bq % Rreal;
        const int b = bq / Rreal;
        h[k] = (double)d[((size_t)b * ldN + i) * NR + q];
    }
}

template <int NR>
__global__ void sig_to_dev(const int32_t* __restrict__ h, int8_t* d, int Rreal, int N, int ldN,
                           int B) {
    const size_t total = (size_t)B * ldN * NR;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const int q = k % NR;
        const size_t bi = k / NR;
        const int i = bi % ldN;
        const int b = bi / ldN;
        d[k] = (i < N && q < Rreal) ? (int8_t)h[((size_t)b * Rreal + q) * N + i] : (int8_t)0;
    }
}

template <int NR>
__global__ void sig_to_traj(const int8_t* __restrict__ d, int32_t* h, int Rreal, int N, int ldN,
                            int B) {
    const size_t total = (size_t)B * Rreal * N;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const int i = k % N;
        const size_t bq = k / N;
        const int q = bq % Rreal;
        const int b = bq / Rreal;
        h[k] = d[((size_t)b * ldN + i) * NR + q];
    }
}

// R_init = hz (default_r_init, orchestrator.cpp:138) for every replica
template <typename T, int NR>
__global__ void rinit_hz_kernel(const T* __restrict__ hz, T* Rs, int Rreal, int N, int ldN,
                                int B) {
    const size_t total = (size_t)B * ldN * NR;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const int q = k % NR;
        const size_t bi = k / NR;
        const int i = bi % ldN;
        Rs[k] = (i < N && q < Rreal) ? hz[bi] : T(0);
    }
}

template <typename T, int NR>
__global__ void mask_kernel(const T* __restrict__ Rs, const int8_t* __restrict__ sig, T* V,
                            size_t total, int N, int ldN, int ldJ, int tc) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const int q = k % NR;
        const size_t bi = k / NR;
        const int i = bi % ldN;
        const int b = bi / ldN;
        if (i < N) put_w<T>(V, tc, ldN, ldJ, NR, b, i, q, Rs[k] * (sig[k] ? T(1) : T(0)));
        else if (!tc) V[k] = T(0);
    }
}

__global__ void traj_flags_kernel(int* fail_gstep, int* fail_idx, int Rreal, int NR, int B) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= B * NR) return;
    fail_gstep[k] = (k % NR) < Rreal ? kFreeTraj : kInactiveTraj;
    fail_idx[k] = INT_MAX;
}

struct DevRecord {
    int i, support;
    double eta, hamiltonian, rmse, hamming, min_e, median_e;
};

// Per trajectory: combine the score partials of this rank's row blocks (in
// order) and count the support / Hamming mismatches over this rank's rows:
// tp[traj] = {w.Gw, hz.w, sum (w - x xi)^2, |sigma|, hamming}.  Row-sharded
// contexts all-reduce tp across ranks before finalize_kernel.
template <int NR>
__global__ void tp_kernel(const double* __restrict__ part, int nRB,
                          const int8_t* __restrict__ sig, const int8_t* __restrict__ xi,
                          int row0, int row1, int ldN, int has_truth, double* tp) {
    const int traj = blockIdx.x;
    const int b = traj / NR, q = traj % NR;
    __shared__ long long s_sup[256], s_ham[256];
    long long sup = 0, ham = 0;
    for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
        const int s = sig[((size_t)b * ldN + i) * NR + q];
        sup += s;
        if (has_truth) ham += abs(s - (int)xi[(size_t)b * ldN + i]);
    }
    s_sup[threadIdx.x] = sup;
    s_ham[threadIdx.x] = ham;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            s_sup[threadIdx.x] += s_sup[threadIdx.x + w];
            s_ham[threadIdx.x] += s_ham[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    double A = 0.0, Bv = 0.0, Cv = 0.0;
    for (int r = 0; r < nRB; ++r) {
        const double* p = part + (((size_t)b * nRB + r) * NR + q) * 4;
        A = A + p[0];
        Bv = Bv + p[1];
        Cv = Cv + p[2];
    }
    double* o = tp + (size_t)traj * 5;
    o[0] = A;
    o[1] = Bv;
    o[2] = Cv;
    o[3] = (double)s_sup[0];
    o[4] = (double)s_ham[0];
}

// Per trajectory: objective / rmse / hamming, the history record, best tracking.
__global__ void finalize_kernel(const double* __restrict__ tp, int ntraj,
                                const unsigned long long* __restrict__ minE,
                                const int* __restrict__ fail_gstep, const AltParams* alt, int N,
                                int has_truth, DevRecord* hist_alt, int* n_hist,
                                double* best_obj, int* improved, double* obj_out,
                                double* rmse_out, double* ham_out) {
    const int traj = blockIdx.x * blockDim.x + threadIdx.x;
    if (traj >= ntraj) return;
    if (improved) improved[traj] = 0;
    if (fail_gstep[traj] != kFreeTraj) return;
    const double* t = tp + (size_t)traj * 5;
    const double lam = alt->lambda;
    // objective_at: 0.5 w.(G w) - hz.w + lambda |sigma|  (orchestrator.cpp:57-62)
    const double obj = 0.5 * t[0] - t[1] + lam * t[3];
    const double rm = has_truth ? sqrt(t[2] / (double)N) : NAN;
    const double hm = has_truth ? t[4] / (double)N : NAN;
    if (obj_out) obj_out[traj] = obj;
    if (rmse_out) rmse_out[traj] = rm;
    if (ham_out) ham_out[traj] = hm;
    if (hist_alt) {
        DevRecord& rec = hist_alt[traj];
        rec.i = alt->alt;
        rec.support = (int)t[3];
        rec.eta = alt->eta;
        rec.hamiltonian = obj;
        rec.rmse = rm;
        rec.hamming = hm;
        rec.min_e = ord_val(minE[traj]);
        n_hist[traj] += 1;
    }
    if (best_obj && obj < best_obj[traj]) {
        best_obj[traj] = obj;
        improved[traj] = 1;
    }
}

// After the failing step is agreed across ranks (MIN over fail_gstep), only
// ranks that saw that step keep their offending index candidate.
__global__ void fail_fix_kernel(const int* __restrict__ local_gstep, const int* __restrict__ gstep,
                                int* fail_idx, int n) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && local_gstep[k] != gstep[k]) fail_idx[k] = INT_MAX;
}

// median(e_final) (orchestrator.cpp:163-168): bitonic sort in shared memory.
template <typename T, int NR>
__global__ void median_kernel(const T* __restrict__ E, const int* __restrict__ fail_gstep, int N,
                              int ldN, int P, DevRecord* hist_alt) {
    extern __shared__ __align__(16) unsigned char msm[];
    T* v = reinterpret_cast<T*>(msm);
    const int traj = blockIdx.x;
    if (fail_gstep[traj] != kFreeTraj) return;
    const int b = traj / NR, q = traj % NR;
    for (int i = threadIdx.x; i < P; i += blockDim.x)
        v[i] = i < N ? E[((size_t)b * ldN + i) * NR + q] : T(INFINITY);
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const T a = v[i], c = v[l];
                    if ((a > c) == up) {
                        v[i] = c;
                        v[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0)
        hist_alt[traj].median_e = N % 2 == 1 ? (double)v[N / 2]
                                             : 0.5 * ((double)v[N / 2 - 1] + (double)v[N / 2]);
}

template <typename T, int NR>
__global__ void best_update_kernel(const int* __restrict__ improved, const T* __restrict__ Rs,
                                   const int8_t* __restrict__ sig, T* bestR, int8_t* bestS, int ldN,
                                   int B) {
    const size_t total = (size_t)B * ldN * NR;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const int q = k % NR;
        const int b = (int)((k / NR) / ldN);
        if (improved[b * NR + q]) {
            bestR[k] = Rs[k];
            bestS[k] = sig[k];
        }
    }
}

int grid_for(size_t n) {
    size_t g = (n + 255) / 256;
    return (int)std::min<size_t>(std::max<size_t>(g, 1), 148 * 16);
}

}  // namespace
