// runtime.cu -- host runtime + C ABI of libcimcs_gpu.so (see include/cimcs_gpu.h).
//
// The alternation driver restates alternating_minimize
// (orchestrator.cpp:170-235) for B instances x R replicas at once: per
// alternation one CUDA graph runs init -> n_steps fused Euler steps (K2),
// one graph runs the support extraction + damped Jacobi refit (K3), one graph
// runs the scorer (K4).  c0 for the next alternation is drawn on a host
// thread pool from each trajectory's std::mt19937_64 stream while the GPU
// runs the current one.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <queue>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cimcs_gpu.h"
#include "host_rng.hpp"
#include "io.hpp"
#include "kernels.cuh"
#include "tc_kernels.cuh"
#include "cg_kernels.cuh"
#include "cluster_kernels.cuh"
#include "sym_kernels.cuh"
#include "sym64_kernels.cuh"
#include "gram_tc_kernels.cuh"
#include "mri_kernels.cuh"

using namespace cimcs;

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

// ======================================================================= ctx
struct cimcs_ctx {
    int device = 0, dtype = CIMCS_F32;
    cudaStream_t stream = nullptr;
    int host_threads = 0;
    bool use_graphs = true;
    bool use_cluster = true;  // small N: whole CIM call / refit in one cluster launch
    bool want_tc = true;  // fp32 contraction on tcgen05 (3xTF32)
    bool tc_requested = true;  // want_tc when the resident problems were set
    // row sharding (one rank per GPU): this rank owns spin rows [row0, row1)
    int world = 1, rank = 0;
    bool sharded = false;  // created by cimcs_create_sharded (padded row layout)
    ncclComm_t comm = nullptr;
    int row0 = 0, row1 = 0, rb0 = 0;
    double* tp = nullptr;        // per-trajectory score partials [B*NR][5]
    int* fail_tmp = nullptr;     // local fail_gstep before the cross-rank MIN
    bool tc = false;      // active for the current problem set
    bool sym = false;      // active for the current problem set
    // fp64 symmetric-tile path on the DMMA tensor cores (sym64_kernels.cuh):
    // unsharded fp64 contexts with N > kClMaxN (option "sym64", default on)
    bool want_sym64 = true;
    bool sym64 = false;
    int nRB6 = 0, ntri6 = 0, nSB6 = 0;      // its geometry: 64-row blocks, 512 x 512 items
    void* dG6 = nullptr;                    // its gram tiles [B][ntri6][64 x 64] fp64
    double *WT0 = nullptr, *WT1 = nullptr;  // fp64 w tiles of W0 / W1 [B][nRB][64][NR]
    double* dPart6 = nullptr;               // partials [B][nRB][nSB][64][NR]
    int ntri = 0;          // upper-triangle tiles per instance
    int nSB = 0;           // super-block items per row of the tile triangle (kSyS tiles)
    struct SymSched {      // LPT placement of the items of nb instances on the CTAs
        int nb = 0, nRB = 0, S = 0, grid = 0;
        int2* items = nullptr;
        int* sched = nullptr;
    };
    std::vector<SymSched> ssched;
    int* dSg = nullptr;    // per-instance gram scale exponent
    float* dSpart = nullptr;  // partial products [B][nRB][nSB][128][NR]
    bool use_pdl = true;      // programmatic dependent launch between the step kernels
    int gram_l2 = 0;          // gram tiles copied with evict_last (L2 time-blocking experiment)
    bool kernel_timing = false;  // eager mode: CUDA events around each step-mode tile kernel
    cudaEvent_t kt_ev[2] = {nullptr, nullptr};
    // tile sharding of the symmetric path (cimcs_create_sharded contexts, option
    // "tile_shard", default on): every rank keeps the full state and streams only
    // the gram tiles of its super-rows [sP0, sP1); the per-rank slot sums are
    // all-reduced (NCCL) before the replicated update -- one collective per step
    int sh_world = 1, sh_rank = 0;  // geometry given at creation
    bool sh_rows = false;           // created sharded
    int tshard_opt = 1;
    bool tshard = false;            // active for the current problem set
    int tworld = 1, trank = 0, sP0 = 0, sP1 = 0;
    float* dH = nullptr;            // [B][nRB][128][NR] summed partial products
    int gram_tc = 0;          // large-N fp32 gram on tcgen05 (gram_tc_kernels.cuh): 0 auto (N >= 8192), 1, -1
    // matrix-free MRI transform-chain problem (mri_kernels.cuh; mri.hpp:46-99)
    bool mri = false;
    int mH = 0, mW = 0, mL = 0;
    float mgamma = 0.f;
    unsigned char* dMaskBr = nullptr;  // [H*W] sampled, bit-reversed coordinates
    float2* dTw = nullptr;             // [L/2] exp(-2 pi i k / L)
    float* dTarget = nullptr;          // [H*W] target image (row-major)
    bool mri_cluster = true;           // per-step apply on one cluster per replica
    __half *WB0 = nullptr, *WB1 = nullptr;  // fp16 B tiles of W0 / W1 [B][nRB][2NR x 128]
    int *WS0 = nullptr, *WS1 = nullptr;     // their scale exponents [B][nRB][NR]
    size_t spart_elems = 0;
    int nch = 0;
    int num_sms = 148;
    // problems
    int B = 0, N = 0, ldN = 0, Mmax = 0;
    std::vector<int> M;
    bool has_truth = false, built = false;
    double *dA = nullptr, *dy = nullptr;
    int* dM = nullptr;
    void* dG = nullptr;      // gram panels [B][nRB][ldJ][RB] in the path's dtype
    int ldJ = 0, nRB = 0, RB = 0;  // nRB: row blocks held by this rank
    void *dD = nullptr, *dhz = nullptr;
    double* dx = nullptr;
    int8_t* dxi = nullptr;
    // trajectory state (NR slots)
    int NR = 0;
    void *Rs = nullptr, *C = nullptr, *E = nullptr, *W0 = nullptr, *W1 = nullptr,
         *Hdbg = nullptr, *bestR = nullptr;
    int8_t *sig = nullptr, *bestS = nullptr;
    int *fail_gstep = nullptr, *fail_idx = nullptr, *n_hist = nullptr, *improved = nullptr,
        *err = nullptr;
    unsigned long long* minE = nullptr;
    double *part = nullptr, *best_obj = nullptr, *stage = nullptr, *obj = nullptr,
           *rmse = nullptr, *ham = nullptr;
    int32_t* stage_i = nullptr;
    size_t stage_elems = 0;
    AltParams* alt = nullptr;
    // reusable host/device buffers and the instantiated solve graphs
    double* pin = nullptr;        // pinned staging for uploads (2 slots)
    size_t pin_bytes = 0;         // per slot
    double* pin_c0 = nullptr;     // pinned c0 double buffer
    size_t pin_c0_elems = 0;
    double* dc0 = nullptr;        // device c0 of the current alternation
    size_t dc0_elems = 0;
    cudaGraphExec_t g_cim = nullptr, g_refit = nullptr;
    std::vector<long long> graph_key;
    double* pump = nullptr;
    int pump_cap = 0;
    DevRecord* hist = nullptr;
    int hist_cap = 0;
    // Positive-P state (allocated on first use): moments n, m, measured amplitude,
    // unit normals in chunks of kPpChunk steps (device and pinned, double buffered)
    void *Pn = nullptr, *Pm = nullptr, *MT = nullptr;
    double *nzd[2] = {nullptr, nullptr}, *nzh[2] = {nullptr, nullptr};
    size_t nz_elems = 0;
    // conjugate-gradient refit state (allocated on first use)
    double *cgX = nullptr, *cgR = nullptr, *cgP = nullptr, *cgGp = nullptr;
    int* cg_act = nullptr;
    void* cg_st = nullptr;        // CgTraj[B*NR]
    int* cg_live = nullptr;       // [0] live counter, [1] last value
    cudaStream_t side = nullptr;  // captures the CG loop body
    cimcs_timing timing{};

    // fp64 state arrays (c, e, R, w, D, hz)
    bool st64() const { return dtype == CIMCS_F64; }
    size_t elt() const { return st64() ? 8 : 4; }
    const void* G() const { return dG; }
    size_t state_elems() const { return (size_t)B * ldN * NR; }
    // contraction-input arrays: [b][i][r], or (tc) [W | W_lo] canonical, 2*NR rows
    size_t w_elems() const { return (size_t)B * (ldJ > ldN ? ldJ : ldN) * NR * (tc ? 2 : 1); }
};

namespace {

// contraction-input layout: the streaming tcgen05 kernel reads W
// as the canonical [W | W_lo] operand (tc_wofs); the symmetric-tile path and
// the CUDA-core paths use [b][i][r] (coalesced float4 rows in the update)
inline int wcanon(const cimcs_ctx*) { return 0; }  // plain [b][i][r] on every path

void drop_graphs(cimcs_ctx* c) {
    if (c->g_cim) cudaGraphExecDestroy(c->g_cim);
    if (c->g_refit) cudaGraphExecDestroy(c->g_refit);
    c->g_cim = c->g_refit = nullptr;
    c->graph_key.clear();
}

void free_state(cimcs_ctx* c) {
    drop_graphs(c);
    void* ptrs[] = {c->Rs,  c->C,        c->E,          c->W0,  c->W1,       c->Hdbg,
                    c->bestR, c->sig,    c->bestS,      c->fail_gstep, c->fail_idx, c->n_hist,
                    c->improved, c->minE, c->part,      c->best_obj, c->obj, c->rmse, c->ham,
                    c->tp, c->fail_tmp, c->cgX, c->cgR, c->cgP, c->cgGp, c->cg_act,
                    c->cg_st, c->cg_live, c->WB0, c->WB1, c->WS0, c->WS1, c->WT0, c->WT1, c->Pn, c->Pm,
                    c->MT, c->nzd[0], c->nzd[1], c->dPart6};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    c->cgX = c->cgR = c->cgP = c->cgGp = nullptr;
    c->WB0 = c->WB1 = nullptr;
    c->WS0 = c->WS1 = nullptr;
    c->WT0 = c->WT1 = c->dPart6 = nullptr;
    c->Pn = c->Pm = c->MT = nullptr;
    c->nzd[0] = c->nzd[1] = nullptr;
    for (double*& h : c->nzh)
        if (h) {
            cudaFreeHost(h);
            h = nullptr;
        }
    c->nz_elems = 0;
    c->cg_act = c->cg_live = nullptr;
    c->cg_st = nullptr;
    c->Rs = c->C = c->E = c->W0 = c->W1 = c->Hdbg = c->bestR = nullptr;
    c->sig = c->bestS = nullptr;
    c->fail_gstep = c->fail_idx = c->n_hist = c->improved = nullptr;
    c->minE = nullptr;
    c->part = c->best_obj = c->obj = c->rmse = c->ham = nullptr;
    c->tp = nullptr;
    c->fail_tmp = nullptr;
    c->NR = 0;
}

void free_problems(cimcs_ctx* c) {
    free_state(c);
    void* ptrs[] = {c->dA, c->dy, c->dM, c->dG, c->dG6, c->dD, c->dhz, c->dx, c->dxi,
                    c->dSg, c->dSpart, c->dMaskBr, c->dTw, c->dTarget,
                    c->dH};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (auto& q : c->ssched) {
        cudaFree(q.items);
        cudaFree(q.sched);
    }
    c->ssched.clear();
    c->dSg = nullptr;
    c->dSpart = nullptr;
    c->dMaskBr = nullptr;
    c->dH = nullptr;
    c->dTw = nullptr;
    c->dTarget = nullptr;
    c->mri = false;
    c->spart_elems = 0;
    c->dA = c->dy = nullptr;
    c->dM = nullptr;
    c->dG = c->dG6 = nullptr;
    c->dD = c->dhz = nullptr;
    c->dx = nullptr;
    c->dxi = nullptr;
    c->B = c->N = c->ldN = 0;
    c->built = false;
}

// Device allocation, zero-filled ON THE CONTEXT STREAM: every later upload,
// kernel and download of the context is ordered after the fill by the stream
// itself (no device-wide sync; round 1 filled on the legacy stream, which does
// not order against the non-blocking context stream, and a second context's
// fill overwrote freshly uploaded instances).
template <typename P>
int dalloc(cimcs_ctx* c, P** p, size_t bytes) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 16));
    if (e != cudaSuccess)
        return fail(CIMCS_CUDA_ERROR, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    e = cudaMemsetAsync(*p, 0, std::max<size_t>(bytes, 16), c->stream);
    if (e != cudaSuccess)
        return fail(CIMCS_CUDA_ERROR, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
    return 0;
}

// Synchronous copy ordered on the context stream (all host <-> device traffic
// of a context goes through its stream; the host buffer may be reused on return).
int copy_sync(cimcs_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess)
        return fail(CIMCS_CUDA_ERROR, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
    return 0;
}

#define NK(x)                                                                           \
    do {                                                                                \
        ncclResult_t r_ = (x);                                                          \
        if (r_ != ncclSuccess)                                                          \
            return fail(CIMCS_CUDA_ERROR, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

// Super-rows [P0, P1) of rank `rank` of `world`: contiguous, balanced by the
// number of upper-triangle tiles (super-row P holds the items (P, Q >= P)).
void tile_shard(int nRB, int world, int rank, int* P0, int* P1) {
    const int nSB = (nRB + kSyS - 1) / kSyS;
    std::vector<long long> w(nSB, 0);
    for (int P = 0; P < nSB; ++P)
        for (int Q = P; Q < nSB; ++Q) {
            const int nI = std::min(kSyS, nRB - P * kSyS), nJ = std::min(kSyS, nRB - Q * kSyS);
            w[P] += P == Q ? nI * (nI + 1) / 2 : nI * nJ;
        }
    long long total = 0;
    for (long long x : w) total += x;
    std::vector<int> cut(world + 1, nSB);
    cut[0] = 0;
    long long acc = 0;
    int P = 0;
    for (int r = 1; r < world; ++r) {
        const long long target = total * r / world;
        while (P < nSB && acc + w[P] / 2 < target) acc += w[P++];
        cut[r] = P;
    }
    *P0 = cut[rank];
    *P1 = cut[rank + 1];
}

// Super-block items of nb instances placed on the persistent CTAs, largest
// first onto the least-loaded CTA (LPT); built once per nb and cached.
int sym_schedule(cimcs_ctx* c, int nb, const cimcs_ctx::SymSched** out, bool s64 = false) {
    const int kS = s64 ? kS6 : kSyS;  // item edge in tiles
    const int nRB = s64 ? c->nRB6 : c->nRB, nSB = s64 ? c->nSB6 : c->nSB;
    for (auto& q : c->ssched)
        if (q.nb == nb && q.nRB == nRB && q.S == kS) {
            *out = &q;
            return 0;
        }
    std::vector<std::pair<int, int2>> items;  // (tiles, item)
    const int P0 = c->tshard && !s64 ? c->sP0 : 0, P1 = c->tshard && !s64 ? c->sP1 : nSB;
    for (int b = 0; b < nb; ++b)
        for (int P = P0; P < P1; ++P)
            for (int Q = P; Q < nSB; ++Q) {
                const int nI = std::min(kS, nRB - P * kS), nJ = std::min(kS, nRB - Q * kS);
                const int t = P == Q ? nI * (nI + 1) / 2 : nI * nJ;
                items.push_back({t, make_int2(b, P << 16 | Q)});
            }
    std::stable_sort(items.begin(), items.end(),
                     [](const auto& x, const auto& y) { return x.first > y.first; });
    const int grid = (int)std::max<size_t>(1, std::min<size_t>(items.size(), (size_t)c->num_sms));
    std::vector<std::vector<int2>> per(grid);
    using L = std::pair<long long, int>;  // (load, cta)
    std::priority_queue<L, std::vector<L>, std::greater<L>> pq;
    for (int g = 0; g < grid; ++g) pq.push({0, g});
    for (const auto& it : items) {
        L l = pq.top();
        pq.pop();
        per[l.second].push_back(it.second);
        pq.push({l.first + it.first, l.second});
    }
    std::vector<int2> flat;
    std::vector<int> beg(grid + 1, 0);
    for (int g = 0; g < grid; ++g) {
        beg[g] = (int)flat.size();
        flat.insert(flat.end(), per[g].begin(), per[g].end());
    }
    beg[grid] = (int)flat.size();
    cimcs_ctx::SymSched q;
    q.nb = nb;
    q.nRB = nRB;
    q.S = kS;
    q.grid = grid;
    int rc;
    if ((rc = dalloc(c, &q.items, flat.size() * sizeof(int2))) ||
        (rc = dalloc(c, &q.sched, beg.size() * sizeof(int))))
        return rc;
    if (int rc_ = copy_sync(c, q.items, flat.data(), flat.size() * sizeof(int2), cudaMemcpyHostToDevice)) return rc_;
    if (int rc_ = copy_sync(c, q.sched, beg.data(), beg.size() * sizeof(int), cudaMemcpyHostToDevice)) return rc_;
    c->ssched.push_back(q);
    *out = &c->ssched.back();
    return 0;
}


int ensure_stage(cimcs_ctx* c, size_t elems) {
    if (c->stage_elems >= elems) return 0;
    if (c->stage) cudaFree(c->stage);
    if (c->stage_i) cudaFree(c->stage_i);
    c->stage = nullptr;
    c->stage_i = nullptr;
    c->stage_elems = 0;
    if (int rc = dalloc(c, &c->stage, elems * 8)) return rc;
    if (int rc = dalloc(c, &c->stage_i, elems * 4)) return rc;
    c->stage_elems = elems;
    return 0;
}

int ensure_state(cimcs_ctx* c, int NR) {
    if (c->NR == NR && c->Rs) return 0;
    free_state(c);
    c->NR = NR;
    const size_t n = c->state_elems(), es = c->elt();
    const int nT = c->B * NR;
    const int nRB = std::max(std::max(c->nRB, c->nRB6), 1);
    int rc = 0;
    const size_t nw = c->w_elems();
    if ((rc = dalloc(c, &c->Rs, n * es)) || (rc = dalloc(c, &c->C, n * es)) ||
        (rc = dalloc(c, &c->E, n * es)) || (rc = dalloc(c, &c->W0, nw * es)) ||
        (rc = dalloc(c, &c->W1, nw * es)) || (rc = dalloc(c, &c->Hdbg, n * es)) ||
        (rc = dalloc(c, &c->bestR, n * es)) || (rc = dalloc(c, &c->sig, n)) ||
        (rc = dalloc(c, &c->bestS, n)) || (rc = dalloc(c, &c->fail_gstep, nT * 4)) ||
        (rc = dalloc(c, &c->fail_idx, nT * 4)) || (rc = dalloc(c, &c->n_hist, nT * 4)) ||
        (rc = dalloc(c, &c->improved, nT * 4)) || (rc = dalloc(c, &c->minE, nT * 8)) ||
        (rc = dalloc(c, &c->part, (size_t)c->B * nRB * NR * 4 * 8)) ||
        (rc = dalloc(c, &c->best_obj, nT * 8)) || (rc = dalloc(c, &c->obj, nT * 8)) ||
        (rc = dalloc(c, &c->rmse, nT * 8)) || (rc = dalloc(c, &c->ham, nT * 8)) ||
        (rc = dalloc(c, &c->tp, (size_t)nT * 5 * 8)) || (rc = dalloc(c, &c->fail_tmp, nT * 4)))
        return rc;
    if (c->mri) {  // G w of the transform chain, one slot: [N][NR]
        const size_t ne = (size_t)c->nRB * kSyT * NR;
        if (c->spart_elems < ne) {
            if (c->dSpart) cudaFree(c->dSpart);
            c->dSpart = nullptr;
            c->spart_elems = 0;
            if ((rc = dalloc(c, &c->dSpart, ne * 4))) return rc;
            c->spart_elems = ne;
        }
    }
    if (c->sym64) {  // fp64 w tiles of W0/W1, the slot partials and the item schedule
        const size_t nw = (size_t)c->B * c->nRB6 * kT6 * NR;
        if ((rc = dalloc(c, &c->WT0, nw * 8)) || (rc = dalloc(c, &c->WT1, nw * 8)) ||
            (rc = dalloc(c, &c->dPart6, nw * c->nSB6 * 8)))
            return rc;
        const cimcs_ctx::SymSched* ss;
        if ((rc = sym_schedule(c, c->B, &ss, true))) return rc;
    }
    if (c->sym) {  // fp16 B tiles of W0/W1 and the partial products of the symmetric kernel
        const size_t nb = (size_t)c->B * c->nRB * 2 * NR * kSyT, ns = (size_t)c->B * c->nRB * NR;
        if ((rc = dalloc(c, &c->WB0, nb * 2)) || (rc = dalloc(c, &c->WB1, nb * 2)) ||
            (rc = dalloc(c, &c->WS0, ns * 4)) || (rc = dalloc(c, &c->WS1, ns * 4)))
            return rc;
        const size_t ne = (size_t)c->B * c->nRB * c->nSB * kSyT * NR;
        // the item schedule (built outside graph capture)
        const cimcs_ctx::SymSched* ss;
        if ((rc = sym_schedule(c, c->B, &ss))) return rc;
        if (ne && c->spart_elems < ne) {
            if (c->dSpart) cudaFree(c->dSpart);
            c->dSpart = nullptr;
            c->spart_elems = 0;
            if ((rc = dalloc(c, &c->dSpart, ne * 4))) return rc;
            c->spart_elems = ne;
        }
        if (c->tshard) {  // slots of other ranks' items stay zero for good
            CK(cudaMemsetAsync(c->dSpart, 0, ne * 4, c->stream));
            if (c->dH) cudaFree(c->dH);
            c->dH = nullptr;
            if ((rc = dalloc(c, &c->dH, (size_t)c->B * c->nRB * kSyT * NR * 4))) return rc;
        }
    }
    return 0;
}

StepScalars make_scalars(const cimcs_hyper* hp) {
    StepScalars s{};
    s.dt = hp->dt;
    s.rt = std::sqrt(hp->tau);
    s.half_rt = s.rt / 2.0;
    s.tau = hp->tau;
    s.nbeta = -hp->beta;
    s.Kj = hp->K * hp->j;
    s.minus_j = hp->mfz_loss_minus_j ? hp->j : 0.0;
    s.one_minus_dtc = 1.0 - hp->dt_c;
    s.dt_c = hp->dt_c;
    s.g2 = hp->g2;
    s.j = hp->j;
    s.pp_scale = std::sqrt(hp->g2 / (4.0 * hp->j * hp->dt));  // solver_pp.cpp:27
    s.pp_sdt = std::sqrt(hp->dt);
    s.pp_sjg = std::sqrt(hp->j * hp->g2);
    s.pp_m2j = -2.0 * (1.0 + hp->j);
    s.mu_abort = hp->mu_abort;
    s.n_steps = hp->n_steps;
    return s;
}

AltParams make_alt(const cimcs_hyper* hp, double eta, int alt) {
    AltParams a{};
    const double rt = std::sqrt(hp->tau);
    a.thresh = eta * eta / 4.0 * rt;  // solver_mfz.cpp:69
    a.thresh_pp = rt * eta * eta / 4.0;  // solver_pp.cpp:59
    a.lambda = eta * eta / 2.0;       // orchestrator.cpp:189
    a.eta = eta;
    a.alt = alt;
    a.gstep_base = alt * hp->n_steps;
    return a;
}

double eta_schedule(int i, double eta_init, double eta_end, int velo) {
    const double linear = eta_init * (1.0 - static_cast<double>(i) / velo);
    return std::max(linear, eta_end);
}

std::vector<double> pump_table(const cimcs_hyper* hp) {
    std::vector<double> p(hp->n_steps);
    double t = 0.0;
    const double T = static_cast<double>(hp->n_steps) * hp->dt;
    for (int k = 0; k < hp->n_steps; ++k) {
        p[k] = hp->pump_kind == CIMCS_PUMP_LINEAR
                   ? hp->pump_end * t / T
                   : (hp->p_thr - hp->d) + 2.0 * hp->d / (1.0 + std::exp(-(t - 4.0) / 2.0));
        t = t + hp->dt;
    }
    return p;
}

// ----------------------------------------------------- typed dispatch
template <typename T, int NR, int MODE>
int launch_gemv_t(cimcs_ctx* c, const GemvArgs& a) {
    auto kern = gemv_fused_kernel<T, NR, MODE>;
    constexpr size_t smem = gemv_smem_bytes<T, NR>();
    static std::atomic<unsigned long long> attr{0};  // per device: the attribute is per context
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr.fetch_or(1ull << c->device);
    }
    if (c->nRB == 0) return 0;  // this rank holds no rows
    dim3 grid(c->nRB, c->B);
    kern<<<grid, kThreads, smem, c->stream>>>(a);
    CK(cudaGetLastError());
    return 0;
}

template <typename T, int NR>
int launch_gemv_nr(cimcs_ctx* c, int mode, const GemvArgs& a) {
    switch (mode) {
        case EPI_STEP_BN: return launch_gemv_t<T, NR, EPI_STEP_BN>(c, a);
        case EPI_STEP_CN: return launch_gemv_t<T, NR, EPI_STEP_CN>(c, a);
        case EPI_JACOBI: return launch_gemv_t<T, NR, EPI_JACOBI>(c, a);
        case EPI_MATVEC: return launch_gemv_t<T, NR, EPI_MATVEC>(c, a);
        case EPI_STEP_PP: return launch_gemv_t<T, NR, EPI_STEP_PP>(c, a);
        default: return launch_gemv_t<T, NR, EPI_SCORE>(c, a);
    }
}

template <typename T>
int launch_gemv_T(cimcs_ctx* c, int mode, const GemvArgs& a) {
    switch (c->NR) {
        case 1: return launch_gemv_nr<T, 1>(c, mode, a);
        case 2: return launch_gemv_nr<T, 2>(c, mode, a);
        case 4: return launch_gemv_nr<T, 4>(c, mode, a);
        case 8: return launch_gemv_nr<T, 8>(c, mode, a);
        default: return launch_gemv_nr<T, 16>(c, mode, a);
    }
}

TcArgs tc_args(const cimcs_ctx* c, const GemvArgs& g) {
    TcArgs a{};
    a.D = g.D;
    a.hz = g.hz;
    a.Win = g.Win;
    a.Wout = g.Wout;
    a.Rs = g.Rs;
    a.C = g.C;
    a.E = g.E;
    a.Hdbg = g.Hdbg;
    a.Mv = g.Mv;
    a.sigma = g.sigma;
    a.fail_gstep = g.fail_gstep;
    a.fail_idx = g.fail_idx;
    a.minE = g.minE;
    a.part = g.part;
    a.pump = g.pump;
    a.alt = g.alt;
    a.xtrue = g.xtrue;
    a.xitrue = g.xitrue;
    a.err = g.err;
    a.p_scalar = g.p_scalar;
    a.step = g.step;
    a.N = c->N;
    a.ldN = c->ldN;
    a.ldJ = c->ldJ;
    a.B = c->B;
    a.nRB = c->nRB;
    a.nch = c->nch;
    a.ntiles = c->B * c->nRB;
    a.rb0 = c->rb0;
    a.s = g.s;
    return a;
}




// symmetric-tile variant (sym_kernels.cuh): half the gram bytes per step.
// The tile kernel, then the slot reduction and the fused update, on the
// context stream (instances [b0, b0 + nb)).
template <int NR, int MODE>
int launch_sym_t(cimcs_ctx* c, const GemvArgs& g, int b0, int nb) {
    cudaStream_t sA = c->stream, sF = c->stream;
    SymArgs sa{};
    sa.t = tc_args(c, g);
    sa.Gs = static_cast<const __half*>(c->dG);
    sa.sg = c->dSg;
    sa.WBin = g.Win == c->W0 ? c->WB0 : c->WB1;
    sa.WSin = g.Win == c->W0 ? c->WS0 : c->WS1;
    sa.WBout = g.Wout == c->W0 ? c->WB0 : c->WB1;
    sa.WSout = g.Wout == c->W0 ? c->WS0 : c->WS1;
    sa.spart = c->dSpart;
    sa.ntri = c->ntri;
    sa.nSB = c->nSB;
    sa.b0 = b0;
    sa.gram_keep = c->gram_l2;
    if (nb == 0 || c->ntri == 0) return 0;
    const cimcs_ctx::SymSched* ss = nullptr;
    if (int rc = sym_schedule(c, nb, &ss)) return rc;
    sa.items = ss->items;
    sa.sched = ss->sched;
    auto kern = sym_step_kernel<NR, MODE>;
    constexpr size_t smem = sy_smem_bytes<NR>();
    static std::atomic<unsigned long long> attr{0};  // per device: the attribute is per context
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr.fetch_or(1ull << c->device);
    }
    // same stream: both kernels use programmatic dependent launch (the next
    // kernel's prologue overlaps this one's tail; griddepcontrol.wait orders data)
    const bool pdl = sF == sA && c->use_pdl && !c->tshard;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ss->grid);
    cfg.blockDim = dim3(kSyThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = sA;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    const bool timed = c->kernel_timing && (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) &&
                       cudaStreamIsCapturing(sA, &cap) == cudaSuccess &&
                       cap == cudaStreamCaptureStatusNone;
    if (timed) {
        if (!c->kt_ev[0]) {
            CK(cudaEventCreate(&c->kt_ev[0]));
            CK(cudaEventCreate(&c->kt_ev[1]));
        }
        CK(cudaEventRecord(c->kt_ev[0], sA));
    }
    CK(cudaLaunchKernelEx(&cfg, kern, sa));
    if (timed) {  // the kernel alone, on its own stream (serialises the step: a measurement mode)
        CK(cudaEventRecord(c->kt_ev[1], sA));
        CK(cudaEventSynchronize(c->kt_ev[1]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->kt_ev[0], c->kt_ev[1]));
        c->timing.tile_kernel_ms += ms;
        c->timing.tile_kernel_launches += 1;
    }
    if (c->tshard) {  // own items' slot sums, then the cross-rank sum (one collective)
        sym_slotsum_kernel<NR><<<dim3(c->nRB, nb), kSyT * NR / 4, 0, sF>>>(c->dSpart, c->dH, c->nRB,
                                                                         c->nSB, b0);
        CK(cudaGetLastError());
        if (c->tworld > 1) {
            const size_t per = (size_t)c->nRB * kSyT * NR;
            NK(ncclAllReduce(c->dH + (size_t)b0 * per, c->dH + (size_t)b0 * per, (size_t)nb * per,
                             ncclFloat32, ncclSum, c->comm, sF));
        }
        sa.spart = c->dH;
        sa.nSB = 1;
    }
    cfg.gridDim = dim3(c->nRB, nb);
    cfg.blockDim = dim3(kSyT * NR / 4);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = sF;
    CK(cudaLaunchKernelEx(&cfg, sym_update_kernel<NR, MODE, float>, sa));
    return 0;
}

template <int NR>
int launch_sym_grp(cimcs_ctx* c, int mode, const GemvArgs& a, int b0, int nb) {
    switch (mode) {
        case EPI_STEP_BN: return launch_sym_t<NR, EPI_STEP_BN>(c, a, b0, nb);
        case EPI_STEP_CN: return launch_sym_t<NR, EPI_STEP_CN>(c, a, b0, nb);
        case EPI_JACOBI: return launch_sym_t<NR, EPI_JACOBI>(c, a, b0, nb);
        case EPI_MATVEC: return launch_sym_t<NR, EPI_MATVEC>(c, a, b0, nb);
        default: return launch_sym_t<NR, EPI_SCORE>(c, a, b0, nb);
    }
}


template <int NR>
int launch_sym_nr(cimcs_ctx* c, int mode, const GemvArgs& a) {
    return launch_sym_grp<NR>(c, mode, a, 0, c->B);
}


// fp64 symmetric-tile path (sym64_kernels.cuh): the DMMA tile kernel, then the
// fused fp64 update, both on the context stream with PDL between them.
template <int NR, int MODE>
int launch_sym64_t(cimcs_ctx* c, const GemvArgs& g) {
    Sym64Args sa{};
    sa.t = tc_args(c, g);
    sa.t.nRB = c->nRB6;
    sa.Gt = static_cast<const double*>(c->dG6);
    sa.WTin = g.Win == c->W0 ? c->WT0 : c->WT1;
    sa.WTout = g.Wout == c->W0 ? c->WT0 : (g.Wout == c->W1 ? c->WT1 : nullptr);
    sa.part = c->dPart6;
    sa.ntri = c->ntri6;
    sa.nSB = c->nSB6;
    const cimcs_ctx::SymSched* ss = nullptr;
    if (int rc = sym_schedule(c, c->B, &ss, true)) return rc;
    sa.items = ss->items;
    sa.sched = ss->sched;
    auto kern = sym64_step_kernel<NR, MODE>;
    constexpr size_t smem = s6_smem_bytes<NR>();
    static std::atomic<unsigned long long> attr{0};
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr.fetch_or(1ull << c->device);
    }
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ss->grid);
    cfg.blockDim = dim3(kT6Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cfg.attrs = at;
    cfg.numAttrs = c->use_pdl ? 1 : 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    const bool timed = c->kernel_timing && (MODE == EPI_STEP_BN || MODE == EPI_STEP_CN) &&
                       cudaStreamIsCapturing(c->stream, &cap) == cudaSuccess &&
                       cap == cudaStreamCaptureStatusNone;
    if (timed) {
        if (!c->kt_ev[0]) {
            CK(cudaEventCreate(&c->kt_ev[0]));
            CK(cudaEventCreate(&c->kt_ev[1]));
        }
        CK(cudaEventRecord(c->kt_ev[0], c->stream));
    }
    CK(cudaLaunchKernelEx(&cfg, kern, sa));
    if (timed) {
        CK(cudaEventRecord(c->kt_ev[1], c->stream));
        CK(cudaEventSynchronize(c->kt_ev[1]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->kt_ev[0], c->kt_ev[1]));
        c->timing.tile_kernel_ms += ms;
        c->timing.tile_kernel_launches += 1;
    }
    cfg.gridDim = dim3(c->nRB6, c->B);
    cfg.blockDim = dim3(kT6 * NR / 4);
    cfg.dynamicSmemBytes = 0;
    CK(cudaLaunchKernelEx(&cfg, sym64_update_kernel<NR, MODE>, sa));
    return 0;
}

template <int NR>
int launch_sym64_nr(cimcs_ctx* c, int mode, const GemvArgs& a) {
    switch (mode) {
        case EPI_STEP_BN: return launch_sym64_t<NR, EPI_STEP_BN>(c, a);
        case EPI_STEP_CN: return launch_sym64_t<NR, EPI_STEP_CN>(c, a);
        case EPI_JACOBI: return launch_sym64_t<NR, EPI_JACOBI>(c, a);
        case EPI_MATVEC: return launch_sym64_t<NR, EPI_MATVEC>(c, a);
        default: return launch_sym64_t<NR, EPI_SCORE>(c, a);
    }
}

// one mri_kernel launch of `grid` CTAs (basis vectors r0.. for DIAG / COLS)
int mri_launch(cimcs_ctx* c, int mode, int grid, int r0, const float* in, float* out) {
    MriArgs ma{};
    ma.H = c->mH;
    ma.W = c->mW;
    ma.N = c->N;
    ma.NR = 1;
    ma.mask_br = c->dMaskBr;
    ma.tw = c->dTw;
    ma.L = c->mL;
    ma.gamma = c->mgamma;
    ma.scale = 1.f / (float)c->N;
    ma.in = in;
    ma.out = out;
    ma.r0 = r0;
    mri_kernel<<<grid, kMriThreads, mri_smem_bytes(c->mH, c->mW, c->mL), c->stream>>>(ma, mode);
    CK(cudaGetLastError());
    return 0;
}

// transform-chain problems: G w by the matrix-free MRI kernel (one CTA per
// replica slot) into the one-slot partial buffer, then the symmetric path's
// update kernel for the fused epilogue of `mode`
template <int NR, int MODE>
int launch_mri_t(cimcs_ctx* c, const GemvArgs& g) {
    MriArgs ma{};
    ma.H = c->mH;
    ma.W = c->mW;
    ma.N = c->N;
    ma.NR = NR;
    ma.mask_br = c->dMaskBr;
    ma.tw = c->dTw;
    ma.L = c->mL;
    ma.gamma = c->mgamma;
    ma.scale = 1.f / (float)c->N;
    ma.in = static_cast<const float*>(g.Win);
    ma.out = c->dSpart;
    if (c->mri_cluster && std::min(c->mH, c->mW) >= 2 * kMriCluster) {
        // one thread-block cluster per replica (mri_cluster_kernel)
        const int CS = mri_cluster_size(c->mH, c->mW);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(NR * CS);
        cfg.blockDim = dim3(kMriCThreads);
        cfg.dynamicSmemBytes = mri_cluster_smem_bytes(c->mH, c->mW);
        cfg.stream = c->stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = c->use_pdl ? 2 : 1;
        CK(cudaLaunchKernelEx(&cfg, mri_cluster_kernel, ma));
    } else {
        const size_t smem = mri_smem_bytes(c->mH, c->mW, c->mL);
        mri_kernel<<<NR, kMriThreads, smem, c->stream>>>(ma, MRI_APPLY);
    }
    CK(cudaGetLastError());
    SymArgs sa{};
    sa.t = tc_args(c, g);
    sa.spart = c->dSpart;
    sa.nSB = 1;
    sa.b0 = 0;
    sa.keep_w = 1;  // the next apply reads the fp32 w
    {
        cudaLaunchConfig_t ucfg{};
        ucfg.gridDim = dim3(c->nRB, 1);
        ucfg.blockDim = dim3(kSyT * NR / 4);
        ucfg.stream = c->stream;
        cudaLaunchAttribute ua[1];
        ua[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        ua[0].val.programmaticStreamSerializationAllowed = 1;
        ucfg.attrs = ua;
        ucfg.numAttrs = c->use_pdl ? 1 : 0;
        CK(cudaLaunchKernelEx(&ucfg, sym_update_kernel<NR, MODE>, sa));
    }
    CK(cudaGetLastError());
    return 0;
}

template <int NR>
int launch_mri_nr(cimcs_ctx* c, int mode, const GemvArgs& a) {
    switch (mode) {
        case EPI_STEP_BN: return launch_mri_t<NR, EPI_STEP_BN>(c, a);
        case EPI_STEP_CN: return launch_mri_t<NR, EPI_STEP_CN>(c, a);
        case EPI_MATVEC: return launch_mri_t<NR, EPI_MATVEC>(c, a);
        case EPI_SCORE: return launch_mri_t<NR, EPI_SCORE>(c, a);
        default: return fail(CIMCS_CONFIG_ERROR, "cdp_minimize_operator: damped Jacobi needs an assembled matrix");
    }
}

int launch_gemv(cimcs_ctx* c, int mode, const GemvArgs& a) {
    if (c->mri) return c->NR == 8 ? launch_mri_nr<8>(c, mode, a) : launch_mri_nr<16>(c, mode, a);
    if (c->sym64)
        return c->NR == 8 ? launch_sym64_nr<8>(c, mode, a) : launch_sym64_nr<16>(c, mode, a);
    if (c->sym) return c->NR == 8 ? launch_sym_nr<8>(c, mode, a) : launch_sym_nr<16>(c, mode, a);
    return c->st64() ? launch_gemv_T<double>(c, mode, a)
                                 : launch_gemv_T<float>(c, mode, a);
}

#define DISPATCH_NR_TC(NRV, ...)                                            \
    if ((NRV) == 8) { constexpr int NR_ = 8; __VA_ARGS__; }                 \
    else { constexpr int NR_ = 16; __VA_ARGS__; }

// symmetric path: refresh the fp16 B tiles of W (W0 or W1) after a writer
// other than the symmetric kernel itself
int sym_sync_w(cimcs_ctx* c, const void* W) {
    const bool w0 = W == c->W0;
    const dim3 g(c->nRB, c->B);
    if (c->sym64) {
        DISPATCH_NR_TC(c->NR, {
            sym64_wconvert_kernel<NR_><<<dim3(c->nRB6, c->B), 256, 0, c->stream>>>(
                static_cast<const double*>(W), c->N, c->ldN, c->nRB6, w0 ? c->WT0 : c->WT1);
        });
        CK(cudaGetLastError());
    }
    if (!c->sym) return 0;
    DISPATCH_NR_TC(c->NR, {
        sym_wconvert_kernel<NR_, float><<<g, 128, 0, c->stream>>>(
            static_cast<const float*>(W), c->N, c->ldN, c->nRB, w0 ? c->WB0 : c->WB1,
            w0 ? c->WS0 : c->WS1);
    });
    CK(cudaGetLastError());
    return 0;
}

// replica slots: a power of two; the tensor-core path needs MMA N in {8, 16}
int slots_for(const cimcs_ctx* c, int R) {
    const int p = pow2_slots(R);
    return c->tc || c->mri || c->sym64 ? std::max(8, p) : p;
}

// Generic NR/T dispatch for the small state kernels.
#define DISPATCH_NR(NRV, ...)                                               \
    switch (NRV) {                                                          \
        case 1: { constexpr int NR_ = 1; __VA_ARGS__; } break;              \
        case 2: { constexpr int NR_ = 2; __VA_ARGS__; } break;              \
        case 4: { constexpr int NR_ = 4; __VA_ARGS__; } break;              \
        case 8: { constexpr int NR_ = 8; __VA_ARGS__; } break;              \
        default: { constexpr int NR_ = 16; __VA_ARGS__; } break;            \
    }

template <typename T>
int run_init_T(cimcs_ctx* c, int Rreal, int bn, const double* dc0, const double* de0, double rt) {
    const int g = grid_for(c->state_elems());
    T* W = static_cast<T*>(c->W0);
    DISPATCH_NR(c->NR, {
        if (bn)
            init_state_kernel<T, NR_, 1><<<g, 256, 0, c->stream>>>(
                dc0, Rreal, c->N, c->ldN, c->B, static_cast<const T*>(c->Rs),
                static_cast<T*>(c->C), static_cast<T*>(c->E), W, c->fail_gstep, c->minE, rt,
                de0, wcanon(c), c->ldJ);
        else
            init_state_kernel<T, NR_, 0><<<g, 256, 0, c->stream>>>(
                dc0, Rreal, c->N, c->ldN, c->B, static_cast<const T*>(c->Rs),
                static_cast<T*>(c->C), static_cast<T*>(c->E), W, c->fail_gstep, c->minE, rt,
                de0, wcanon(c), c->ldJ);
    });
    CK(cudaGetLastError());
    return sym_sync_w(c, c->W0);
}

int run_init(cimcs_ctx* c, int Rreal, int bn, const double* dc0, const double* de0, double rt) {
    return c->st64() ? run_init_T<double>(c, Rreal, bn, dc0, de0, rt)
                                 : run_init_T<float>(c, Rreal, bn, dc0, de0, rt);
}

template <typename T>
int run_support_T(cimcs_ctx* c) {
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        support_kernel<T, NR_><<<g, 256, 0, c->stream>>>(
            static_cast<const T*>(c->C), static_cast<const T*>(c->Rs), c->sig,
            static_cast<T*>(c->W0), c->fail_gstep, c->N, c->ldN, c->B, wcanon(c), c->ldJ);
    });
    CK(cudaGetLastError());
    return sym_sync_w(c, c->W0);
}

int run_support(cimcs_ctx* c) {
    return c->st64() ? run_support_T<double>(c) : run_support_T<float>(c);
}

template <typename T>
int upload_traj_T(cimcs_ctx* c, const double* h, void* d, int Rreal, T pad) {
    const size_t n = (size_t)c->B * Rreal * c->N;
    if (int rc = ensure_stage(c, std::max(n, c->state_elems()))) return rc;
    CK(cudaMemcpyAsync(c->stage, h, n * 8, cudaMemcpyHostToDevice, c->stream));
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        traj_to_dev<T, NR_><<<g, 256, 0, c->stream>>>(c->stage, static_cast<T*>(d), Rreal, c->N,
                                                      c->ldN, c->B, pad);
    });
    CK(cudaGetLastError());
    return 0;
}

int upload_traj(cimcs_ctx* c, const double* h, void* d, int Rreal, double pad = 0.0) {
    return c->st64() ? upload_traj_T<double>(c, h, d, Rreal, pad)
                                 : upload_traj_T<float>(c, h, d, Rreal, (float)pad);
}

template <typename T>
int download_traj_T(cimcs_ctx* c, const void* d, double* h, int Rreal) {
    const size_t n = (size_t)c->B * Rreal * c->N;
    if (int rc = ensure_stage(c, std::max(n, c->state_elems()))) return rc;
    const int g = grid_for(n);
    DISPATCH_NR(c->NR, {
        dev_to_traj<T, NR_><<<g, 256, 0, c->stream>>>(static_cast<const T*>(d), c->stage, Rreal,
                                                      c->N, c->ldN, c->B);
    });
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, c->stage, n * 8, cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

int download_traj(cimcs_ctx* c, const void* d, double* h, int Rreal) {
    return c->st64() ? download_traj_T<double>(c, d, h, Rreal)
                                 : download_traj_T<float>(c, d, h, Rreal);
}

int upload_sig(cimcs_ctx* c, const int32_t* h, int8_t* d, int Rreal) {
    const size_t n = (size_t)c->B * Rreal * c->N;
    if (int rc = ensure_stage(c, std::max(n, c->state_elems()))) return rc;
    for (size_t k = 0; k < n; ++k)
        if (h[k] != 0 && h[k] != 1) return fail(CIMCS_INPUT_ERROR, "sigma must be 0/1");
    CK(cudaMemcpyAsync(c->stage_i, h, n * 4, cudaMemcpyHostToDevice, c->stream));
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        sig_to_dev<NR_><<<g, 256, 0, c->stream>>>(c->stage_i, d, Rreal, c->N, c->ldN, c->B);
    });
    CK(cudaGetLastError());
    return 0;
}

int download_sig(cimcs_ctx* c, const int8_t* d, int32_t* h, int Rreal) {
    const size_t n = (size_t)c->B * Rreal * c->N;
    if (int rc = ensure_stage(c, std::max(n, c->state_elems()))) return rc;
    const int g = grid_for(n);
    DISPATCH_NR(c->NR, {
        sig_to_traj<NR_><<<g, 256, 0, c->stream>>>(d, c->stage_i, Rreal, c->N, c->ldN, c->B);
    });
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, c->stage_i, n * 4, cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

template <typename T>
int rinit_hz_T(cimcs_ctx* c, int Rreal) {
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        rinit_hz_kernel<T, NR_><<<g, 256, 0, c->stream>>>(static_cast<const T*>(c->dhz),
                                                          static_cast<T*>(c->Rs), Rreal, c->N,
                                                          c->ldN, c->B);
    });
    CK(cudaGetLastError());
    return 0;
}

template <typename T>
int mask_T(cimcs_ctx* c, void* V) {
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        mask_kernel<T, NR_><<<g, 256, 0, c->stream>>>(static_cast<const T*>(c->Rs), c->sig,
                                                      static_cast<T*>(V), c->state_elems(), c->N,
                                                      c->ldN, c->ldJ, wcanon(c));
    });
    CK(cudaGetLastError());
    return sym_sync_w(c, V);
}

int reset_flags(cimcs_ctx* c, int Rreal) {
    const int nT = c->B * c->NR;
    traj_flags_kernel<<<(nT + 255) / 256, 256, 0, c->stream>>>(c->fail_gstep, c->fail_idx, Rreal,
                                                              c->NR, c->B);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(c->n_hist, 0, nT * 4, c->stream));
    CK(cudaMemsetAsync(c->err, 0x7f, 4, c->stream));
    return 0;
}

GemvArgs base_args(cimcs_ctx* c, const StepScalars& s) {
    GemvArgs a{};
    a.G = c->G();
    a.D = c->dD;
    a.hz = c->dhz;
    a.Rs = c->Rs;
    a.C = c->C;
    a.E = c->E;
    a.sigma = c->sig;
    a.fail_gstep = c->fail_gstep;
    a.fail_idx = c->fail_idx;
    a.minE = c->minE;
    a.part = c->part;
    a.alt = c->alt;
    a.xtrue = c->has_truth ? c->dx : nullptr;
    a.xitrue = c->dxi;
    a.err = c->err;
    a.N = c->N;
    a.ldN = c->ldN;
    a.ldJ = c->ldJ;
    a.B = c->B;
    a.rb0 = c->rb0;
    a.s = s;
    return a;
}

// row blocks of the score partials: the contraction that scores (sym64 if present)
int nRB_of(const cimcs_ctx* c) { return c->sym64 ? c->nRB6 : c->nRB; }

// ------------------------------------------------ row-sharding collectives

ncclDataType_t nccl_t(const cimcs_ctx* c) {
    return c->st64() ? ncclFloat64 : ncclFloat32;
}

// All-gather this rank's rows of a per-instance array X[b][rows][row_elems]
// (rows padded to world * per): in place, one call per instance, grouped.
int allgather_rows(cimcs_ctx* c, void* X, size_t row_elems, size_t inst_elems,
                   ncclDataType_t t, size_t esize) {
    if (c->world == 1) return 0;
    const size_t per = (size_t)(c->ldN / c->world);
    NK(ncclGroupStart());
    for (int b = 0; b < c->B; ++b) {
        char* base = static_cast<char*>(X) + (size_t)b * inst_elems * esize;
        NK(ncclAllGather(base + (size_t)c->rank * per * row_elems * esize, base, per * row_elems, t,
                         c->comm, c->stream));
    }
    NK(ncclGroupEnd());
    return 0;
}

// contraction input (w or the refit's V)
int allgather_w(cimcs_ctx* c, void* W) {
    return allgather_rows(c, W, c->NR, (size_t)c->ldN * c->NR, nccl_t(c), c->elt());
}
int allgather_state(cimcs_ctx* c, void* X) {
    return allgather_rows(c, X, c->NR, (size_t)c->ldN * c->NR, nccl_t(c), c->elt());
}
int allgather_sig(cimcs_ctx* c, int8_t* S) {
    return allgather_rows(c, S, c->NR, (size_t)c->ldN * c->NR, ncclInt8, 1);
}

// After a CIM call: agree on divergence (first step, then first spin of that
// step) and on min_e across ranks.
int reconcile_cim(cimcs_ctx* c) {
    if (c->world == 1) return 0;
    const int nT = c->B * c->NR;
    CK(cudaMemcpyAsync(c->fail_tmp, c->fail_gstep, nT * 4, cudaMemcpyDeviceToDevice, c->stream));
    NK(ncclAllReduce(c->fail_gstep, c->fail_gstep, nT, ncclInt32, ncclMin, c->comm, c->stream));
    fail_fix_kernel<<<(nT + 255) / 256, 256, 0, c->stream>>>(c->fail_tmp, c->fail_gstep,
                                                             c->fail_idx, nT);
    CK(cudaGetLastError());
    NK(ncclAllReduce(c->fail_idx, c->fail_idx, nT, ncclInt32, ncclMin, c->comm, c->stream));
    NK(ncclAllReduce(c->minE, c->minE, nT, ncclUint64, ncclMin, c->comm, c->stream));
    return 0;
}

// Enqueue the n_steps fused Euler steps of one CIM call (graph-capturable).
// ------------------------------------------ small-N cluster loop (N <= 512)
// Replica slots the register-resident G slice leaves room for.
int cluster_max_nr(const cimcs_ctx* c) { return c->st64() ? 4 : 8; }

bool cluster_ok(const cimcs_ctx* c) {
    return c->use_cluster && !c->mri && c->world == 1 && !c->sharded && c->N <= kClMaxN &&
           c->NR <= cluster_max_nr(c);
}

template <typename T, int NR, int MODE>
int launch_cluster_t(cimcs_ctx* c, GemvArgs a, int n_iters) {
    auto kern = cluster_loop_kernel<T, NR, MODE>;
    constexpr size_t smem = cluster_smem_bytes<T, NR>();
    static std::atomic<unsigned long long> attr{0};  // per device: the attribute is per context
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr.fetch_or(1ull << c->device);
    }
    const unsigned cs = (unsigned)((c->N + kClRows - 1) / kClRows);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c->B * cs);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, a, c->nRB, c->nch, n_iters));
    return 0;
}

template <typename T, int NR>
int launch_cluster_nr(cimcs_ctx* c, int mode, const GemvArgs& a, int n_iters) {
    switch (mode) {
        case EPI_STEP_BN: return launch_cluster_t<T, NR, EPI_STEP_BN>(c, a, n_iters);
        case EPI_STEP_CN: return launch_cluster_t<T, NR, EPI_STEP_CN>(c, a, n_iters);
        default: return launch_cluster_t<T, NR, EPI_JACOBI>(c, a, n_iters);
    }
}

template <typename T>
int launch_cluster_T(cimcs_ctx* c, int mode, const GemvArgs& a, int n_iters) {
    switch (c->NR) {
        case 1: return launch_cluster_nr<T, 1>(c, mode, a, n_iters);
        case 2: return launch_cluster_nr<T, 2>(c, mode, a, n_iters);
        case 4: return launch_cluster_nr<T, 4>(c, mode, a, n_iters);
        default:
            if constexpr (sizeof(T) == 4) return launch_cluster_nr<T, 8>(c, mode, a, n_iters);
            return fail(CIMCS_CONFIG_ERROR, "cluster loop: too many replica slots");
    }
}

int launch_cluster(cimcs_ctx* c, int mode, const GemvArgs& a, int n_iters) {
    return c->st64() ? launch_cluster_T<double>(c, mode, a, n_iters)
                                 : launch_cluster_T<float>(c, mode, a, n_iters);
}

// n_iters launches of `mode` with W ping-pong (Euler steps or Jacobi sweeps) on
// the symmetric path (pipelining instance groups over two streams was measured
// slower: DESIGN.md section 4).
int enqueue_sym_loop(cimcs_ctx* c, int mode, GemvArgs a, int n_iters, bool steps) {
    for (int k = 0; k < n_iters; ++k) {
        if (steps) a.step = k;
        a.Win = (k & 1) ? c->W1 : c->W0;
        a.Wout = (k & 1) ? c->W0 : c->W1;
        if (int rc = launch_gemv(c, mode, a)) return rc;
    }
    return 0;
}

int enqueue_steps(cimcs_ctx* c, int bn, const StepScalars& s, int n_steps) {
    GemvArgs a = base_args(c, s);
    a.pump = c->pump;
    a.Hdbg = nullptr;
    if (cluster_ok(c)) {  // all n_steps in one launch; final w in W[n_steps & 1]
        a.step = 0;
        a.Win = c->W0;
        a.Wout = (n_steps & 1) ? c->W1 : c->W0;
        return launch_cluster(c, bn ? EPI_STEP_BN : EPI_STEP_CN, a, n_steps);
    }
    if (c->sym || c->sym64)
        return enqueue_sym_loop(c, bn ? EPI_STEP_BN : EPI_STEP_CN, a, n_steps, true);
    for (int k = 0; k < n_steps; ++k) {
        a.step = k;
        a.Win = (k & 1) ? c->W1 : c->W0;
        a.Wout = (k & 1) ? c->W0 : c->W1;
        if (int rc = launch_gemv(c, bn ? EPI_STEP_BN : EPI_STEP_CN, a)) return rc;
        if (int rc = allgather_w(c, a.Wout)) return rc;  // row sharding: exchange w
    }
    return reconcile_cim(c);
}

// support + masked Jacobi sweeps (graph-capturable).  Final V in W[iters&1].
int enqueue_refit(cimcs_ctx* c, const StepScalars& s, int iters, bool do_support) {
    if (do_support) {
        if (int rc = run_support(c)) return rc;
    }
    if (int rc = allgather_w(c, c->W0)) return rc;
    GemvArgs a = base_args(c, s);
    if (cluster_ok(c) && iters > 0) {  // all sweeps in one launch; final V in W[iters & 1]
        a.Win = c->W0;
        a.Wout = (iters & 1) ? c->W1 : c->W0;
        return launch_cluster(c, EPI_JACOBI, a, iters);
    }
    if (c->sym || c->sym64) {
        if (int rc = enqueue_sym_loop(c, EPI_JACOBI, a, iters, false)) return rc;
        return 0;
    }
    for (int it = 0; it < iters; ++it) {
        a.Win = (it & 1) ? c->W1 : c->W0;
        a.Wout = (it & 1) ? c->W0 : c->W1;
        if (int rc = launch_gemv(c, EPI_JACOBI, a)) return rc;
        if (int rc = allgather_w(c, a.Wout)) return rc;
    }
    if (c->world > 1) {
        if (int rc = allgather_state(c, c->Rs)) return rc;
        NK(ncclAllReduce(c->err, c->err, 1, ncclInt32, ncclMin, c->comm, c->stream));
    }
    return 0;
}

// ---------------------------------------------------- CG refit (cdp="cg")
int ensure_cg(cimcs_ctx* c) {  // outside any capture: allocates
    if (c->cgX) return 0;
    const size_t n = c->state_elems();
    for (double** p : {&c->cgX, &c->cgR, &c->cgP, &c->cgGp})
        if (int rc = dalloc(c, p, n * 8)) return rc;
    if (int rc = dalloc(c, &c->cg_act, n * 4)) return rc;
    if (int rc = dalloc(c, &c->cg_st, (size_t)c->B * c->NR * sizeof(CgTraj))) return rc;
    if (int rc = dalloc(c, &c->cg_live, 2 * 4)) return rc;
    if (!c->side) CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    return 0;
}

CgArgs cg_args(cimcs_ctx* c, const cimcs_hyper* hp) {
    CgArgs a{};
    a.Rs = c->Rs;
    a.sig = c->sig;
    a.hz = c->dhz;
    a.X = c->cgX;
    a.Rr = c->cgR;
    a.P = c->cgP;
    a.Gp = c->cgGp;
    a.act = c->cg_act;
    a.st = static_cast<CgTraj*>(c->cg_st);
    a.fail_gstep = c->fail_gstep;
    a.W = c->W0;
    a.n_live = c->cg_live;
    a.tc = wcanon(c);
    a.ldJ = c->ldJ;
    a.N = c->N;
    a.ldN = c->ldN;
    a.max_iters = hp->cg_max_iters;
    a.tol = hp->cg_tol;
    return a;
}

template <typename T>
int cg_launch(cimcs_ctx* c, int which, const CgArgs& a) {
    const int nT = c->B * c->NR;
    DISPATCH_NR(c->NR, {
        if (which == 0) cg_init_kernel<T, NR_><<<nT, kCgThreads, 0, c->stream>>>(a);
        else if (which == 1) cg_iter_kernel<T, NR_><<<nT, kCgThreads, 0, c->stream>>>(a);
        else cg_final_kernel<T, NR_><<<nT, kCgThreads, 0, c->stream>>>(a);
    });
    CK(cudaGetLastError());
    return 0;
}

int cg_kernel(cimcs_ctx* c, int which, const CgArgs& a) {
    return c->st64() ? cg_launch<double>(c, which, a) : cg_launch<float>(c, which, a);
}

// G p for every trajectory (the EPI_MATVEC contraction of W0 into cgGp)
int cg_matvec(cimcs_ctx* c, const StepScalars& s) {
    GemvArgs g = base_args(c, s);
    g.Win = c->W0;
    g.Wout = nullptr;
    g.Mv = c->cgGp;
    return launch_gemv(c, EPI_MATVEC, g);
}

int cg_cond(cimcs_ctx* c, cudaGraphConditionalHandle h, int use) {
    cg_cond_kernel<<<1, 1, 0, c->stream>>>(c->cg_live, c->cg_live + 1, h, use);
    CK(cudaGetLastError());
    return 0;
}

// The whole masked CG refit of every trajectory on its current support
// (sig), Rs in/out; afterwards W0 = Rs∘sig for the scorer.  Inside a stream
// capture the data-dependent loop is a conditional WHILE node (the body is
// captured on the side stream), so the refit stays one graph launch; outside
// a capture the host polls the live count after every iteration.
int enqueue_cg(cimcs_ctx* c, const StepScalars& s, const cimcs_hyper* hp) {
    if (c->world > 1) return fail(CIMCS_CONFIG_ERROR, "cdp=cg is not supported on row-sharded contexts");
    if (int rc = ensure_cg(c)) return rc;
    cudaStreamCaptureStatus cs;
    cudaGraph_t cgraph = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CK(cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &cgraph, &deps, &ndeps));
    const bool in_graph = cs == cudaStreamCaptureStatusActive;
    cudaGraphConditionalHandle h{};
    if (in_graph) CK(cudaGraphConditionalHandleCreate(&h, cgraph, 0, 0));
    const CgArgs a = cg_args(c, hp);
    int rc = c->st64() ? mask_T<double>(c, c->W0) : mask_T<float>(c, c->W0);
    if (!rc) rc = cg_matvec(c, s);  // G x0
    if (!rc) rc = cg_kernel(c, 0, a);
    if (!rc) rc = sym_sync_w(c, c->W0);
    if (!rc) rc = cg_cond(c, h, in_graph ? 1 : 0);
    if (rc) return rc;
    if (in_graph) {
        CK(cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &cgraph, &deps, &ndeps));
        cudaGraphNodeParams np{};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, cgraph, deps, ndeps, &np));
        cudaGraph_t body = np.conditional.phGraph_out[0];
        CK(cudaStreamUpdateCaptureDependencies(c->stream, &node, 1,
                                               cudaStreamSetCaptureDependencies));
        cudaStream_t main = c->stream;
        c->stream = c->side;
        cudaError_t e = cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0,
                                                      cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            rc = cg_matvec(c, s);
            if (!rc) rc = cg_kernel(c, 1, a);
            if (!rc) rc = sym_sync_w(c, c->W0);
            if (!rc) rc = cg_cond(c, h, 1);
            cudaGraph_t out;
            e = cudaStreamEndCapture(c->stream, &out);
        }
        c->stream = main;
        if (rc) return rc;
        CK(e);
    } else {
        int live = 0;
        CK(cudaMemcpyAsync(&live, c->cg_live + 1, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        while (live > 0) {
            if ((rc = cg_matvec(c, s)) || (rc = cg_kernel(c, 1, a)) ||
                (rc = sym_sync_w(c, c->W0)) || (rc = cg_cond(c, h, 0)))
                return rc;
            CK(cudaMemcpyAsync(&live, c->cg_live + 1, 4, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
    }
    rc = cg_kernel(c, 2, a);
    if (!rc) rc = c->st64() ? mask_T<double>(c, c->W0) : mask_T<float>(c, c->W0);
    return rc;
}

template <typename T>
int enqueue_median_T(cimcs_ctx* c, DevRecord* hist_alt) {
    int P = 1;
    while (P < c->N) P <<= 1;
    const size_t smem = (size_t)P * sizeof(T);
    if (smem > 200 * 1024) return 0;  // median left as NaN beyond 25k/51k spins
    DISPATCH_NR(c->NR, {
        auto k = median_kernel<T, NR_>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<c->B * c->NR, 1024, smem, c->stream>>>(static_cast<const T*>(c->E), c->fail_gstep,
                                                  c->N, c->ldN, P, hist_alt);
    });
    CK(cudaGetLastError());
    return 0;
}

// scorer on V = W[v_slot]: score GEMV + finalize (+ history, + best tracking)
int enqueue_score(cimcs_ctx* c, const StepScalars& s, int v_slot, DevRecord* hist_alt,
                  bool track_best) {
    GemvArgs a = base_args(c, s);
    a.Win = v_slot ? c->W1 : c->W0;
    a.Wout = nullptr;
    if (int rc = launch_gemv(c, EPI_SCORE, a)) return rc;
    const int nT = c->B * c->NR;
    DISPATCH_NR(c->NR, {
        tp_kernel<NR_><<<nT, 256, 0, c->stream>>>(c->part, nRB_of(c), c->sig, c->dxi, c->row0,
                                                  c->row1, c->ldN, c->has_truth ? 1 : 0, c->tp);
    });
    CK(cudaGetLastError());
    if (c->world > 1)
        NK(ncclAllReduce(c->tp, c->tp, (size_t)nT * 5, ncclFloat64, ncclSum, c->comm, c->stream));
    finalize_kernel<<<(nT + 127) / 128, 128, 0, c->stream>>>(
        c->tp, nT, c->minE, c->fail_gstep, c->alt, c->N, c->has_truth ? 1 : 0, hist_alt,
        c->n_hist, track_best ? c->best_obj : nullptr, c->improved, c->obj, c->rmse, c->ham);
    CK(cudaGetLastError());
    if (hist_alt && c->world > 1) {
        if (int rc = allgather_state(c, c->E)) return rc;
    }
    if (hist_alt) {
        if (int rc = c->st64() ? enqueue_median_T<double>(c, hist_alt)
                                           : enqueue_median_T<float>(c, hist_alt))
            return rc;
    }
    if (track_best) {
        const int g = grid_for(c->state_elems());
        if (c->st64()) {
            DISPATCH_NR(c->NR, {
                best_update_kernel<double, NR_><<<g, 256, 0, c->stream>>>(
                    c->improved, static_cast<const double*>(c->Rs), c->sig,
                    static_cast<double*>(c->bestR), c->bestS, c->ldN, c->B);
            });
        } else {
            DISPATCH_NR(c->NR, {
                best_update_kernel<float, NR_><<<g, 256, 0, c->stream>>>(
                    c->improved, static_cast<const float*>(c->Rs), c->sig,
                    static_cast<float*>(c->bestR), c->bestS, c->ldN, c->B);
            });
        }
        CK(cudaGetLastError());
    }
    return 0;
}

int check_ready(cimcs_ctx* c, int R) {
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    if (!c->built) return fail(CIMCS_INPUT_ERROR, "coupling not built (cimcs_build_coupling)");
    if (R < 1 || R > 16) return fail(CIMCS_INPUT_ERROR, "R must be in [1, 16]");
    return 0;
}

int validate(const cimcs_hyper* h) {
    if (!h) return fail(CIMCS_CONFIG_ERROR, "null hyper-parameters");
    if (!(h->dt > 0)) return fail(CIMCS_CONFIG_ERROR, "dt must be > 0");
    if (h->n_steps < 1) return fail(CIMCS_CONFIG_ERROR, "n_steps must be >= 1");
    if (!(h->tau > 0)) return fail(CIMCS_CONFIG_ERROR, "tau must be > 0");
    if (h->g2 < 0) return fail(CIMCS_CONFIG_ERROR, "g2 must be >= 0");
    if (h->eta_init < h->eta_end || h->eta_end < 0)
        return fail(CIMCS_CONFIG_ERROR, "need eta_init >= eta_end >= 0");
    if (h->velo < 1) return fail(CIMCS_CONFIG_ERROR, "velo must be >= 1");
    if (h->pump_kind != CIMCS_PUMP_SIGMOID && h->pump_kind != CIMCS_PUMP_LINEAR)
        return fail(CIMCS_CONFIG_ERROR, "pump_kind must be sigmoid or linear");
    return 0;
}

int upload_pump(cimcs_ctx* c, const cimcs_hyper* hp) {
    const std::vector<double> p = pump_table(hp);
    for (double v : p)
        if (!std::isfinite(v)) return fail(CIMCS_INPUT_ERROR, "mfz_step: non-finite pump");
    if (c->pump_cap < hp->n_steps) {
        // cached graphs bake the pump pointer: drop them with the old buffer
        drop_graphs(c);
        if (c->pump) cudaFree(c->pump);
        c->pump = nullptr;
        if (int rc = dalloc(c, &c->pump, (size_t)hp->n_steps * 8)) return rc;
        c->pump_cap = hp->n_steps;
    }
    if (int rc_ = copy_sync(c, c->pump, p.data(), (size_t)hp->n_steps * 8, cudaMemcpyHostToDevice)) return rc_;
    return 0;
}

int set_alt(cimcs_ctx* c, const AltParams& ap) {
    CK(cudaMemcpyAsync(c->alt, &ap, sizeof(AltParams), cudaMemcpyHostToDevice, c->stream));
    return 0;
}

// Host c0 generator pool: trajectory streams split contiguously over threads.
void gen_c0(std::vector<HostRng>& rngs, int N, double* out, int threads) {
    const int nt = (int)rngs.size();
    threads = std::max(1, std::min(threads, nt));
    auto work = [&](int t0, int t1) {
        for (int t = t0; t < t1; ++t) {
            double* o = out + (size_t)t * N;
            for (int i = 0; i < N; ++i) o[i] = 0.01 * rngs[t].gauss();  // init_mfz :27
        }
    };
    if (threads == 1) {
        work(0, nt);
        return;
    }
    std::vector<std::thread> pool;
    const int per = (nt + threads - 1) / threads;
    for (int k = 0; k < threads; ++k) {
        const int t0 = k * per, t1 = std::min(nt, t0 + per);
        if (t0 < t1) pool.emplace_back(work, t0, t1);
    }
    for (auto& th : pool) th.join();
}

// Host -> device upload of B variable-size pieces through two pinned slots:
// host threads pack a slot while the DMA engine drains the other.
template <class SizeF, class SrcF, class DstF>
int staged_upload(cimcs_ctx* c, int B, SizeF size_of, SrcF src_of, DstF dst_of) {
    const size_t slot = (size_t)64 << 20;
    if (c->pin_bytes < slot) {
        if (c->pin) cudaFreeHost(c->pin);
        c->pin = nullptr;
        CK(cudaMallocHost(&c->pin, 2 * slot));
        c->pin_bytes = slot;
    }
    cudaEvent_t done[2];
    CK(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    std::unique_ptr<cudaEvent_t[], void (*)(cudaEvent_t*)> guard(done, [](cudaEvent_t* e) {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
    });
    const int threads = std::max(1, std::min(c->host_threads, 16));
    int k = 0;
    char* base = reinterpret_cast<char*>(c->pin);
    for (int b = 0; b < B; ++b) {
        const size_t n = size_of(b);
        const char* src = src_of(b);
        char* dst = dst_of(b);
        for (size_t off = 0; off < n; off += slot, ++k) {
            const size_t len = std::min(slot, n - off);
            char* buf = base + (size_t)(k & 1) * slot;
            if (k >= 2) CK(cudaEventSynchronize(done[k & 1]));
            const int nt = len >= ((size_t)8 << 20) ? threads : 1;
            if (nt == 1) {
                std::memcpy(buf, src + off, len);
            } else {
                std::vector<std::thread> pool;
                const size_t per = (len + nt - 1) / nt;
                for (int t = 0; t < nt; ++t) {
                    const size_t o = (size_t)t * per;
                    if (o >= len) break;
                    pool.emplace_back([=] { std::memcpy(buf + o, src + off + o, std::min(per, len - o)); });
                }
                for (auto& th : pool) th.join();
            }
            CK(cudaMemcpyAsync(dst + off, buf, len, cudaMemcpyHostToDevice, c->stream));
            CK(cudaEventRecord(done[k & 1], c->stream));
        }
    }
    // the slots are reused by the next upload: drain them before returning
    if (k >= 1) CK(cudaEventSynchronize(done[(k - 1) & 1]));
    if (k >= 2) CK(cudaEventSynchronize(done[k & 1]));
    return 0;
}

struct Graph {
    cudaGraphExec_t exec = nullptr;
    ~Graph() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

template <typename F>
int capture(cimcs_ctx* c, Graph& g, F&& body) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = body();
    cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
    if (rc) {
        if (e == cudaSuccess) cudaGraphDestroy(graph);
        return rc;
    }
    CK(e);
    CK(cudaGraphInstantiate(&g.exec, graph, 0));
    cudaGraphDestroy(graph);
    return 0;
}

struct Events {
    std::vector<cudaEvent_t> ev;
    explicit Events(size_t n) : ev(n, nullptr) {
        for (auto& e : ev) cudaEventCreate(&e);
    }
    ~Events() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
    float ms(size_t a, size_t b) const {
        float t = 0.f;
        cudaEventElapsedTime(&t, ev[a], ev[b]);
        return t;
    }
};

// ------------------------------------------------------ Positive-P backend
constexpr int kPpChunk = 64;  // steps of unit normals per host -> device chunk

int ensure_pp(cimcs_ctx* c) {  // outside any capture
    if (c->mri)
        return fail(CIMCS_CONFIG_ERROR, "pp backend: not on matrix-free MRI problems (fp32 MFZ only)");
    if (c->tc)
        return fail(CIMCS_CONFIG_ERROR,
                    "pp backend: use an fp64 context or tensor_cores=0 (the tcgen05 epilogues "
                    "implement the MFZ update only)");
    if (c->world > 1)
        return fail(CIMCS_CONFIG_ERROR, "pp backend is not supported on row-sharded contexts");
    const size_t n = c->state_elems();
    if (!c->Pn) {
        int rc;
        if ((rc = dalloc(c, &c->Pn, n * c->elt())) || (rc = dalloc(c, &c->Pm, n * c->elt())) ||
            (rc = dalloc(c, &c->MT, n * c->elt())))
            return rc;
    }
    const size_t nz = (size_t)kPpChunk * n;
    if (c->nz_elems < nz) {
        for (int k = 0; k < 2; ++k) {
            if (c->nzd[k]) cudaFree(c->nzd[k]);
            if (c->nzh[k]) cudaFreeHost(c->nzh[k]);
            c->nzd[k] = c->nzh[k] = nullptr;
        }
        for (int k = 0; k < 2; ++k) {
            if (int rc = dalloc(c, &c->nzd[k], nz * 8)) return rc;
            CK(cudaMallocHost(&c->nzh[k], nz * 8));
            std::memset(c->nzh[k], 0, nz * 8);  // padded slots stay zero
        }
        c->nz_elems = nz;
    }
    return 0;
}

// kc steps of unit normals per trajectory (make_noise_draw, solver_pp.cpp:9: N
// deviates per step from the trial stream), device layout [kc][B][ldN][NR]
void gen_noise(cimcs_ctx* c, std::vector<HostRng>& rngs, int Rreal, int kc, double* out) {
    const int nt = (int)rngs.size();
    const size_t S = c->state_elems();
    auto work = [&](int t0, int t1) {
        for (int t = t0; t < t1; ++t) {
            const int b = t / Rreal, r = t % Rreal;
            for (int k = 0; k < kc; ++k) {
                double* o = out + (size_t)k * S + ((size_t)b * c->ldN) * c->NR + r;
                for (int i = 0; i < c->N; ++i) o[(size_t)i * c->NR] = rngs[t].gauss();
            }
        }
    };
    const int threads = std::max(1, std::min(c->host_threads, nt));
    if (threads == 1) {
        work(0, nt);
        return;
    }
    std::vector<std::thread> pool;
    const int per = (nt + threads - 1) / threads;
    for (int k = 0; k < threads; ++k) {
        const int t0 = k * per, t1 = std::min(nt, t0 + per);
        if (t0 < t1) pool.emplace_back(work, t0, t1);
    }
    for (auto& th : pool) th.join();
}

template <typename T>
int pp_init_T(cimcs_ctx* c, int Rreal, const double* nz0, const StepScalars& s) {
    const int g = grid_for(c->state_elems());
    DISPATCH_NR(c->NR, {
        init_pp_kernel<T, NR_><<<g, 256, 0, c->stream>>>(
            Rreal, c->N, c->ldN, c->B, static_cast<const T*>(c->Rs), static_cast<T*>(c->C),
            static_cast<T*>(c->E), static_cast<T*>(c->Pn), static_cast<T*>(c->Pm),
            static_cast<T*>(c->MT), static_cast<T*>(c->W0), c->fail_gstep, c->minE, nz0,
            s.pp_scale, s.rt);
    });
    CK(cudaGetLastError());
    return 0;
}

// One Positive-P CIM call (run_pp, solver_pp.cpp:100-132) for all trajectories.
// The unit normals are drawn on the host from each trajectory's reference
// stream (bit-exact) and uploaded in chunks of kPpChunk steps while the GPU
// integrates the previous chunk.  Host-driven (not captured).  Afterwards C
// holds mu and MT the last measured amplitude (the sigma source, run_pp :126-129).
int run_pp_cim(cimcs_ctx* c, int Rreal, const StepScalars& s, const cimcs_hyper* hp,
               std::vector<HostRng>& rngs) {
    const int n_steps = hp->n_steps, K = std::min(kPpChunk, n_steps);
    const int nch = (n_steps + K - 1) / K;
    const size_t S = c->state_elems();
    Events cp(2);
    auto stage = [&](int ch) -> int {
        const int sl = ch & 1, kc = std::min(K, n_steps - ch * K);
        gen_noise(c, rngs, Rreal, kc, c->nzh[sl]);
        CK(cudaMemcpyAsync(c->nzd[sl], c->nzh[sl], (size_t)kc * S * 8, cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaEventRecord(cp.ev[sl], c->stream));
        return 0;
    };
    int rc = stage(0);
    if (!rc && nch > 1) rc = stage(1);
    if (!rc)
        rc = c->st64() ? pp_init_T<double>(c, Rreal, c->nzd[0], s)
                                   : pp_init_T<float>(c, Rreal, c->nzd[0], s);
    GemvArgs a = base_args(c, s);
    a.pump = c->pump;
    a.Hdbg = nullptr;
    a.Pn = c->Pn;
    a.Pm = c->Pm;
    a.MT = c->MT;
    for (int ch = 0; ch < nch && !rc; ++ch) {
        const int k0 = ch * K, kc = std::min(K, n_steps - k0);
        for (int k = k0; k < k0 + kc && !rc; ++k) {
            a.step = k;
            a.Win = (k & 1) ? c->W1 : c->W0;
            a.Wout = (k & 1) ? c->W0 : c->W1;
            a.nz = c->nzd[ch & 1] + (size_t)(k - k0) * S;
            a.nz_next = k + 1 >= n_steps ? a.nz
                        : k + 1 < k0 + kc ? a.nz + S
                                          : c->nzd[(ch + 1) & 1];
            rc = launch_gemv(c, EPI_STEP_PP, a);
        }
        if (!rc && ch + 2 < nch) {
            CK(cudaEventSynchronize(cp.ev[ch & 1]));  // its pinned slot has been copied
            rc = stage(ch + 2);
        }
    }
    // the next call refills both pinned slots at once: the copies still queued
    // behind this call's kernels must have read them first
    CK(cudaEventSynchronize(cp.ev[0]));
    CK(cudaEventSynchronize(cp.ev[1]));
    return rc;
}

// C = the measured amplitude (CimCallResult::amplitude of the PP backend), so the
// support / refit path (support_kernel: sigma = C > 0) serves both backends
int pp_amplitude_to_c(cimcs_ctx* c) {
    CK(cudaMemcpyAsync(c->C, c->MT, c->state_elems() * c->elt(), cudaMemcpyDeviceToDevice,
                       c->stream));
    return 0;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

int cimcs_abi_version(void) { return CIMCS_ABI_VERSION; }
const char* cimcs_last_error(void) { return g_err.c_str(); }

void cimcs_hyper_default(cimcs_hyper* h) {
    h->g2 = 1e-7;
    h->j = 1.0;
    h->K = 1.0;
    h->beta = 0.2;
    h->tau = 1.0;
    h->dt = 0.02;
    h->n_steps = 1000;
    h->p_thr = 1.0;
    h->d = 0.4;
    h->eta_init = 0.8;
    h->eta_end = 0.18;
    h->velo = 51;
    h->dt_c = 0.1;
    h->jacobi_iters = 100;
    h->cg_max_iters = 10000;
    h->cg_tol = 1e-10;
    h->gamma = 1e-4;
    h->mfz_loss_minus_j = 0;
    h->mu_abort = 100.0;
    h->pump_kind = CIMCS_PUMP_SIGMOID;
    h->pump_end = 1.2;
}

int cimcs_hyper_validate(const cimcs_hyper* h) { return validate(h); }
uint64_t cimcs_mix_seed(uint64_t base, uint64_t salt) { return mix_seed(base, salt); }

int cimcs_gemv_order(int dtype, int32_t* nseg, int32_t* gran) {
    (void)dtype;
    if (nseg) *nseg = kSeg;
    if (gran) *gran = kGran;
    return 0;
}

// The fp64 contraction order of the resident problem set (ORC_CANON's
// (nseg, gran)): the DMMA symmetric path sums 512-column segments, the grid and
// cluster kernels 8 interleaved segments of 8-column granules.
int cimcs_canon_order(const cimcs_ctx* c, int32_t* nseg, int32_t* gran) {
    if (!c || c->B < 1) return fail(CIMCS_INPUT_ERROR, "no problems set");
    const bool s64 = c->sym64;
    if (nseg) *nseg = s64 ? c->nSB6 : kSeg;
    if (gran) *gran = s64 ? kT6Seg : kGran;
    return 0;
}

int cimcs_gen_dims(int32_t N, double alpha, double a, int32_t* M, int32_t* K) {
    int m = 0, k = 0;
    if (gen_dims(N, alpha, a, &m, &k)) return fail(CIMCS_INPUT_ERROR, "gen_instance: bad dims");
    if (M) *M = m;
    if (K) *K = k;
    return 0;
}

// ------------------------------------------------ bundles and CSV (io.hpp)
int cimcs_format_double(double v, char* buf, int32_t cap) {
    const std::string s = cimcs_io::fmt_double(v);
    if (!buf || cap < (int32_t)s.size() + 1) return fail(CIMCS_INPUT_ERROR, "format_double: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

uint64_t cimcs_fnv1a64(const char* bytes, uint64_t n) {
    return cimcs_io::fnv1a(reinterpret_cast<const unsigned char*>(bytes), (size_t)n);
}

int cimcs_save_instance(const char* dir, int32_t N, int32_t M, const double* A, const double* y,
                        const double* x_true, const int32_t* xi_true, double a, double alpha,
                        double nu, uint64_t seed) {
    if (!dir || N < 1 || M < 1 || !A || !y) return fail(CIMCS_INPUT_ERROR, "save_instance: bad arguments");
    cimcs_io::Meta m;
    m.N = N;
    m.M = M;
    m.a = a;
    m.alpha = alpha;
    m.nu = nu;
    m.seed = seed;
    std::string err;
    if (!cimcs_io::save_bundle(dir, m, A, y, x_true, xi_true, &err)) return fail(CIMCS_INPUT_ERROR, err);
    return 0;
}

int cimcs_load_instance(const char* dir, int32_t* N, int32_t* M, int32_t* has_truth, double* a,
                        double* alpha, double* nu, uint64_t* seed, double* A, double* y,
                        double* x_true, int32_t* xi_true) {
    if (!dir || !N || !M) return fail(CIMCS_INPUT_ERROR, "load_instance: bad arguments");
    cimcs_io::Meta m;
    bool truth = false;
    std::string err;
    if (!cimcs_io::load_meta(dir, &m, &truth, &err)) return fail(CIMCS_INPUT_ERROR, err);
    if (A) {  // phase 2: the caller sized the arrays from phase 1
        if (*N != m.N || *M != m.M) return fail(CIMCS_INPUT_ERROR, "load_instance: size mismatch");
        if (!y || !cimcs_io::load_arrays(dir, m, A, y, truth ? x_true : nullptr,
                                         truth ? xi_true : nullptr, &err))
            return fail(CIMCS_INPUT_ERROR, err.empty() ? "load_instance: bad arguments" : err);
    }
    *N = m.N;
    *M = m.M;
    if (has_truth) *has_truth = truth ? 1 : 0;
    if (a) *a = m.a;
    if (alpha) *alpha = m.alpha;
    if (nu) *nu = m.nu;
    if (seed) *seed = m.seed;
    return 0;
}

struct cimcs_csv : cimcs_io::Csv {};

int cimcs_csv_open(const char* path, const char* const* comments, int32_t ncomments,
                   const char* const* columns, int32_t ncols, cimcs_csv** out) {
    if (!path || !out || ncols < 0 || ncomments < 0) return fail(CIMCS_INPUT_ERROR, "csv_open: bad arguments");
    auto* w = new cimcs_csv();
    w->path = path;
    w->ncols = (size_t)ncols;
    for (int k = 0; k < ncomments; ++k) (w->buf += "# ") += std::string(comments[k]) + "\n";
    for (int k = 0; k < ncols; ++k) {
        if (k) w->buf += ',';
        w->buf += columns[k];
    }
    w->buf += '\n';
    *out = w;
    return 0;
}

int cimcs_csv_row(cimcs_csv* w, const char* const* cells, int32_t n) {
    if (!w || n < 0 || (size_t)n != w->ncols) return fail(CIMCS_INPUT_ERROR, "CsvWriter: cell count mismatch");
    for (int k = 0; k < n; ++k) {
        if (k) w->buf += ',';
        w->buf += cells[k];
    }
    w->buf += '\n';
    return 0;
}

int cimcs_csv_close(cimcs_csv* w) {
    if (!w) return 0;
    std::error_code ec;
    const std::filesystem::path p(w->path);
    std::filesystem::create_directories(p.parent_path().empty() ? "." : p.parent_path(), ec);
    std::string err;
    const bool ok = cimcs_io::put_file(p, w->buf, &err);
    delete w;
    return ok ? 0 : fail(CIMCS_INPUT_ERROR, err);
}

int cimcs_gen_instance(int32_t N, double alpha, double a, double nu, uint64_t seed, double* A,
                       double* y, double* x_true, int32_t* xi_true) {
    if (gen_instance(N, alpha, a, nu, seed, A, y, x_true, xi_true))
        return fail(CIMCS_INPUT_ERROR, "gen_instance: bad arguments");
    return 0;
}

int cimcs_gen_instances(int32_t B, int32_t N, const double* alpha, const double* a,
                        const double* nu, const uint64_t* seeds, double* const* A,
                        double* const* y, double* const* x_true, int32_t* const* xi_true,
                        int32_t threads) {
    std::atomic<int> next{0}, bad{0};
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    // fewer instances than threads: the spare threads transform each instance's A
    const int inner = std::max(1, threads / std::max(1, B));
    auto work = [&] {
        for (int b = next.fetch_add(1); b < B; b = next.fetch_add(1))
            if (gen_instance(N, alpha[b], a[b], nu[b], seeds[b], A[b], y[b], x_true[b],
                             xi_true[b], inner))
                bad = 1;
    };
    threads = std::max(1, std::min<int>(threads, B));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    return bad ? fail(CIMCS_INPUT_ERROR, "gen_instance: bad arguments") : 0;
}

int cimcs_create(int32_t device, int32_t dtype, cimcs_ctx** out) {
    if (!out) return fail(CIMCS_INPUT_ERROR, "null out");
    if (dtype != CIMCS_F32 && dtype != CIMCS_F64) return fail(CIMCS_CONFIG_ERROR, "bad dtype");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CIMCS_CONFIG_ERROR, "bad device");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(CIMCS_CUDA_ERROR, "libcimcs_gpu is built for sm_100a (B200) only");
    auto* c = new cimcs_ctx();
    c->num_sms = prop.multiProcessorCount;
    c->device = device;
    c->dtype = dtype;
    c->host_threads = std::max(1u, std::thread::hardware_concurrency());
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return fail(CIMCS_CUDA_ERROR, "stream create failed");
    }
    if (dalloc(c, &c->alt, sizeof(AltParams)) || dalloc(c, &c->err, 16)) {
        delete c;
        return CIMCS_CUDA_ERROR;
    }
    *out = c;
    return 0;
}

int cimcs_nccl_unique_id(uint8_t* out, int32_t nbytes) {
    if (!out || nbytes < (int32_t)sizeof(ncclUniqueId))
        return fail(CIMCS_INPUT_ERROR, "need a 128-byte buffer");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return 0;
}

int cimcs_create_sharded(int32_t device, int32_t dtype, int32_t world, int32_t rank,
                         const uint8_t* nccl_id, cimcs_ctx** out) {
    if (world < 1 || rank < 0 || rank >= world || !nccl_id)
        return fail(CIMCS_CONFIG_ERROR, "bad world/rank/id");
    if (int rc = cimcs_create(device, dtype, out)) return rc;
    cimcs_ctx* c = *out;
    c->world = c->sh_world = world;
    c->rank = c->sh_rank = rank;
    c->sharded = c->sh_rows = true;
    if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        const ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            cimcs_destroy(c);
            *out = nullptr;
            return fail(CIMCS_CUDA_ERROR, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
    }
    return 0;
}

void cimcs_destroy(cimcs_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    free_problems(c);
    if (c->stage) cudaFree(c->stage);
    if (c->stage_i) cudaFree(c->stage_i);
    if (c->alt) cudaFree(c->alt);
    if (c->err) cudaFree(c->err);
    if (c->pump) cudaFree(c->pump);
    if (c->hist) cudaFree(c->hist);
    if (c->pin) cudaFreeHost(c->pin);
    if (c->pin_c0) cudaFreeHost(c->pin_c0);
    if (c->dc0) cudaFree(c->dc0);
    drop_graphs(c);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->side) cudaStreamDestroy(c->side);
    cudaStreamDestroy(c->stream);
    delete c;
}

int cimcs_set_option(cimcs_ctx* c, const char* key, int64_t v) {
    if (!c || !key) return fail(CIMCS_INPUT_ERROR, "null argument");
    const std::string k(key);
    if (k == "host_threads") c->host_threads = (int)std::max<int64_t>(1, v);
    else if (k == "use_graphs") c->use_graphs = v != 0;
    else if (k == "gram_tc") c->gram_tc = v > 0 ? 1 : (v < 0 ? -1 : 0);
    else if (k == "kernel_timing") {
        c->kernel_timing = v != 0;
        c->timing.tile_kernel_ms = 0.0;
        c->timing.tile_kernel_launches = 0;
        drop_graphs(c);
    } else if (k == "tile_shard") {
        if (c->B > 0) return fail(CIMCS_CONFIG_ERROR, "set tile_shard before set_problems");
        c->tshard_opt = v != 0 ? 1 : 0;
    } else if (k == "mri_cluster") {
        c->mri_cluster = v != 0;
        drop_graphs(c);
    } else if (k == "gram_l2") {
        c->gram_l2 = v != 0;
        drop_graphs(c);
    } else if (k == "pdl") {
        c->use_pdl = v != 0;
        drop_graphs(c);
    }
    else if (k == "cluster_loop") {
        c->use_cluster = v != 0;
        drop_graphs(c);
    }
    else if (k == "tensor_cores") {
        if (c->B > 0) return fail(CIMCS_CONFIG_ERROR, "set tensor_cores before set_problems");
        c->want_tc = v != 0;
    } else if (k == "sym64") {
        if (c->B > 0) return fail(CIMCS_CONFIG_ERROR, "set sym64 before set_problems");
        c->want_sym64 = v != 0;
    }
    else return fail(CIMCS_CONFIG_ERROR, "unknown option " + k);
    return 0;
}

// Problem-set layout decisions and device allocations shared by set_problems
// (host instances) and set_generated_problems (instances generated on the GPU).
int prepare_problems(cimcs_ctx* c, int32_t B, int32_t N, const int32_t* M, bool truth) {
    CK(cudaSetDevice(c->device));
    // same shapes as the resident problem set: keep every device allocation
    const bool reuse = c->dA && c->B == B && c->N == N && c->has_truth == truth &&
                       std::equal(c->M.begin(), c->M.end(), M) && (int)c->M.size() == B &&
                       c->want_tc == c->tc_requested && !c->sh_rows;
    if (!reuse) free_problems(c);
    c->built = false;
    c->tc_requested = c->want_tc;
    c->B = B;
    c->N = N;
    c->ldN = (N + 31) / 32 * 32;
    c->ldJ = (N + kChunk - 1) / kChunk * kChunk;
    // fp32 tensor cores = the symmetric-tile path, for N above the cluster-loop
    // range, unsharded or tile-sharded; everything else runs on CUDA cores
    c->tc = c->dtype == CIMCS_F32 && c->want_tc && N > kClMaxN && (!c->sh_rows || c->tshard_opt);
    c->RB = c->tc ? kTcRows : (c->st64() ? row_block<double>() : row_block<float>());
    c->row0 = 0;
    c->row1 = N;
    c->rb0 = 0;
    c->nRB = (N + c->RB - 1) / c->RB;
    // sharded contexts on the symmetric path split gram TILES (replicated
    // state, one all-reduce per step); otherwise gram ROWS (all-gather of w)
    c->world = c->sh_rows ? c->sh_world : 1;
    c->rank = c->sh_rows ? c->sh_rank : 0;
    c->sharded = c->sh_rows;
    c->tshard = c->sh_rows && c->tc;
    c->tworld = c->tshard ? c->world : 1;
    c->trank = c->tshard ? c->rank : 0;
    if (c->tshard) {
        c->world = 1;
        c->rank = 0;
        c->sharded = false;
    }
    if (c->sharded) {
        // row sharding: equal slices of whole 128-row tiles (sharding.row_shard)
        const int per = (N + c->world * 128 - 1) / (c->world * 128) * 128;
        c->ldN = c->ldJ = per * c->world;
        c->row0 = std::min(N, c->rank * per);
        c->row1 = std::min(N, c->row0 + per);
        c->rb0 = c->row0 / c->RB;
        c->nRB = c->row1 > c->row0 ? (c->row1 - c->row0 + c->RB - 1) / c->RB : 0;
    }
    c->nch = c->ldJ / kTcChunk;
    c->sym = c->tc;
    // fp64: DMMA symmetric tiles for unsharded contexts above the cluster range
    // (64-row blocks = row_block<double>(), 512 x 512 items)
    c->sym64 = c->dtype == CIMCS_F64 && c->want_sym64 && !c->sh_rows && N > kClMaxN;
    c->nRB6 = c->sym64 ? (N + kT6 - 1) / kT6 : 0;
    c->ntri6 = c->nRB6 * (c->nRB6 + 1) / 2;
    c->nSB6 = (c->nRB6 + kS6 - 1) / kS6;
    c->ntri = c->sym ? c->nRB * (c->nRB + 1) / 2 : 0;
    c->nSB = (c->nRB + kSyS - 1) / kSyS;
    if (c->tshard) tile_shard(c->nRB, c->tworld, c->trank, &c->sP0, &c->sP1);
    c->M.assign(M, M + B);
    c->Mmax = *std::max_element(c->M.begin(), c->M.end());
    c->has_truth = truth;
    const size_t astride = (size_t)c->Mmax * N;
    int rc;
    if (!reuse && ((rc = dalloc(c, &c->dA, (size_t)B * astride * 8)) ||
                   (rc = dalloc(c, &c->dy, (size_t)B * c->Mmax * 8)) ||
                   (rc = dalloc(c, &c->dM, (size_t)B * 4))))
        return rc;
    if (truth && !c->dx) {
        if ((rc = dalloc(c, &c->dx, (size_t)B * c->ldN * 8)) ||
            (rc = dalloc(c, &c->dxi, (size_t)B * c->ldN)))
            return rc;
    }
    return 0;
}

// ---------------------------------------- counter-based device generator
// SURVEY 8f row 4, the documented deviation: config-4-scale instances (A alone
// is 5e9 normals) drawn on the GPU from Philox4x32-10 streams instead of the
// reference's single sequential mt19937_64 stream (datagen.cpp:15-55), whose
// bit-exact reproduction needs that stream's order and glibc's log/cos.  Same
// recipe and shapes: A_kr = N(0,1)/sqrt(M) (draw index k N + r, stream 0),
// x_r = N(0,1) (stream 1), support = the K positions with the smallest
// Philox keys (stream 2, a uniform K-subset), y = A (xi . x) + nu N(0,1)
// (stream 3) summed over the support in ascending order as gen_instance does.
// Different numbers from the reference's instances -- never used for parity.
__host__ __device__ inline void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
        const uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
        const uint32_t n0 = h1 ^ c[1] ^ k0, n2 = h0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = l1;
        c[2] = n2;
        c[3] = l0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}
__host__ __device__ inline void philox_u64x2(uint64_t seed, uint32_t stream, uint64_t idx,
                                             uint64_t* a, uint64_t* b) {
    uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), stream, 0x5eedu};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    *a = (uint64_t)c[0] | ((uint64_t)c[1] << 32);
    *b = (uint64_t)c[2] | ((uint64_t)c[3] << 32);
}
__device__ inline double philox_normal(uint64_t seed, uint32_t stream, uint64_t idx) {
    uint64_t a, b;
    philox_u64x2(seed, stream, idx, &a, &b);
    const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53, u2 = (double)(b >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);  // rng.hpp's Box-Muller form
}
__global__ void devgen_a_kernel(double* A, int M, int N, uint64_t seed, double col_std) {
    const size_t total = (size_t)M * N;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t r = t / M, k = t % M;  // column-major storage, row-major draw index
        A[t] = col_std * philox_normal(seed, 0, (uint64_t)k * N + r);
    }
}
__global__ void devgen_x_kernel(double* x, int N, uint64_t seed) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x)
        x[r] = philox_normal(seed, 1, r);
}
__global__ void devgen_y_kernel(const double* __restrict__ A, int M, const int* __restrict__ supp,
                                int K, const double* __restrict__ x, double nu, uint64_t seed,
                                double* y) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < M; k += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < K; ++s) acc = acc + A[(size_t)supp[s] * M + k] * x[supp[s]];
        y[k] = acc + nu * philox_normal(seed, 3, k);
    }
}

int cimcs_set_generated_problems(cimcs_ctx* c, int32_t B, int32_t N, const double* alpha,
                                 const double* a, const double* nu, const uint64_t* seeds) {
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    if (B < 1 || N < 1 || !alpha || !a || !nu || !seeds)
        return fail(CIMCS_INPUT_ERROR, "set_generated_problems: bad arguments");
    std::vector<int32_t> M(B), K(B);
    for (int b = 0; b < B; ++b)
        if (gen_dims(N, alpha[b], a[b], &M[b], &K[b]) || nu[b] < 0.0)
            return fail(CIMCS_INPUT_ERROR, "gen_instance: bad arguments");
    if (int rc = prepare_problems(c, B, N, M.data(), true)) return rc;
    const size_t astride = (size_t)c->Mmax * N;
    int* dsupp = nullptr;
    if (int rc = dalloc(c, &dsupp, (size_t)N * 4)) return rc;
    std::unique_ptr<int, decltype(&cudaFree)> g(dsupp, &cudaFree);
    CK(cudaMemsetAsync(c->dx, 0, (size_t)B * c->ldN * 8, c->stream));
    CK(cudaMemsetAsync(c->dxi, 0, (size_t)B * c->ldN, c->stream));
    CK(cudaMemcpyAsync(c->dM, M.data(), (size_t)B * 4, cudaMemcpyHostToDevice, c->stream));
    for (int b = 0; b < B; ++b) {
        // support: the K smallest stream-2 keys (host, O(N log N))
        std::vector<std::pair<uint64_t, int>> key(N);
        for (int r = 0; r < N; ++r) {
            uint64_t k0, k1;
            philox_u64x2(seeds[b], 2, (uint64_t)r, &k0, &k1);
            key[r] = {k0, r};
        }
        std::partial_sort(key.begin(), key.begin() + K[b], key.end());
        std::vector<int> supp(K[b]);
        for (int s = 0; s < K[b]; ++s) supp[s] = key[s].second;
        std::sort(supp.begin(), supp.end());
        std::vector<int8_t> xi8((size_t)c->ldN, 0);
        for (int r : supp) xi8[r] = 1;
        double* Ab = c->dA + (size_t)b * astride;
        double* xb = c->dx + (size_t)b * c->ldN;
        devgen_a_kernel<<<8 * c->num_sms, 256, 0, c->stream>>>(Ab, M[b], N, seeds[b],
                                                              1.0 / std::sqrt((double)M[b]));
        devgen_x_kernel<<<(N + 255) / 256, 256, 0, c->stream>>>(xb, N, seeds[b]);
        CK(cudaMemcpyAsync(c->dxi + (size_t)b * c->ldN, xi8.data(), xi8.size(),
                           cudaMemcpyHostToDevice, c->stream));
        if (K[b] > 0)
            CK(cudaMemcpyAsync(dsupp, supp.data(), (size_t)K[b] * 4, cudaMemcpyHostToDevice,
                               c->stream));
        devgen_y_kernel<<<(M[b] + 255) / 256, 256, 0, c->stream>>>(
            Ab, M[b], dsupp, K[b], xb, nu[b], seeds[b], c->dy + (size_t)b * c->Mmax);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));  // xi8 / supp are reused next instance
    }
    return 0;
}

// the resident instance b back on the host (A column-major M x N; truth when set)
int cimcs_get_instance(cimcs_ctx* c, int32_t b, double* A, double* y, double* x_true,
                       int32_t* xi_true) {
    if (!c || b < 0 || b >= c->B || c->mri || !c->dA) return fail(CIMCS_INPUT_ERROR, "bad instance");
    CK(cudaStreamSynchronize(c->stream));  // cudaMemcpy does not order against c->stream
    const int N = c->N, M = c->M[b];
    const size_t astride = (size_t)c->Mmax * N;
    if (A) {
        if (int rc_ = copy_sync(c, A, c->dA + (size_t)b * astride, (size_t)M * N * 8,
                                cudaMemcpyDeviceToHost))
            return rc_;
    }
    if (y) {
        if (int rc_ = copy_sync(c, y, c->dy + (size_t)b * c->Mmax, (size_t)M * 8,
                                cudaMemcpyDeviceToHost))
            return rc_;
    }
    if (c->has_truth && x_true)
        if (int rc_ = copy_sync(c, x_true, c->dx + (size_t)b * c->ldN, (size_t)N * 8, cudaMemcpyDeviceToHost)) return rc_;
    if (c->has_truth && xi_true) {
        std::vector<int8_t> t((size_t)N);
        if (int rc_ = copy_sync(c, t.data(), c->dxi + (size_t)b * c->ldN, (size_t)N, cudaMemcpyDeviceToHost)) return rc_;
        for (int i = 0; i < N; ++i) xi_true[i] = t[i];
    }
    return 0;
}

int cimcs_set_problems(cimcs_ctx* c, int32_t B, int32_t N, const int32_t* M,
                       const double* const* A, const double* const* y,
                       const double* const* x_true, const int32_t* const* xi_true) {
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    if (B < 1 || N < 1) return fail(CIMCS_INPUT_ERROR, "need B >= 1 and N >= 1");
    for (int b = 0; b < B; ++b)
        if (M[b] < 1 || !A[b] || !y[b]) return fail(CIMCS_INPUT_ERROR, "empty A");
    const bool truth = x_true != nullptr && xi_true != nullptr;
    if (int rc = prepare_problems(c, B, N, M, truth)) return rc;
    const size_t astride = (size_t)c->Mmax * N;
    // A and y go through a pinned double buffer filled by host threads
    // (pageable cudaMemcpy runs at a fraction of the link rate)
    if (int rc2 = staged_upload(c, B, [&](int b) { return (size_t)M[b] * N * 8; },
                                [&](int b) { return reinterpret_cast<const char*>(A[b]); },
                                [&](int b) { return reinterpret_cast<char*>(c->dA + (size_t)b * astride); }))
        return rc2;
    if (int rc2 = staged_upload(c, B, [&](int b) { return (size_t)M[b] * 8; },
                                [&](int b) { return reinterpret_cast<const char*>(y[b]); },
                                [&](int b) { return reinterpret_cast<char*>(c->dy + (size_t)b * c->Mmax); }))
        return rc2;
    CK(cudaMemcpyAsync(c->dM, M, (size_t)B * 4, cudaMemcpyHostToDevice, c->stream));
    if (c->has_truth) {
        std::vector<int8_t> xi8((size_t)B * c->ldN, 0);
        for (int b = 0; b < B; ++b) {
            CK(cudaMemcpyAsync(c->dx + (size_t)b * c->ldN, x_true[b], (size_t)N * 8,
                               cudaMemcpyHostToDevice, c->stream));
            for (int i = 0; i < N; ++i) {
                if (xi_true[b][i] != 0 && xi_true[b][i] != 1)
                    return fail(CIMCS_INPUT_ERROR, "xi_true must be 0/1");
                xi8[(size_t)b * c->ldN + i] = (int8_t)xi_true[b][i];
            }
        }
        CK(cudaMemcpyAsync(c->dxi, xi8.data(), xi8.size(), cudaMemcpyHostToDevice, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int cimcs_mri_lasso(cimcs_ctx* c, double lambda, int32_t max_iters, double tol, double step,
                    double* x_out, int32_t* iterations, double* objective) {
    if (!c || !c->mri || !c->built) return fail(CIMCS_INPUT_ERROR, "mri_lasso: no built MRI problem");
    if (lambda < 0.0) return fail(CIMCS_INPUT_ERROR, "lasso: lambda_l1 must be >= 0");
    if (!(step > 0.0)) return fail(CIMCS_INPUT_ERROR, "lasso: step must be > 0");
    if (max_iters < 0 || !x_out) return fail(CIMCS_INPUT_ERROR, "mri_lasso: bad arguments");
    CK(cudaSetDevice(c->device));
    const int N = c->N;
    float *zx = nullptr, *gzx = nullptr;
    LassoState* st = nullptr;
    int rc;
    if ((rc = dalloc(c, &zx, (size_t)N * 2 * 4)) || (rc = dalloc(c, &gzx, (size_t)N * 2 * 4)) ||
        (rc = dalloc(c, &st, sizeof(LassoState))))
        return rc;
    std::unique_ptr<float, decltype(&cudaFree)> g1(zx, &cudaFree), g2(gzx, &cudaFree);
    std::unique_ptr<LassoState, decltype(&cudaFree)> g3(st, &cudaFree);
    LassoState s0{1.0, 0.0, 0.0, 0, max_iters == 0 ? 1 : 0};
    CK(cudaMemsetAsync(zx, 0, (size_t)N * 2 * 4, c->stream));
    CK(cudaMemcpyAsync(st, &s0, sizeof s0, cudaMemcpyHostToDevice, c->stream));
    MriArgs ma{};
    ma.H = c->mH;
    ma.W = c->mW;
    ma.N = N;
    ma.NR = 2;
    ma.mask_br = c->dMaskBr;
    ma.tw = c->dTw;
    ma.L = c->mL;
    ma.gamma = 0.f;  // apply_fit: Re(A^H A), no smoothness (mri.cpp:299-301)
    ma.scale = 1.f / (float)N;
    ma.in = zx;
    ma.out = gzx;
    const size_t smem = mri_smem_bytes(c->mH, c->mW, c->mL);
    LassoState hs = s0;
    while (!hs.done) {
        for (int k = 0; k < 64; ++k) {  // device-side stop: launches after it return at once
            mri_kernel<<<2, kMriThreads, smem, c->stream>>>(ma, MRI_APPLY);
            lasso_kernel<<<1, kLassoThreads, 0, c->stream>>>(gzx, zx, static_cast<const float*>(c->dhz),
                                                             N, lambda, step, tol, max_iters, st);
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    std::vector<float> h((size_t)N * 2);
    if (int rc_ = copy_sync(c, h.data(), zx, h.size() * 4, cudaMemcpyDeviceToHost)) return rc_;
    for (int i = 0; i < N; ++i) x_out[i] = h[2 * i + 1];
    if (iterations) *iterations = hs.it;
    if (objective) *objective = hs.f;
    return 0;
}

int cimcs_tile_shard(int32_t nRB, int32_t world, int32_t rank, int32_t* P0, int32_t* P1) {
    if (nRB < 1 || world < 1 || rank < 0 || rank >= world || !P0 || !P1)
        return fail(CIMCS_INPUT_ERROR, "tile_shard: bad arguments");
    int a = 0, b = 0;
    tile_shard(nRB, world, rank, &a, &b);
    *P0 = a;
    *P1 = b;
    return 0;
}

int cimcs_make_mask(int32_t H, int32_t W, int32_t M, uint64_t seed, int32_t* out) {
    const long long N = (long long)H * W;
    if (H < 1 || W < 1) return fail(CIMCS_INPUT_ERROR, "make_mask: dims must be >= 1");
    if (M < 1 || M > N) return fail(CIMCS_INPUT_ERROR, "make_mask: M out of range");
    std::vector<int> pool((size_t)N);
    for (long long k = 0; k < N; ++k) pool[k] = (int)k;
    HostRng rng(seed);  // partial Fisher-Yates, mri.cpp:185-207
    for (int i = 0; i < M; ++i) {
        const long long pick = i + (long long)rng.uniform_below((uint64_t)(N - i));
        std::swap(pool[i], pool[pick]);
    }
    std::sort(pool.begin(), pool.begin() + M);
    std::copy(pool.begin(), pool.begin() + M, out);
    return 0;
}

int cimcs_set_mri_problem(cimcs_ctx* c, int32_t H, int32_t W, const double* target,
                          int32_t M, const int32_t* mask, double gamma, const double* x_true) {
    if (!c) return fail(CIMCS_INPUT_ERROR, "null context");
    auto pow2 = [](int v) { return v >= 1 && (v & (v - 1)) == 0; };
    if (!pow2(H) || !pow2(W)) return fail(CIMCS_INPUT_ERROR, "MriTransform: dimensions must be powers of two");
    if (H < 2 || W < 2 || H > kMriMaxLine || W > kMriMaxLine)
        return fail(CIMCS_INPUT_ERROR,
                    "MriTransform: need 2 <= H, W <= 128 (an FFT line lives in one warp's registers)");
    if (!(gamma >= 0.0)) return fail(CIMCS_INPUT_ERROR, "MriTransform: gamma must be >= 0");
    if (!target || !mask || M < 1) return fail(CIMCS_INPUT_ERROR, "MriTransform: mask indices must be unique and in range");
    std::vector<int> idx(mask, mask + M);
    std::sort(idx.begin(), idx.end());
    if (idx.front() < 0 || idx.back() >= H * W || std::adjacent_find(idx.begin(), idx.end()) != idx.end())
        return fail(CIMCS_INPUT_ERROR, "MriTransform: mask indices must be unique and in range");
    if (c->dtype != CIMCS_F32) return fail(CIMCS_CONFIG_ERROR, "matrix-free MRI problems run in fp32 contexts");
    if (c->world > 1 || c->sharded) return fail(CIMCS_CONFIG_ERROR, "matrix-free MRI problems are single-GPU");
    CK(cudaSetDevice(c->device));
    free_problems(c);
    const int N = H * W;
    c->built = false;
    c->mri = true;
    c->mH = H;
    c->mW = W;
    c->mL = std::max(H, W);
    c->mgamma = (float)gamma;
    c->B = 1;
    c->N = N;
    c->ldN = c->ldJ = (N + 31) / 32 * 32;
    c->tc = c->sym = c->sym64 = false;
    c->RB = kSyT;
    c->row0 = 0;
    c->row1 = N;
    c->rb0 = 0;
    c->nRB = (N + kSyT - 1) / kSyT;
    c->nSB = 1;
    c->ntri = 0;
    c->nch = 0;
    c->M.assign(1, M);
    c->Mmax = M;
    c->has_truth = x_true != nullptr;
    // mask in the bit-reversed coordinates of the DIF spectrum, twiddles, target
    auto rev = [](int v, int n) {
        int r = 0;
        for (int b = 1; b < n; b <<= 1, v >>= 1) r = (r << 1) | (v & 1);
        return r;
    };
    std::vector<unsigned char> full((size_t)N, 0), br((size_t)N, 0);
    for (int k : idx) full[k] = 1;
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) br[(size_t)i * W + j] = full[(size_t)rev(i, H) * W + rev(j, W)];
    std::vector<float2> tw(64);  // exp(-2 pi i k / 128): every line length divides 128
    for (int k = 0; k < 64; ++k) {
        const double a = -2.0 * M_PI * k / 128.0;
        tw[k] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    std::vector<float> tgt((size_t)N);
    for (int k = 0; k < N; ++k) tgt[k] = (float)target[k];
    int rc;
    if ((rc = dalloc(c, &c->dMaskBr, (size_t)N)) || (rc = dalloc(c, &c->dTw, tw.size() * sizeof(float2))) ||
        (rc = dalloc(c, &c->dTarget, (size_t)N * 4)))
        return rc;
    if (int rc_ = copy_sync(c, c->dMaskBr, br.data(), br.size(), cudaMemcpyHostToDevice)) return rc_;
    if (int rc_ = copy_sync(c, c->dTw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice)) return rc_;
    if (int rc_ = copy_sync(c, c->dTarget, tgt.data(), tgt.size() * 4, cudaMemcpyHostToDevice)) return rc_;
    static std::atomic<unsigned long long> attr{0};
    if (!(attr.load() >> c->device & 1ull)) {
        CK(cudaFuncSetAttribute(mri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)mri_smem_bytes(128, 128, 128)));
        CK(cudaFuncSetAttribute(mri_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)mri_cluster_smem_bytes(128, 128)));
        attr.fetch_or(1ull << c->device);
    }
    if (c->has_truth) {  // make_problem(t, &truth): xi = (x != 0) (mri.cpp:398-405)
        if ((rc = dalloc(c, &c->dx, (size_t)c->ldN * 8)) || (rc = dalloc(c, &c->dxi, (size_t)c->ldN)))
            return rc;
        std::vector<int8_t> xi8((size_t)c->ldN, 0);
        for (int i = 0; i < N; ++i) xi8[i] = x_true[i] != 0.0 ? 1 : 0;
        if (int rc_ = copy_sync(c, c->dx, x_true, (size_t)N * 8, cudaMemcpyHostToDevice)) return rc_;
        if (int rc_ = copy_sync(c, c->dxi, xi8.data(), xi8.size(), cudaMemcpyHostToDevice)) return rc_;
    }
    return 0;
}

int cimcs_build_coupling(cimcs_ctx* c) {
    if (!c || c->B < 1) return fail(CIMCS_INPUT_ERROR, "no problems set");
    CK(cudaSetDevice(c->device));
    if (c->mri) {  // hz = Re(A^H y) and diag(G) of the transform chain (mri.cpp:236-254)
        int rc;
        const size_t nv = (size_t)c->ldN;
        if (!c->dhz && (rc = dalloc(c, &c->dhz, nv * 4))) return rc;
        if (!c->dD && (rc = dalloc(c, &c->dD, nv * 4))) return rc;
        Events ev(2);
        cudaEventRecord(ev.ev[0], c->stream);
        CK(cudaMemsetAsync(c->dhz, 0, nv * 4, c->stream));
        CK(cudaMemsetAsync(c->dD, 0, nv * 4, c->stream));
        if ((rc = mri_launch(c, MRI_HZ, 1, 0, c->dTarget, static_cast<float*>(c->dhz))) ||
            (rc = mri_launch(c, MRI_DIAG, c->N, 0, nullptr, static_cast<float*>(c->dD))))
            return rc;
        cudaEventRecord(ev.ev[1], c->stream);
        CK(cudaStreamSynchronize(c->stream));
        c->timing.gram_ms = ev.ms(0, 1);
        c->timing.other_launches += 2;
        c->built = true;
        return 0;
    }
    const size_t es = c->elt();
    // gram bytes: symmetric fp16 hi/lo tiles, symmetric fp64 tiles, or CUDA-core panels
    const size_t gbytes = c->sym     ? (size_t)c->B * c->ntri * 2 * kSyPlaneBytes
                          : c->sym64 ? 16
                                     : (size_t)c->B * c->nRB * c->ldJ * c->RB * es;
    if (c->sym64 && !c->dG6) {
        if (int rc = dalloc(c, &c->dG6, (size_t)c->B * c->ntri6 * kT6TileBytes)) return rc;
    }
    const size_t nv = (size_t)c->B * c->ldN;
    int rc;
    if (!c->dG && (rc = dalloc(c, &c->dG, gbytes))) return rc;
    if (!c->dhz && (rc = dalloc(c, &c->dhz, nv * es))) return rc;
    if (!c->dD && (rc = dalloc(c, &c->dD, nv * es))) return rc;
    if (c->sym && !c->dSg && (rc = dalloc(c, &c->dSg, c->B * 4))) return rc;
    Events ev(2);
    cudaEventRecord(ev.ev[0], c->stream);
    CK(cudaMemsetAsync(c->dG, 0, gbytes, c->stream));
    const int nt = (c->N + kG2T - 1) / kG2T;
    const int bi0 = c->row0 / kG2T;
    const int nti = c->world == 1 ? nt : (c->row1 - c->row0 + kG2T - 1) / kG2T;
    const int mirror = c->world == 1 ? 1 : 0;
    const size_t astride = (size_t)c->Mmax * c->N;
    // hz = A^T y, D = diag(G) first: the symmetric tiles are scaled by max D
    const dim3 g2((c->N + 127) / 128, c->B);
    if (c->st64())
        hz_diag_kernel<double><<<g2, 128, 0, c->stream>>>(
            c->dA, c->dy, c->dM, c->N, c->ldN, astride, c->Mmax, static_cast<double*>(c->dhz),
            static_cast<double*>(c->dD), c->B);
    else
        hz_diag_kernel<float><<<g2, 128, 0, c->stream>>>(
            c->dA, c->dy, c->dM, c->N, c->ldN, astride, c->Mmax, static_cast<float*>(c->dhz),
            static_cast<float*>(c->dD), c->B);
    CK(cudaGetLastError());
    if (c->sym) {
        sym_scale_kernel<float><<<c->B, 256, 0, c->stream>>>(
            static_cast<const float*>(c->dD), c->N, c->ldN, c->dSg);
        CK(cudaGetLastError());
    }
    // large instances on the symmetric path (N >= 8192: configs 3 and 4): G = A^T A
    // on the tcgen05 tensor cores from fp16 hi/lo splits of A, written straight into
    // the fp16 hi/lo tiles (gram_tc_kernels.cuh); option "gram_tc": 0 auto, 1 on, -1 off
    const bool blas = c->sym && (c->gram_tc > 0 || (c->gram_tc == 0 && c->N >= 8192));
    if (blas) {
        const int Np = c->nRB * kSyT;
        const int nchx = (c->Mmax + kGtK - 1) / kGtK;
        __half* Pv = nullptr;
        unsigned long long* amax = nullptr;
        if ((rc = dalloc(c, &Pv, (size_t)nchx * 2 * Np * kGtK * 2)) ||
            (rc = dalloc(c, &amax, (size_t)c->B * 8)))
            return rc;
        std::unique_ptr<__half, decltype(&cudaFree)> pguard(Pv, &cudaFree);
        std::unique_ptr<unsigned long long, decltype(&cudaFree)> aguard(amax, &cudaFree);
        static std::atomic<unsigned long long> attr{0};
        if (!(attr.load() >> c->device & 1ull)) {
            CK(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kGtSmem));
            attr.fetch_or(1ull << c->device);
        }
        // tile-sharded: only the row blocks of this rank's super-rows
        const int Ib = c->tshard ? c->sP0 * kSyS : 0;
        const int Ie = c->tshard ? std::min(c->nRB, c->sP1 * kSyS) : c->nRB;
        long long ntile = 0;
        for (int I = Ib; I < Ie; ++I) ntile += c->nRB - I;
        for (int b = 0; b < c->B && ntile > 0; ++b) {
            const int M = c->M[b], nch = (M + kGtK - 1) / kGtK;
            const double* Ab = c->dA + (size_t)b * astride;
            gt_absmax_kernel<<<8 * c->num_sms, 256, 0, c->stream>>>(Ab, (size_t)M * c->N, amax + b);
            gt_split_kernel<<<8 * c->num_sms, 256, 0, c->stream>>>(Ab, M, c->N, Np, nch, amax + b, Pv);
            CK(cudaGetLastError());
            GtArgs ga{};
            ga.P = Pv;
            ga.amax = amax + b;
            ga.out = SymOut{static_cast<__half*>(c->dG), c->dSg, c->nRB, c->ntri};
            ga.b = b;
            ga.N = c->N;
            ga.Np = Np;
            ga.nch = nch;
            ga.I0 = Ib;
            ga.I1 = Ie;
            ga.nRB = c->nRB;
            ga.ntile = ntile;
            const int grid = (int)std::min<long long>(ntile, c->num_sms);
            gram_tc_kernel<<<grid, kGtThreads, kGtSmem, c->stream>>>(ga);
            CK(cudaGetLastError());
            c->timing.other_launches += 3;
        }
        CK(cudaStreamSynchronize(c->stream));  // P is freed on return
    }
    // one launch per run of equal M (instances of a phase grid differ in M)
    for (int b = 0; b < c->B && !blas;) {
        int e = b;
        while (e < c->B && c->M[e] == c->M[b]) ++e;
        const dim3 grid(nt, nti, e - b);
        const double* Ab = c->dA + (size_t)b * astride;
        if (nti == 0) {
            b = e;
            continue;
        }
        const Sym64Out o64{c->sym64 ? static_cast<double*>(c->dG6) + (size_t)b * c->ntri6 * (kT6 * kT6)
                                    : nullptr,
                           c->nRB6, c->ntri6};
        if (c->sym64) {
            gram128_kernel<<<grid, 256, 0, c->stream>>>(Ab, c->M[b], c->N, astride, o64, bi0, mirror);
        } else if (c->sym) {
            SymOut o{static_cast<__half*>(c->dG) + (size_t)b * c->ntri * 2 * kSyPlaneHalfs,
                     c->dSg + b, c->nRB, c->ntri};
            gram128_kernel<<<grid, 256, 0, c->stream>>>(Ab, c->M[b], c->N, astride, o, bi0, mirror);
        } else if (c->st64()) {
            PanelOut<double, row_block<double>()> o{
                static_cast<double*>(c->dG) + (size_t)b * c->nRB * c->ldJ * c->RB, c->ldJ, c->nRB,
                c->row0};
            gram128_kernel<<<grid, 256, 0, c->stream>>>(Ab, c->M[b], c->N, astride, o, bi0, mirror);
        } else {
            PanelOut<float, row_block<float>()> o{
                static_cast<float*>(c->dG) + (size_t)b * c->nRB * c->ldJ * c->RB, c->ldJ, c->nRB,
                c->row0};
            gram128_kernel<<<grid, 256, 0, c->stream>>>(Ab, c->M[b], c->N, astride, o, bi0, mirror);
        }
        CK(cudaGetLastError());
        b = e;
    }
    cudaEventRecord(ev.ev[1], c->stream);
    CK(cudaStreamSynchronize(c->stream));
    c->timing.gram_ms = ev.ms(0, 1);
    c->timing.other_launches += 2;
    c->built = true;
    return 0;
}

int cimcs_get_coupling(cimcs_ctx* c, int32_t b, double* G, double* hz, double* D) {
    if (!c || !c->built || b < 0 || b >= c->B) return fail(CIMCS_INPUT_ERROR, "bad instance");
    if (c->world > 1 || c->tworld > 1)
        return fail(CIMCS_CONFIG_ERROR, "get_coupling: not on a sharded context");
    const int N = c->N, ld = c->ldN, RB = c->RB, ldJ = c->ldJ;
    const size_t gstride = (size_t)c->nRB * ldJ * RB;
    auto fetch = [&](const void* d, size_t off, size_t n, std::vector<double>& h) -> int {
        h.resize(n);
        if (c->st64()) {
            if (int rc_ = copy_sync(c, h.data(), static_cast<const double*>(d) + off, n * 8,
                                    cudaMemcpyDeviceToHost))
                return rc_;
        } else {
            std::vector<float> f(n);
            if (int rc_ = copy_sync(c, f.data(), static_cast<const float*>(d) + off, n * 4,
                                    cudaMemcpyDeviceToHost))
                return rc_;
            for (size_t k = 0; k < n; ++k) h[k] = f[k];
        }
        return 0;
    };
    std::vector<double> h;
    if (G && c->mri) {  // never stored: the columns G e_r of the transform chain
        float* P = nullptr;
        if (int rc = dalloc(c, &P, (size_t)N * N * 4)) return rc;
        std::unique_ptr<float, decltype(&cudaFree)> pguard(P, &cudaFree);
        if (int rc = mri_launch(c, MRI_COLS, N, 0, nullptr, P)) return rc;
        std::vector<float> f((size_t)N * N);
        if (int rc_ = copy_sync(c, f.data(), P, f.size() * 4, cudaMemcpyDeviceToHost)) return rc_;
        for (size_t k = 0; k < f.size(); ++k) G[k] = f[k];
    } else if (G && c->sym64) {
        const size_t nt = (size_t)c->ntri6 * kT6 * kT6;
        std::vector<double> t(nt);
        if (int rc_ = copy_sync(c, t.data(), static_cast<const double*>(c->dG6) + (size_t)b * nt,
                                nt * 8, cudaMemcpyDeviceToHost))
            return rc_;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                int r = i, q = j;  // stored upper triangle: G[i][j] = G[j][i]
                if (r / kT6 > q / kT6) std::swap(r, q);
                G[(size_t)i * N + j] = t[(size_t)sy_tri(r / kT6, q / kT6, c->nRB6) * kT6 * kT6 +
                                         s6_gofs(r % kT6, q % kT6)];
            }
    } else if (G && c->sym) {
        const size_t nh = (size_t)c->ntri * 2 * kSyPlaneHalfs;
        std::vector<__half> t(nh);
        int sg = 0;
        if (int rc_ = copy_sync(c, t.data(), static_cast<const __half*>(c->dG) + (size_t)b * nh,
                                nh * 2, cudaMemcpyDeviceToHost))
            return rc_;
        if (int rc_ = copy_sync(c, &sg, c->dSg + b, 4, cudaMemcpyDeviceToHost)) return rc_;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                int r = i, q = j;  // stored upper triangle: G[i][j] = G[j][i]
                if (r / kSyT > q / kSyT) std::swap(r, q);
                const size_t o = (size_t)sy_tri(r / kSyT, q / kSyT, c->nRB) * 2 * kSyPlaneHalfs +
                                 sy_offk(r % kSyT, q % kSyT, kSyT) / 2;
                const double v = (double)__half2float(t[o]) + (double)__half2float(t[o + kSyPlaneHalfs]);
                G[(size_t)i * N + j] = std::ldexp(v, -sg);
            }
    } else if (G) {
        if (int rc = fetch(c->dG, (size_t)b * gstride, gstride, h)) return rc;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j)
                G[(size_t)i * N + j] = h[((size_t)(i / RB) * ldJ + j) * RB + (i % RB)];
    }
    if (hz) {
        if (int rc = fetch(c->dhz, (size_t)b * ld, N, h)) return rc;
        std::copy(h.begin(), h.end(), hz);
    }
    if (D) {
        if (int rc = fetch(c->dD, (size_t)b * ld, N, h)) return rc;
        std::copy(h.begin(), h.end(), D);
    }
    return 0;
}

int cimcs_mfz_step(cimcs_ctx* c, int32_t R, int32_t backend, const cimcs_hyper* hp, double eta,
                   double p, const double* Rsig, const double* cin, const double* ein,
                   double* c_out, double* e_out, double* h_out, int32_t* fail_index) {
    if (int rc = check_ready(c, R)) return rc;
    if (int rc = validate(hp)) return rc;
    if (!std::isfinite(p)) return fail(CIMCS_INPUT_ERROR, "mfz_step: non-finite pump");
    if (backend != CIMCS_MFZ_BN && backend != CIMCS_MFZ_CN)
        return fail(CIMCS_CONFIG_ERROR, "backend must be mfz-bn or mfz-cn");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    const size_t n = (size_t)c->B * R * c->N;
    if (int rc = reset_flags(c, R)) return rc;
    if (int rc = set_alt(c, make_alt(hp, eta, 0))) return rc;
    if (int rc = upload_traj(c, Rsig, c->Rs, R)) return rc;
    // c and e go through a second staging area (the init kernel reads host layout)
    double* dce = nullptr;
    if (int rc = dalloc(c, &dce, 2 * n * 8)) return rc;
    CK(cudaMemcpyAsync(dce, cin, n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dce + n, ein, n * 8, cudaMemcpyHostToDevice, c->stream));
    const StepScalars s = make_scalars(hp);
    int rc = run_init(c, R, backend == CIMCS_MFZ_BN, dce, dce + n, s.rt);
    if (!rc) {
        GemvArgs a = base_args(c, s);
        a.pump = nullptr;
        a.p_scalar = p;
        a.step = 0;
        a.Win = c->W0;
        a.Wout = c->W1;
        a.Hdbg = c->Hdbg;
        rc = launch_gemv(c, backend == CIMCS_MFZ_BN ? EPI_STEP_BN : EPI_STEP_CN, a);
        if (!rc) rc = reconcile_cim(c);
        if (!rc && c->world > 1) {
            rc = allgather_state(c, c->C);
            if (!rc) rc = allgather_state(c, c->E);
            if (!rc) rc = allgather_state(c, c->Hdbg);
        }
    }
    if (!rc && c_out) rc = download_traj(c, c->C, c_out, R);
    if (!rc && e_out) rc = download_traj(c, c->E, e_out, R);
    if (!rc && h_out) rc = download_traj(c, c->Hdbg, h_out, R);
    std::vector<int> fi(c->B * c->NR);
    if (!rc)
        if (cudaMemcpyAsync(fi.data(), c->fail_idx, fi.size() * 4, cudaMemcpyDeviceToHost,
                            c->stream) != cudaSuccess)
            rc = fail(CIMCS_CUDA_ERROR, "copy");
    cudaStreamSynchronize(c->stream);
    cudaFree(dce);
    if (rc) return rc;
    bool div = false;
    for (int b = 0; b < c->B; ++b)
        for (int r = 0; r < R; ++r) {
            const int v = fi[b * c->NR + r];
            if (fail_index) fail_index[b * R + r] = v == INT_MAX ? -1 : v;
            div |= v != INT_MAX;
        }
    return div ? fail(CIMCS_DIVERGENCE, "mfz_step: non-finite amplitude") : 0;
}

int cimcs_run_pp(cimcs_ctx* c, int32_t R, const cimcs_hyper* hp, double eta, const double* Rsig,
                 const uint64_t* seeds, double* mu_out, double* e_out, double* mt_out,
                 int32_t* sigma_out, double* min_e, int32_t* fail_index) {
    if (int rc = check_ready(c, R)) return rc;
    if (int rc = validate(hp)) return rc;
    if (!(hp->j > 0.0)) return fail(CIMCS_CONFIG_ERROR, "measured_amplitude: j must be positive");
    if (!seeds) return fail(CIMCS_INPUT_ERROR, "null seeds");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    if (int rc = ensure_pp(c)) return rc;
    if (int rc = upload_pump(c, hp)) return rc;
    if (int rc = reset_flags(c, R)) return rc;
    if (int rc = set_alt(c, make_alt(hp, eta, 0))) return rc;
    if (int rc = upload_traj(c, Rsig, c->Rs, R)) return rc;
    std::vector<HostRng> rngs;
    for (int t = 0; t < c->B * R; ++t) rngs.emplace_back(seeds[t]);
    const StepScalars s = make_scalars(hp);
    Events ev(2);
    cudaEventRecord(ev.ev[0], c->stream);
    int rc = run_pp_cim(c, R, s, hp, rngs);
    cudaEventRecord(ev.ev[1], c->stream);
    if (!rc && mu_out) rc = download_traj(c, c->C, mu_out, R);
    if (!rc) rc = pp_amplitude_to_c(c);
    if (!rc) rc = run_support(c);  // sigma = mu~ > 0
    if (!rc && mt_out) rc = download_traj(c, c->C, mt_out, R);
    if (!rc && e_out) rc = download_traj(c, c->E, e_out, R);
    if (!rc && sigma_out) rc = download_sig(c, c->sig, sigma_out, R);
    std::vector<int> fi(c->B * c->NR);
    std::vector<unsigned long long> me(c->B * c->NR);
    if (!rc) {
        cudaMemcpyAsync(fi.data(), c->fail_idx, fi.size() * 4, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(me.data(), c->minE, me.size() * 8, cudaMemcpyDeviceToHost, c->stream);
    }
    cudaError_t se = cudaStreamSynchronize(c->stream);
    if (rc) return rc;
    if (se != cudaSuccess) return fail(CIMCS_CUDA_ERROR, cudaGetErrorString(se));
    c->timing.cim_ms = ev.ms(0, 1);
    c->timing.step_launches = hp->n_steps;
    bool div = false;
    int kind = 0;
    for (int b = 0; b < c->B; ++b)
        for (int r = 0; r < R; ++r) {
            const int v = fi[b * c->NR + r];
            const bool f = v != INT_MAX;
            if (fail_index) fail_index[b * R + r] = f ? (v & ((1 << 30) - 1)) : -1;
            if (min_e) min_e[b * R + r] = ord_val(me[b * c->NR + r]);
            if (f && !div) kind = v >> 30;
            div |= f;
        }
    return div ? fail(CIMCS_DIVERGENCE, kind ? "run_pp: |mu| exceeded mu_abort"
                                             : "pp_step: non-finite value")
               : 0;
}

int cimcs_run_cim(cimcs_ctx* c, int32_t R, int32_t backend, const cimcs_hyper* hp, double eta,
                  const double* Rsig, const double* c0, double* c_out, double* e_out,
                  int32_t* sigma_out, double* min_e, int32_t* fail_index) {
    if (int rc = check_ready(c, R)) return rc;
    if (int rc = validate(hp)) return rc;
    if (backend != CIMCS_MFZ_BN && backend != CIMCS_MFZ_CN)
        return fail(CIMCS_CONFIG_ERROR, "backend must be mfz-bn or mfz-cn");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    if (int rc = upload_pump(c, hp)) return rc;
    const size_t n = (size_t)c->B * R * c->N;
    if (int rc = reset_flags(c, R)) return rc;
    if (int rc = set_alt(c, make_alt(hp, eta, 0))) return rc;
    if (int rc = upload_traj(c, Rsig, c->Rs, R)) return rc;
    double* dc0 = nullptr;
    if (int rc = dalloc(c, &dc0, n * 8)) return rc;
    CK(cudaMemcpyAsync(dc0, c0, n * 8, cudaMemcpyHostToDevice, c->stream));
    const StepScalars s = make_scalars(hp);
    Events ev(2);
    cudaEventRecord(ev.ev[0], c->stream);
    int rc = run_init(c, R, backend == CIMCS_MFZ_BN, dc0, nullptr, s.rt);
    if (!rc) rc = enqueue_steps(c, backend == CIMCS_MFZ_BN, s, hp->n_steps);
    cudaEventRecord(ev.ev[1], c->stream);
    if (!rc) rc = run_support(c);
    if (!rc && c->world > 1) {
        rc = allgather_state(c, c->C);
        if (!rc) rc = allgather_state(c, c->E);
        if (!rc) rc = allgather_sig(c, c->sig);
    }
    if (!rc && c_out) rc = download_traj(c, c->C, c_out, R);
    if (!rc && e_out) rc = download_traj(c, c->E, e_out, R);
    if (!rc && sigma_out) rc = download_sig(c, c->sig, sigma_out, R);
    std::vector<int> fi(c->B * c->NR);
    std::vector<unsigned long long> me(c->B * c->NR);
    if (!rc) {
        cudaMemcpyAsync(fi.data(), c->fail_idx, fi.size() * 4, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(me.data(), c->minE, me.size() * 8, cudaMemcpyDeviceToHost, c->stream);
    }
    cudaError_t se = cudaStreamSynchronize(c->stream);
    cudaFree(dc0);
    if (rc) return rc;
    if (se != cudaSuccess) return fail(CIMCS_CUDA_ERROR, cudaGetErrorString(se));
    c->timing.cim_ms = ev.ms(0, 1);
    c->timing.step_launches = hp->n_steps;
    bool div = false;
    for (int b = 0; b < c->B; ++b)
        for (int r = 0; r < R; ++r) {
            const int v = fi[b * c->NR + r];
            if (fail_index) fail_index[b * R + r] = v == INT_MAX ? -1 : v;
            if (min_e) min_e[b * R + r] = ord_val(me[b * c->NR + r]);
            div |= v != INT_MAX;
        }
    return div ? fail(CIMCS_DIVERGENCE, "mfz_step: non-finite amplitude") : 0;
}

int cimcs_cdp_minimize(cimcs_ctx* c, int32_t R, const int32_t* sigma, const double* R_prev,
                       int32_t method, const cimcs_hyper* hp, double* R_out,
                       int32_t* iterations) {
    if (int rc = check_ready(c, R)) return rc;
    if (!hp) return fail(CIMCS_CONFIG_ERROR, "null hyper-parameters");
    if (method != CIMCS_CDP_JACOBI && method != CIMCS_CDP_CG)
        return fail(CIMCS_CONFIG_ERROR, "cdp method must be jacobi or cg");
    if (method == CIMCS_CDP_CG && c->world > 1)
        return fail(CIMCS_CONFIG_ERROR, "cdp=cg is not supported on row-sharded contexts");
    if (c->mri && method == CIMCS_CDP_JACOBI)  // cdp.cpp:158-159
        return fail(CIMCS_CONFIG_ERROR, "cdp_minimize_operator: damped Jacobi needs an assembled matrix");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    if (method == CIMCS_CDP_CG)
        if (int rc = ensure_cg(c)) return rc;
    if (int rc = reset_flags(c, R)) return rc;
    if (int rc = upload_traj(c, R_prev, c->Rs, R)) return rc;
    if (int rc = upload_sig(c, sigma, c->sig, R)) return rc;
    const StepScalars s = make_scalars(hp);
    int rc = c->st64() ? mask_T<double>(c, c->W0) : mask_T<float>(c, c->W0);
    Events ev(2);
    cudaEventRecord(ev.ev[0], c->stream);
    if (!rc)
        rc = method == CIMCS_CDP_JACOBI ? enqueue_refit(c, s, hp->jacobi_iters, false)
                                        : enqueue_cg(c, s, hp);
    cudaEventRecord(ev.ev[1], c->stream);
    if (!rc) rc = download_traj(c, c->Rs, R_out, R);
    int err = INT_MAX;
    std::vector<CgTraj> st(method == CIMCS_CDP_CG ? c->B * c->NR : 0);
    cudaMemcpyAsync(&err, c->err, 4, cudaMemcpyDeviceToHost, c->stream);
    if (!rc && !st.empty())
        cudaMemcpyAsync(st.data(), c->cg_st, st.size() * sizeof(CgTraj), cudaMemcpyDeviceToHost,
                        c->stream);
    CK(cudaStreamSynchronize(c->stream));
    if (rc) return rc;
    c->timing.refit_ms = ev.ms(0, 1);
    if (iterations)
        for (int b = 0; b < c->B; ++b)
            for (int q = 0; q < R; ++q)
                iterations[b * R + q] =
                    method == CIMCS_CDP_CG ? st[b * c->NR + q].it : hp->jacobi_iters;
    if (method == CIMCS_CDP_JACOBI && err != 0x7f7f7f7f && err != INT_MAX)
        return fail(CIMCS_INPUT_ERROR,
                    "jacobi_solve: singular diagonal at active index " + std::to_string(err));
    return 0;
}

int cimcs_refit(cimcs_ctx* c, int32_t R, const int32_t* sigma, const double* R_prev,
                double* R_out, const cimcs_hyper* hp) {
    return cimcs_cdp_minimize(c, R, sigma, R_prev, CIMCS_CDP_JACOBI, hp, R_out, nullptr);
}

int cimcs_score(cimcs_ctx* c, int32_t R, const double* Rsig, const int32_t* sigma, double lambda,
                double* objective, double* rmse, double* hamming) {
    if (int rc = check_ready(c, R)) return rc;
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_state(c, slots_for(c, R))) return rc;
    if (int rc = reset_flags(c, R)) return rc;
    AltParams ap{};
    ap.lambda = lambda;
    if (int rc = set_alt(c, ap)) return rc;
    if (int rc = upload_traj(c, Rsig, c->Rs, R)) return rc;
    if (int rc = upload_sig(c, sigma, c->sig, R)) return rc;
    cimcs_hyper h;
    cimcs_hyper_default(&h);
    const StepScalars s = make_scalars(&h);
    int rc = c->st64() ? mask_T<double>(c, c->W0) : mask_T<float>(c, c->W0);
    if (!rc) rc = enqueue_score(c, s, 0, nullptr, false);
    const int nT = c->B * c->NR;
    std::vector<double> o(nT), r(nT), h_(nT);
    if (!rc) {
        cudaMemcpyAsync(o.data(), c->obj, nT * 8, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(r.data(), c->rmse, nT * 8, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(h_.data(), c->ham, nT * 8, cudaMemcpyDeviceToHost, c->stream);
    }
    CK(cudaStreamSynchronize(c->stream));
    if (rc) return rc;
    for (int b = 0; b < c->B; ++b)
        for (int q = 0; q < R; ++q) {
            if (objective) objective[b * R + q] = o[b * c->NR + q];
            if (rmse) rmse[b * R + q] = r[b * c->NR + q];
            if (hamming) hamming[b * R + q] = h_[b * c->NR + q];
        }
    return 0;
}

int cimcs_solve(cimcs_ctx* c, int32_t R, int32_t backend, const cimcs_hyper* hp, int32_t cdp,
                const uint64_t* seeds, const double* R_init, int32_t track_best, double* R_out,
                int32_t* sigma_out, cimcs_record* hist, int32_t* n_hist, int32_t* fail_alt,
                int32_t* fail_index) {
    if (int rc = check_ready(c, R)) return rc;
    if (int rc = validate(hp)) return rc;
    if (backend != CIMCS_MFZ_BN && backend != CIMCS_MFZ_CN && backend != CIMCS_PP)
        return fail(CIMCS_CONFIG_ERROR, "backend must be mfz-bn, mfz-cn or pp");
    const bool pp = backend == CIMCS_PP;
    if (pp && !(hp->j > 0.0))
        return fail(CIMCS_CONFIG_ERROR, "measured_amplitude: j must be positive");
    if (cdp != CIMCS_CDP_JACOBI && cdp != CIMCS_CDP_CG)
        return fail(CIMCS_CONFIG_ERROR, "cdp must be jacobi or cg");
    if (cdp == CIMCS_CDP_CG && c->world > 1)
        return fail(CIMCS_CONFIG_ERROR, "cdp=cg is not supported on row-sharded contexts");
    if (c->mri) cdp = CIMCS_CDP_CG;  // transform-chain problems always use CG (orchestrator.cpp:128-133)
    if (!seeds) return fail(CIMCS_INPUT_ERROR, "null seeds");
    CK(cudaSetDevice(c->device));
    const int NR = slots_for(c, R);
    if (int rc = ensure_state(c, NR)) return rc;
    if (cdp == CIMCS_CDP_CG)
        if (int rc = ensure_cg(c)) return rc;
    if (pp)
        if (int rc = ensure_pp(c)) return rc;
    if (int rc = upload_pump(c, hp)) return rc;
    const int nalt = hp->velo + 1;
    const int nT = c->B * NR;
    if (c->hist_cap < nalt * nT) {
        if (c->hist) cudaFree(c->hist);
        c->hist = nullptr;
        if (int rc = dalloc(c, &c->hist, (size_t)nalt * nT * sizeof(DevRecord))) return rc;
        c->hist_cap = nalt * nT;
    }
    const int bn = backend == CIMCS_MFZ_BN;
    const StepScalars s = make_scalars(hp);
    const int ntraj = c->B * R;
    const size_t nc0 = (size_t)ntraj * c->N;

    // host streams + pinned double buffer for c0
    std::vector<HostRng> rngs;
    rngs.reserve(ntraj);
    for (int t = 0; t < ntraj; ++t) rngs.emplace_back(seeds[t]);
    if (c->pin_c0_elems < nc0) {
        if (c->pin_c0) cudaFreeHost(c->pin_c0);
        c->pin_c0 = nullptr;
        CK(cudaMallocHost(&c->pin_c0, 2 * nc0 * 8));
        c->pin_c0_elems = nc0;
    }
    if (c->dc0_elems < nc0) {
        if (c->dc0) cudaFree(c->dc0);
        c->dc0 = nullptr;
        drop_graphs(c);  // the CIM graph reads dc0
        if (int rc = dalloc(c, &c->dc0, nc0 * 8)) return rc;
        c->dc0_elems = nc0;
    }
    double* pinned = c->pin_c0;
    double* dc0 = c->dc0;
    std::vector<AltParams> alts(nalt);
    for (int i = 0; i < nalt; ++i)
        alts[i] = make_alt(hp, eta_schedule(i, hp->eta_init, hp->eta_end, hp->velo), i);
    AltParams* halts = nullptr;
    CK(cudaMallocHost(&halts, nalt * sizeof(AltParams)));
    std::unique_ptr<AltParams, decltype(&cudaFreeHost)> alt_guard(halts, &cudaFreeHost);
    std::copy(alts.begin(), alts.end(), halts);

    Events ev(4 * nalt + 2);
    Events slot_done(2);
    cudaEventRecord(ev.ev[4 * nalt], c->stream);

    // initial state: R_init (default hz), flags, best objective = +inf
    int rc = reset_flags(c, R);
    if (!rc) {
        if (R_init)
            rc = upload_traj(c, R_init, c->Rs, R);
        else
            rc = c->st64() ? rinit_hz_T<double>(c, R) : rinit_hz_T<float>(c, R);
    }
    if (rc) return rc;
    CK(cudaMemsetAsync(c->sig, 0, c->state_elems(), c->stream));
    {
        std::vector<double> inf(nT, INFINITY);
        CK(cudaMemcpyAsync(c->best_obj, inf.data(), nT * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemsetAsync(c->improved, 0, nT * 4, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // `inf` leaves scope
    }
    if (track_best) {
        CK(cudaMemcpyAsync(c->bestR, c->Rs, c->state_elems() * c->elt(), cudaMemcpyDeviceToDevice,
                           c->stream));
        CK(cudaMemsetAsync(c->bestS, 0, c->state_elems(), c->stream));
    }

    // graphs: [init + steps], [support + jacobi], [score + finalize + median (+best)]
    // The history slot differs per alternation, so the score graph is per-alternation
    // cheap; the two heavy graphs are captured once and replayed.
    // the two heavy graphs are cached across solves with the same shape and
    // schedule (the scalars they bake in are part of the key)
    if (c->use_graphs) {
        auto bits = [](double v) {
            long long u;
            std::memcpy(&u, &v, 8);
            return u;
        };
        const std::vector<long long> key = {R, NR, bn, hp->n_steps, hp->jacobi_iters,
                                            (long long)(uintptr_t)dc0, bits(s.dt), bits(s.rt),
                                            bits(s.nbeta), bits(s.Kj), bits(s.minus_j),
                                            bits(s.dt_c), c->B, c->N, cdp, hp->cg_max_iters,
                                            bits(hp->cg_tol), backend};
        if (key != c->graph_key || (!pp && !c->g_cim) || !c->g_refit) {
            drop_graphs(c);
            Graph gc, gr;
            if (!pp)  // the Positive-P CIM call is host-driven (chunked noise upload)
                rc = capture(c, gc, [&] {
                    int r2 = run_init(c, R, bn, dc0, nullptr, s.rt);
                    return r2 ? r2 : enqueue_steps(c, bn, s, hp->n_steps);
                });
            if (!rc)
                rc = capture(c, gr, [&] {
                    if (cdp == CIMCS_CDP_CG) {
                        int r2 = run_support(c);
                        return r2 ? r2 : enqueue_cg(c, s, hp);
                    }
                    return enqueue_refit(c, s, hp->jacobi_iters, true);
                });
            if (rc) return rc;
            c->g_cim = gc.exec;
            c->g_refit = gr.exec;
            gc.exec = gr.exec = nullptr;
            c->graph_key = key;
        }
    }
    const int v_slot = cdp == CIMCS_CDP_CG ? 0 : hp->jacobi_iters & 1;
    if (!pp) gen_c0(rngs, c->N, pinned, c->host_threads);
    for (int i = 0; i < nalt; ++i) {
        double* slot = pinned + (size_t)(i & 1) * nc0;
        CK(cudaMemcpyAsync(c->alt, &halts[i], sizeof(AltParams), cudaMemcpyHostToDevice,
                           c->stream));
        if (!pp) {
            CK(cudaMemcpyAsync(dc0, slot, nc0 * 8, cudaMemcpyHostToDevice, c->stream));
            CK(cudaEventRecord(slot_done.ev[i & 1], c->stream));
        }
        CK(cudaEventRecord(ev.ev[4 * i + 0], c->stream));
        if (pp) {
            if ((rc = run_pp_cim(c, R, s, hp, rngs)) || (rc = pp_amplitude_to_c(c))) return rc;
        } else if (c->use_graphs) {
            CK(cudaGraphLaunch(c->g_cim, c->stream));
        } else {
            rc = run_init(c, R, bn, dc0, nullptr, s.rt);
            if (!rc) rc = enqueue_steps(c, bn, s, hp->n_steps);
            if (rc) return rc;
        }
        CK(cudaEventRecord(ev.ev[4 * i + 1], c->stream));
        if (c->use_graphs) {
            CK(cudaGraphLaunch(c->g_refit, c->stream));
        } else if (cdp == CIMCS_CDP_CG) {
            if ((rc = run_support(c)) || (rc = enqueue_cg(c, s, hp))) return rc;
        } else if ((rc = enqueue_refit(c, s, hp->jacobi_iters, true))) {
            return rc;
        }
        CK(cudaEventRecord(ev.ev[4 * i + 2], c->stream));
        if ((rc = enqueue_score(c, s, v_slot, c->hist + (size_t)i * nT, track_best != 0)))
            return rc;
        CK(cudaEventRecord(ev.ev[4 * i + 3], c->stream));
        if (i + 1 < nalt && !pp) {
            // draw the next alternation's c0 while the GPU works on this one
            CK(cudaEventSynchronize(slot_done.ev[(i + 1) & 1]));
            gen_c0(rngs, c->N, pinned + (size_t)((i + 1) & 1) * nc0, c->host_threads);
        }
    }
    cudaEventRecord(ev.ev[4 * nalt + 1], c->stream);

    // results
    if (c->world > 1) {  // every rank returns the full vectors
        if ((rc = allgather_sig(c, c->sig))) return rc;
        if (track_best && (rc = allgather_sig(c, c->bestS))) return rc;
    }
    const void* Rsrc = track_best ? c->bestR : c->Rs;
    const int8_t* Ssrc = track_best ? c->bestS : c->sig;
    if (track_best) {
        // best is only used when some alternation was recorded (isfinite(best_energy))
        // -- trajectories with no record keep their current R/sigma.
        std::vector<double> bo(nT);
        CK(cudaMemcpyAsync(bo.data(), c->best_obj, nT * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        bool all = true;
        for (int b = 0; b < c->B; ++b)
            for (int q = 0; q < R; ++q) all &= std::isfinite(bo[b * NR + q]);
        if (!all) {
            // copy current state into best slots of unrecorded trajectories
            std::vector<int> imp(nT, 0);
            for (int b = 0; b < c->B; ++b)
                for (int q = 0; q < R; ++q) imp[b * NR + q] = !std::isfinite(bo[b * NR + q]);
            CK(cudaMemcpyAsync(c->improved, imp.data(), nT * 4, cudaMemcpyHostToDevice,
                               c->stream));
            const int g = grid_for(c->state_elems());
            if (c->st64()) {
                DISPATCH_NR(NR, {
                    best_update_kernel<double, NR_><<<g, 256, 0, c->stream>>>(
                        c->improved, static_cast<const double*>(c->Rs), c->sig,
                        static_cast<double*>(c->bestR), c->bestS, c->ldN, c->B);
                });
            } else {
                DISPATCH_NR(NR, {
                    best_update_kernel<float, NR_><<<g, 256, 0, c->stream>>>(
                        c->improved, static_cast<const float*>(c->Rs), c->sig,
                        static_cast<float*>(c->bestR), c->bestS, c->ldN, c->B);
                });
            }
            CK(cudaStreamSynchronize(c->stream));
        }
    }
    if (R_out && (rc = download_traj(c, Rsrc, R_out, R))) return rc;
    if (sigma_out && (rc = download_sig(c, Ssrc, sigma_out, R))) return rc;
    std::vector<DevRecord> dh((size_t)nalt * nT);
    std::vector<int> nh(nT), fg(nT), fi(nT);
    CK(cudaMemcpyAsync(dh.data(), c->hist, dh.size() * sizeof(DevRecord), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaMemcpyAsync(nh.data(), c->n_hist, nT * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(fg.data(), c->fail_gstep, nT * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(fi.data(), c->fail_idx, nT * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    int err = 0;
    if (int rc_ = copy_sync(c, &err, c->err, 4, cudaMemcpyDeviceToHost)) return rc_;
    if (err != 0x7f7f7f7f && err != INT_MAX)
        return fail(CIMCS_INPUT_ERROR,
                    "jacobi_solve: singular diagonal at active index " + std::to_string(err));

    cimcs_timing& tm = c->timing;
    tm.total_ms = ev.ms(4 * nalt, 4 * nalt + 1);
    tm.cim_ms = tm.refit_ms = tm.score_ms = 0.0;
    for (int i = 0; i < nalt; ++i) {
        tm.cim_ms += ev.ms(4 * i + 0, 4 * i + 1);
        tm.refit_ms += ev.ms(4 * i + 1, 4 * i + 2);
        tm.score_ms += ev.ms(4 * i + 2, 4 * i + 3);
    }
    // kernels of this library per alternation: init + steps | support + sweeps |
    // score contraction, tp, finalize, median (+ best).  The small-N cluster loop
    // runs a whole CIM call / refit in one launch; CG counts its last iteration total.
    const bool cl = cluster_ok(c) && !pp;
    const int per = c->sym || c->sym64 ? 2 : 1;  // symmetric paths: tile kernel + update kernel
    tm.step_launches = (int64_t)nalt * (cl ? 1 : per * hp->n_steps + (pp ? 1 : 0));
    if (cdp == CIMCS_CDP_CG) {
        std::vector<CgTraj> st(nT);
        if (int rc_ = copy_sync(c, st.data(), c->cg_st, nT * sizeof(CgTraj), cudaMemcpyDeviceToHost))
            return rc_;
        int mx = 0;
        for (const CgTraj& t : st) mx = std::max(mx, t.it);
        tm.refit_launches = (int64_t)nalt * (6 + 3 * (int64_t)mx);
    } else {
        tm.refit_launches = (int64_t)nalt * (cl ? 1 : per * hp->jacobi_iters);
    }
    tm.other_launches = (int64_t)nalt * (2 + 4 + (track_best ? 1 : 0));
    tm.step_bytes = (double)c->B * c->N * (double)c->N * c->elt();  // dense G share
    tm.step_flops = 2.0 * c->B * (double)c->N * c->N * R;

    for (int b = 0; b < c->B; ++b)
        for (int q = 0; q < R; ++q) {
            const int dt = b * NR + q, ht = b * R + q;
            if (n_hist) n_hist[ht] = nh[dt];
            const bool failed = fg[dt] != kFreeTraj;
            if (fail_alt) fail_alt[ht] = failed ? fg[dt] / hp->n_steps : -1;
            if (fail_index) fail_index[ht] = failed ? (fi[dt] & ((1 << 30) - 1)) : -1;
            if (hist)
                for (int i = 0; i < nalt; ++i) {
                    cimcs_record& o = hist[(size_t)ht * nalt + i];
                    if (i < nh[dt]) {
                        const DevRecord& d = dh[(size_t)i * nT + dt];
                        o.i = d.i;
                        o.support = d.support;
                        o.eta = d.eta;
                        o.hamiltonian = d.hamiltonian;
                        o.rmse = d.rmse;
                        o.hamming = d.hamming;
                        o.min_e = d.min_e;
                        o.median_e = d.median_e;
                    } else {
                        std::memset(&o, 0, sizeof(o));
                        o.i = -1;
                    }
                }
        }
    return 0;
}

int cimcs_get_timing(const cimcs_ctx* c, cimcs_timing* out) {
    if (!c || !out) return fail(CIMCS_INPUT_ERROR, "null argument");
    *out = c->timing;
    return 0;
}

}  // extern "C"
