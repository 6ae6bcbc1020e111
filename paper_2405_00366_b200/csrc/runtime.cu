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
#include <nvtx3/nvToolsExt.h>

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
#include "cmp_kernels.cuh"
#include "mri_kernels.cuh"
#include "dct_kernels.cuh"

using namespace cimcs;

// The runtime is ONE translation unit assembled from parts split by concern:
#include "rt_aux_kernels.cuh"
#include "rt_context.cuh"
#include "rt_memory.cuh"
#include "rt_launch.cuh"
#include "rt_enqueue.cuh"
#include "rt_abi_core.cuh"
#include "rt_abi_context.cuh"
#include "rt_abi_problems.cuh"
#include "rt_abi_solve.cuh"
