"""B200-native MFZ-CIM L0-regularised compressed-sensing hot path (arXiv 2405.00366).

The CUDA kernels and the C ABI live in ``csrc/`` and ``include/cimcs_gpu.h``;
this package is the Python mirror of the reference's ``cimcs`` module.
"""
from .cimcs import (  # noqa: F401
    BACKENDS, ConfigError, Context, CudaError, DivergenceError, HyperParams, InputError,
    Instance, baseline_params, eta_schedule, gemv_order, gen_dims, gen_instance,
    gen_instances, mix_seed, nccl_unique_id, pump_schedule, replica_seeds, solve, solve_batch,
)
