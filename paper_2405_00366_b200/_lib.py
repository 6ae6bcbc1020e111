"""ctypes binding of libcimcs_gpu.so (the C ABI in include/cimcs_gpu.h).

No fallback: if the shared library is missing or cannot be loaded the import
of any GPU entry point raises.  Build it with ``python -m
paper_2405_00366_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CIMCS_GPU_LIB") or os.path.join(HERE, "libcimcs_gpu.so")

OK, INPUT_ERROR, CONFIG_ERROR, DIVERGENCE, CUDA_ERROR = 0, 1, 2, 3, 4
F32, F64 = 0, 1
MFZ_CN, MFZ_BN, PP = 0, 1, 2
CDP_JACOBI, CDP_CG = 0, 1
PUMP_SIGMOID, PUMP_LINEAR = 0, 1

# every symbol include/cimcs_gpu.h declares
EXPORTS = (
    "cimcs_abi_version", "cimcs_last_error", "cimcs_hyper_default", "cimcs_hyper_validate",
    "cimcs_mix_seed", "cimcs_gemv_order", "cimcs_canon_order", "cimcs_gen_dims", "cimcs_gen_instance",
    "cimcs_gen_instances", "cimcs_create", "cimcs_destroy", "cimcs_set_option",
    "cimcs_set_problems", "cimcs_build_coupling", "cimcs_get_coupling", "cimcs_mfz_step",
    "cimcs_run_cim", "cimcs_run_pp", "cimcs_refit", "cimcs_cdp_minimize", "cimcs_score", "cimcs_solve", "cimcs_get_timing",
    "cimcs_get_timeline",
    "cimcs_nccl_unique_id", "cimcs_create_sharded", "cimcs_format_double", "cimcs_fnv1a64",
    "cimcs_save_instance", "cimcs_load_instance", "cimcs_csv_open", "cimcs_csv_row",
    "cimcs_csv_close", "cimcs_make_mask", "cimcs_set_mri_problem", "cimcs_set_dct_problem",
    "cimcs_mri_lasso", "cimcs_tile_shard", "cimcs_set_generated_problems",
    "cimcs_get_instance",
)


class Hyper(C.Structure):
    _fields_ = [
        ("g2", C.c_double), ("j", C.c_double), ("K", C.c_double), ("beta", C.c_double),
        ("tau", C.c_double), ("dt", C.c_double), ("n_steps", C.c_int32),
        ("p_thr", C.c_double), ("d", C.c_double), ("eta_init", C.c_double),
        ("eta_end", C.c_double), ("velo", C.c_int32), ("dt_c", C.c_double),
        ("jacobi_iters", C.c_int32), ("cg_max_iters", C.c_int32), ("cg_tol", C.c_double),
        ("gamma", C.c_double), ("mfz_loss_minus_j", C.c_int32), ("mu_abort", C.c_double),
        ("pump_kind", C.c_int32), ("pump_end", C.c_double),
    ]


class Record(C.Structure):
    _fields_ = [
        ("i", C.c_int32), ("support", C.c_int32), ("eta", C.c_double),
        ("hamiltonian", C.c_double), ("rmse", C.c_double), ("hamming", C.c_double),
        ("min_e", C.c_double), ("median_e", C.c_double),
    ]


class Timing(C.Structure):
    _fields_ = [
        ("total_ms", C.c_double), ("gram_ms", C.c_double), ("cim_ms", C.c_double),
        ("refit_ms", C.c_double), ("score_ms", C.c_double), ("h2d_ms", C.c_double),
        ("d2h_ms", C.c_double), ("step_launches", C.c_int64), ("refit_launches", C.c_int64),
        ("other_launches", C.c_int64), ("step_bytes", C.c_double), ("step_flops", C.c_double),
        ("tile_kernel_ms", C.c_double), ("tile_kernel_launches", C.c_int64),
    ]


_lib = None


def load() -> C.CDLL:
    """Load libcimcs_gpu.so (raises OSError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -m paper_2405_00366_b200.build)")
    L = C.CDLL(LIB_PATH)
    vp, i32, d, u64 = C.c_void_p, C.c_int32, C.c_double, C.c_uint64
    L.cimcs_last_error.restype = C.c_char_p
    L.cimcs_mix_seed.restype = u64
    L.cimcs_mix_seed.argtypes = [u64, u64]
    L.cimcs_gemv_order.argtypes = [C.c_int, vp, vp]
    L.cimcs_canon_order.argtypes = [vp, vp, vp]
    L.cimcs_gen_dims.argtypes = [i32, d, d, vp, vp]
    L.cimcs_gen_instance.argtypes = [i32, d, d, d, u64, vp, vp, vp, vp]
    L.cimcs_gen_instances.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, i32]
    L.cimcs_hyper_default.argtypes = [vp]
    L.cimcs_hyper_validate.argtypes = [vp]
    L.cimcs_create.argtypes = [i32, i32, vp]
    L.cimcs_destroy.argtypes = [vp]
    L.cimcs_set_option.argtypes = [vp, C.c_char_p, C.c_int64]
    L.cimcs_set_problems.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp]
    L.cimcs_build_coupling.argtypes = [vp]
    L.cimcs_get_coupling.argtypes = [vp, i32, vp, vp, vp]
    L.cimcs_mfz_step.argtypes = [vp, i32, i32, vp, d, d, vp, vp, vp, vp, vp, vp, vp]
    L.cimcs_run_cim.argtypes = [vp, i32, i32, vp, d, vp, vp, vp, vp, vp, vp, vp]
    L.cimcs_refit.argtypes = [vp, i32, vp, vp, vp, vp]
    L.cimcs_run_pp.argtypes = [vp, i32, vp, C.c_double, vp, vp, vp, vp, vp, vp, vp, vp]
    L.cimcs_cdp_minimize.argtypes = [vp, i32, vp, vp, i32, vp, vp, vp]
    L.cimcs_score.argtypes = [vp, i32, vp, vp, d, vp, vp, vp]
    L.cimcs_solve.argtypes = [vp, i32, i32, vp, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp]
    L.cimcs_get_timing.argtypes = [vp, vp]
    L.cimcs_get_timeline.argtypes = [vp, vp, C.c_int64, vp]
    L.cimcs_nccl_unique_id.argtypes = [vp, i32]
    L.cimcs_create_sharded.argtypes = [i32, i32, i32, i32, vp, vp]
    L.cimcs_format_double.argtypes = [d, C.c_char_p, i32]
    L.cimcs_fnv1a64.restype = u64
    L.cimcs_fnv1a64.argtypes = [C.c_char_p, u64]
    L.cimcs_save_instance.argtypes = [C.c_char_p, i32, i32, vp, vp, vp, vp, d, d, d, u64]
    L.cimcs_load_instance.argtypes = [C.c_char_p, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.cimcs_csv_open.argtypes = [C.c_char_p, vp, i32, vp, i32, vp]
    L.cimcs_csv_row.argtypes = [vp, vp, i32]
    L.cimcs_csv_close.argtypes = [vp]
    L.cimcs_make_mask.argtypes = [i32, i32, i32, u64, vp]
    L.cimcs_tile_shard.argtypes = [i32, i32, i32, vp, vp]
    L.cimcs_set_generated_problems.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    L.cimcs_get_instance.argtypes = [vp, i32, vp, vp, vp, vp]
    L.cimcs_set_mri_problem.argtypes = [vp, i32, i32, vp, i32, vp, d, vp]
    L.cimcs_mri_lasso.argtypes = [vp, d, i32, d, d, vp, vp, vp]
    L.cimcs_set_dct_problem.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    _lib = L
    return L


def last_error() -> str:
    return load().cimcs_last_error().decode()
