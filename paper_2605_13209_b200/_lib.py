"""ctypes binding of ``libhsolve_cuda.so`` (the C ABI in include/hs_cuda.h).

The library is built in-tree by ``paper_2605_13209_b200._build`` (or
``__graft_entry__.build()``). There is no fallback: if the shared object is
missing or fails to load, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

_LIB = None

HS_OK = 0
HS_ERR_CONFIG = 1
HS_ERR_NOT_SPD = 2
HS_ERR_SINGULAR_BLOCK = 3
HS_ERR_NUMERICAL = 4
HS_ERR_NOT_CONVERGED = 5
HS_ERR_RESIDENCY = 6
HS_ERR_FORMAT = 7
HS_ERR_VERSION_MISMATCH = 8
HS_ERR_TRUNCATED_FILE = 9
HS_ERR_IO = 10
HS_ERR_CUDA = 100

# Every symbol include/hs_cuda.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "hs_last_error", "hs_last_error_payload", "hs_error_kind_name",
    "hs_ctx_create", "hs_nccl_unique_id", "hs_ctx_create_nccl", "hs_ctx_destroy", "hs_ctx_trim",
    "hs_ctx_create_custom_comm",
    "hs_ctx_rank", "hs_ctx_world", "hs_ctx_stream", "hs_ctx_kernel_launches",
    "hs_ctx_set_cholesky_gemm", "hs_device_count", "hs_device_alloc", "hs_device_free",
    "hs_memcpy",
    "hs_group_create", "hs_group_destroy", "hs_group_world", "hs_group_transport",
    "hs_group_ctx", "hs_group_set_row_fraction", "hs_group_set_cholesky_gemm", "hs_group_run",
    "hs_group_solve_cg_host", "hs_group_factorize_host", "hs_group_solve_spd_host",
    "hs_rng_at", "hs_rng_uniform_pm1", "hs_generate_inputs",
    "hs_median_pairwise_distance", "hs_generate_rhs",
    "hs_partition_for_fraction", "hs_cholesky_border", "hs_partition_rows",
    "hs_matrix_create", "hs_matrix_create_cyclic", "hs_matrix_destroy", "hs_matrix_info", "hs_matrix_upload",
    "hs_matrix_download", "hs_matrix_copy", "hs_matrix_device_data",
    "hs_assemble_se", "hs_generate_spd",
    "hs_cg_solve", "hs_solve_cg_host", "hs_symv", "hs_true_residual",
    "hs_potrf", "hs_trsv_lower", "hs_trsv_upper", "hs_solve_spd", "hs_solve_spd_refine",
    "hs_factorize_host", "hs_solve_spd_host", "hs_forward_substitute_host",
    "hs_back_substitute_host", "hs_potf_tiles", "hs_gemm_update_tiles", "hs_oz_gemm_tiles",
    "hs_trsm_tiles", "hs_block_vec_op", "hs_range_op", "hs_block_exact", "hs_symv_exact",
    "hs_oz_set_profile",
    "hs_prof_enable", "hs_prof_symv", "hs_prof_reset", "hs_probe_hbm_read",
    "hs_ctx_ledger_size", "hs_ctx_ledger_read", "hs_ctx_ledger_clear",
    "hs_bspd1_probe", "hs_bspd1_read", "hs_bspd1_write", "hs_vector_probe",
    "hs_vector_read", "hs_vector_write", "hs_matrix_load_bspd1", "hs_matrix_save_bspd1",
]


class CgParams(C.Structure):
    _fields_ = [("eps", C.c_double), ("max_iters", C.c_uint64),
                ("recompute_interval", C.c_uint64), ("record_trace", C.c_int)]


class CgStats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("recomputations", C.c_uint64),
                ("converged", C.c_int), ("u0", C.c_double),
                ("true_residual", C.c_double), ("wall_ms", C.c_double),
                ("compute_ms", C.c_double), ("transfer_ms", C.c_double),
                ("error_iteration", C.c_int64)]


class CholStats(C.Structure):
    _fields_ = [("factor_ms", C.c_double), ("solve_ms", C.c_double),
                ("wall_ms", C.c_double), ("compute_ms", C.c_double),
                ("transfer_ms", C.c_double), ("true_residual", C.c_double)]


class RefineStats(C.Structure):
    _fields_ = [("factor_ms", C.c_double), ("solve_ms", C.c_double),
                ("wall_ms", C.c_double), ("rel_residual", C.c_double),
                ("iterations", C.c_int), ("slices", C.c_int)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
REDUCE_SCATTER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
BROADCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int)
ALLREDUCE_MAX_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t)


class CommOps(C.Structure):  # hs_comm_ops
    _fields_ = [("allgather", ALLGATHER_FN), ("reduce_scatter", REDUCE_SCATTER_FN),
                ("broadcast", BROADCAST_FN), ("allreduce_max_i64", ALLREDUCE_MAX_FN),
                ("user", C.c_void_p)]


class LedgerEntry(C.Structure):  # hs_ledger_entry
    _fields_ = [("kind", C.c_uint8), ("direction", C.c_uint8), ("bytes", C.c_uint64),
                ("step", C.c_int64)]


def lib_path() -> str:
    return _build.CUDA_LIB


def lib():
    """Load libhsolve_cuda.so (raises if it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2605_13209_b200._build` "
            "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, sz, dp, u64, i64 = C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint64, C.c_int64
    pp = C.POINTER(C.c_void_p)
    sig = {
        "hs_last_error": (C.c_char_p, []),
        "hs_last_error_payload": (None, [C.POINTER(i64), C.POINTER(i64)]),
        "hs_error_kind_name": (C.c_char_p, [C.c_int]),
        "hs_ctx_create": (C.c_int, [C.c_int, vp, pp]),
        "hs_nccl_unique_id": (C.c_int, [vp]),
        "hs_ctx_create_nccl": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, vp, pp]),
        "hs_ctx_create_custom_comm": (C.c_int, [C.c_int, vp, C.c_int, C.c_int,
                                                C.POINTER(CommOps), pp]),
        "hs_ctx_destroy": (None, [vp]),
        "hs_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "hs_device_alloc": (C.c_int, [vp, sz, pp]),
        "hs_device_free": (None, [vp, vp]),
        "hs_memcpy": (C.c_int, [vp, vp, vp, sz]),
        "hs_group_create": (C.c_int, [C.c_int, vp, C.c_int, pp]),
        "hs_group_destroy": (None, [vp]),
        "hs_group_world": (C.c_int, [vp]),
        "hs_group_transport": (C.c_int, [vp]),
        "hs_group_ctx": (vp, [vp, C.c_int]),
        "hs_group_set_row_fraction": (C.c_int, [vp, C.c_double]),
        "hs_group_set_cholesky_gemm": (C.c_int, [vp, C.c_int]),
        "hs_group_run": (C.c_int, [vp, vp, vp]),
        "hs_group_solve_cg_host": (C.c_int, [vp, sz, sz, dp, dp, C.POINTER(CgParams), dp,
                                             C.POINTER(CgStats), dp]),
        "hs_group_factorize_host": (C.c_int, [vp, sz, sz, dp, C.POINTER(CholStats)]),
        "hs_group_solve_spd_host": (C.c_int, [vp, sz, sz, dp, dp, dp, C.POINTER(CholStats)]),
        "hs_ctx_trim": (C.c_int, [vp]),
        "hs_ctx_rank": (C.c_int, [vp]),
        "hs_ctx_world": (C.c_int, [vp]),
        "hs_ctx_stream": (vp, [vp]),
        "hs_ctx_kernel_launches": (u64, [vp]),
        "hs_ctx_set_cholesky_gemm": (C.c_int, [vp, C.c_int]),
        "hs_rng_at": (u64, [u64, u64]),
        "hs_rng_uniform_pm1": (C.c_double, [u64, u64]),
        "hs_generate_inputs": (C.c_int, [sz, sz, u64, dp]),
        "hs_median_pairwise_distance": (C.c_double, [dp, sz, sz]),
        "hs_generate_rhs": (C.c_int, [sz, sz, u64, dp]),
        "hs_partition_for_fraction": (C.c_int, [C.c_double, sz, C.POINTER(sz)]),
        "hs_cholesky_border": (C.c_int, [C.c_double, sz, sz, C.POINTER(sz)]),
        "hs_partition_rows": (C.c_int, [sz, C.c_int, dp]),
        "hs_matrix_create": (C.c_int, [vp, sz, sz, pp]),
        "hs_matrix_create_cyclic": (C.c_int, [vp, sz, sz, pp]),
        "hs_matrix_destroy": (None, [vp]),
        "hs_matrix_info": (C.c_int, [vp, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz),
                                     C.POINTER(sz)]),
        "hs_matrix_upload": (C.c_int, [vp, dp]),
        "hs_matrix_download": (C.c_int, [vp, dp]),
        "hs_matrix_copy": (C.c_int, [vp, vp]),
        "hs_matrix_device_data": (vp, [vp]),
        "hs_assemble_se": (C.c_int, [vp, dp, sz, C.c_double, C.c_double, C.c_double]),
        "hs_generate_spd": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, sz, u64]),
        "hs_cg_solve": (C.c_int, [vp, vp, dp, C.POINTER(CgParams), dp,
                                  C.POINTER(CgStats), dp]),
        "hs_solve_cg_host": (C.c_int, [vp, sz, sz, dp, dp, C.POINTER(CgParams), dp,
                                       C.POINTER(CgStats), dp]),
        "hs_symv": (C.c_int, [vp, vp, dp, dp]),
        "hs_true_residual": (C.c_int, [vp, vp, dp, dp, C.POINTER(C.c_double)]),
        "hs_potrf": (C.c_int, [vp, vp, C.POINTER(CholStats)]),
        "hs_trsv_lower": (C.c_int, [vp, vp, dp]),
        "hs_trsv_upper": (C.c_int, [vp, vp, dp]),
        "hs_solve_spd": (C.c_int, [vp, vp, dp, dp, vp, C.POINTER(CholStats)]),
        "hs_solve_spd_refine": (C.c_int, [vp, vp, vp, dp, dp, C.c_int, C.c_int, C.c_double,
                                          C.POINTER(RefineStats)]),
        "hs_factorize_host": (C.c_int, [vp, sz, sz, dp, C.POINTER(CholStats)]),
        "hs_solve_spd_host": (C.c_int, [vp, sz, sz, dp, dp, dp, C.POINTER(CholStats)]),
        "hs_forward_substitute_host": (C.c_int, [vp, sz, sz, dp, dp, dp]),
        "hs_back_substitute_host": (C.c_int, [vp, sz, sz, dp, dp, dp]),
        "hs_potf_tiles": (C.c_int, [vp, dp, sz, sz, C.POINTER(i64)]),
        "hs_gemm_update_tiles": (C.c_int, [vp, dp, dp, dp, sz, sz, C.c_int]),
        "hs_oz_gemm_tiles": (C.c_int, [vp, dp, dp, dp, sz, sz, C.c_int, C.c_int]),
        "hs_oz_set_profile": (None, [vp]),
        "hs_trsm_tiles": (C.c_int, [vp, dp, dp, sz, sz]),
        "hs_block_exact": (C.c_int, [vp, C.c_int, dp, dp, dp, sz, C.POINTER(i64)]),
        "hs_symv_exact": (C.c_int, [vp, dp, dp, dp, sz, sz, sz, sz]),
        "hs_block_vec_op": (C.c_int, [vp, C.c_int, dp, dp, dp, sz]),
        "hs_range_op": (C.c_int, [vp, C.c_int, dp, dp, dp, C.c_double, sz, sz, sz]),
        "hs_prof_enable": (None, [vp, C.c_int]),
        "hs_prof_symv": (None, [vp, C.POINTER(u64), C.POINTER(C.c_double)]),
        "hs_prof_reset": (None, [vp]),
        "hs_probe_hbm_read": (C.c_int, [vp, sz, C.c_int, C.c_int, C.POINTER(C.c_double)]),
        "hs_ctx_ledger_size": (sz, [vp]),
        "hs_ctx_ledger_read": (sz, [vp, C.POINTER(LedgerEntry), sz]),
        "hs_ctx_ledger_clear": (None, [vp]),
        "hs_bspd1_probe": (C.c_int, [C.c_char_p, C.POINTER(sz), C.POINTER(sz)]),
        "hs_bspd1_read": (C.c_int, [C.c_char_p, dp, sz]),
        "hs_bspd1_write": (C.c_int, [C.c_char_p, sz, sz, dp]),
        "hs_vector_probe": (C.c_int, [C.c_char_p, C.POINTER(sz)]),
        "hs_vector_read": (C.c_int, [C.c_char_p, dp, sz]),
        "hs_vector_write": (C.c_int, [C.c_char_p, sz, dp]),
        "hs_matrix_load_bspd1": (C.c_int, [vp, C.c_char_p, C.c_int, pp]),
        "hs_matrix_save_bspd1": (C.c_int, [vp, C.c_char_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


def last_error() -> tuple[str, int, int]:
    L = lib()
    a, b = C.c_int64(-1), C.c_int64(-1)
    L.hs_last_error_payload(C.byref(a), C.byref(b))
    return L.hs_last_error().decode(), a.value, b.value
