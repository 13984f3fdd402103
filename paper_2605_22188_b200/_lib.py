"""Loader for the in-tree libbnbg.so (the sm_100a engine + C-ABI, include/bnbg.h).

There is no CPU fallback: if the shared object is missing or fails to load,
every entry point raises.  Build it with ``make -C paper_2605_22188_b200/csrc``
(or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BNBG_LIB_PATH: load another build of the library (kernel-variant experiments)
LIB_PATH = os.environ.get("BNBG_LIB_PATH") or os.path.join(_HERE, "libbnbg.so")
_lib = None


class RelaxCfgC(C.Structure):
    _fields_ = [("max_iterations", C.c_int), ("gap_tolerance", C.c_double),
                ("check_interval", C.c_int), ("acceleration", C.c_int),
                ("smoothness", C.c_double), ("workers", C.c_int)]


class SolverCfgC(C.Structure):
    _fields_ = [("batch_size", C.c_int), ("memory_budget", C.c_uint64),
                ("time_limit", C.c_double), ("prune_slack", C.c_double),
                ("relax", RelaxCfgC), ("profile", C.c_int), ("workers", C.c_int)]


class CertC(C.Structure):
    _fields_ = [("optimal_value", C.c_double), ("support_len", C.c_int),
                ("support", C.POINTER(C.c_int32)), ("coefficients", C.POINTER(C.c_double)),
                ("gap_percent", C.c_double), ("lower_bound", C.c_double),
                ("nodes_processed", C.c_longlong), ("lb_batches", C.c_longlong),
                ("reopt_batches", C.c_longlong), ("batch_size_used", C.c_int),
                ("lower_bound_seconds", C.c_double), ("reoptimization_seconds", C.c_double),
                ("transfer_seconds", C.c_double), ("branch_generate_seconds", C.c_double),
                ("total_seconds", C.c_double), ("status", C.c_int),
                ("relax_iterations", C.c_longlong), ("node_iterations", C.c_longlong),
                ("reopt_supports", C.c_longlong), ("device_seconds", C.c_double)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                           C.POINTER(C.c_int64))


class CommOpsC(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_int), ("world", C.c_int),
                ("allgather", ALLGATHER_FN), ("alltoallv", ALLTOALLV_FN)]


TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_double)
DUAL_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_int32), C.c_int,
                        C.POINTER(C.c_int32), C.c_double)
BOUNDARY_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_double, C.c_double)

dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")

#: every symbol declared in include/bnbg.h
EXPORTS = [
    "bnbg_relax_cfg_default", "bnbg_solver_cfg_default", "bnbg_auto_batch_size",
    "bnbg_generate_synthetic", "bnbg_validate", "bnbg_create", "bnbg_destroy",
    "bnbg_last_error", "bnbg_smoothness", "bnbg_relax_batch", "bnbg_pack_batch",
    "bnbg_round_support",
    "bnbg_select_branch", "bnbg_reoptimize", "bnbg_prox_step", "bnbg_conjugate_prox",
    "bnbg_g_value", "bnbg_g_conjugate", "bnbg_gemm", "bnbg_solve", "bnbg_collect_rashomon",
    "bnbg_pool_size", "bnbg_pool_record", "bnbg_pool_free", "bnbg_kernel_launches",
    "bnbg_gemm_stats", "bnbg_set_timing", "bnbg_kernel_stats", "bnbg_transfer_bytes",
    "bnbg_pass_profile", "bnbg_nccl_unique_id", "bnbg_nccl_init", "bnbg_solve_sharded",
    "bnbg_balance_plan", "bnbg_pool_root", "bnbg_pool_relax", "bnbg_pool_branch",
    "bnbg_shard_stats",
]


def lib():
    """The loaded libbnbg.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build the CUDA engine first "
                          "(make -C paper_2605_22188_b200/csrc); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    d, i, u64, vp, ll = C.c_double, C.c_int, C.c_uint64, C.c_void_p, C.c_longlong
    L.bnbg_relax_cfg_default.argtypes = [C.POINTER(RelaxCfgC)]
    L.bnbg_relax_cfg_default.restype = None
    L.bnbg_solver_cfg_default.argtypes = [C.POINTER(SolverCfgC)]
    L.bnbg_solver_cfg_default.restype = None
    L.bnbg_auto_batch_size.argtypes = [u64, i, i, i, i]
    L.bnbg_generate_synthetic.argtypes = [i, i, i, d, i, d, u64, dp, dp, ip]
    L.bnbg_validate.argtypes = [dp, dp, i, i, i, i, d, d]
    L.bnbg_create.argtypes = [dp, dp, i, i, i, i, d, d, d, i, C.POINTER(vp)]
    L.bnbg_destroy.argtypes = [vp]
    L.bnbg_destroy.restype = None
    L.bnbg_last_error.argtypes = [vp]
    L.bnbg_last_error.restype = C.c_char_p
    L.bnbg_smoothness.argtypes = [vp]
    L.bnbg_smoothness.restype = d
    L.bnbg_relax_batch.argtypes = [vp, C.POINTER(RelaxCfgC), i, up, ip, dp, d, dp, dp, ip, ip,
                                   TRACE_FN, vp]
    L.bnbg_round_support.argtypes = [vp, i, dp, up, ip, ip, ip, ip, ip]
    L.bnbg_select_branch.argtypes = [vp, i, dp, up, ip]
    L.bnbg_pack_batch.argtypes = [vp, i, ip, ip, ip, ip, up, ip, ip]
    L.bnbg_shard_stats.argtypes = [vp, C.POINTER(C.c_longlong), i]
    L.bnbg_reoptimize.argtypes = [vp, i, ip, ip, dp, dp]
    L.bnbg_prox_step.argtypes = [i, i, i, dp, d, d, up, ip, d, dp]
    L.bnbg_conjugate_prox.argtypes = [i, i, i, dp, d, up, ip, d, dp]
    L.bnbg_g_value.argtypes = [i, i, i, dp, up, ip, d, dp]
    L.bnbg_g_conjugate.argtypes = [i, i, i, dp, up, ip, d, dp]
    L.bnbg_gemm.argtypes = [vp, i, i, dp, dp]
    L.bnbg_solve.argtypes = [vp, C.POINTER(SolverCfgC), C.POINTER(CertC), DUAL_HOOK,
                             BOUNDARY_HOOK, vp]
    L.bnbg_collect_rashomon.argtypes = [vp, C.POINTER(SolverCfgC), d, ll, C.POINTER(CertC),
                                        C.POINTER(vp)]
    L.bnbg_pool_size.argtypes = [vp]
    L.bnbg_pool_record.argtypes = [vp, i, ip, dp, C.POINTER(d)]
    L.bnbg_pool_free.argtypes = [vp]
    L.bnbg_pool_free.restype = None
    L.bnbg_kernel_launches.argtypes = [vp]
    L.bnbg_kernel_launches.restype = ll
    L.bnbg_gemm_stats.argtypes = [vp, C.POINTER(d), C.POINTER(d), C.POINTER(ll)]
    L.bnbg_set_timing.argtypes = [vp, i]
    L.bnbg_set_timing.restype = None
    L.bnbg_kernel_stats.argtypes = [vp, i, C.POINTER(d), C.POINTER(d), C.POINTER(ll)]
    L.bnbg_transfer_bytes.argtypes = [vp, C.POINTER(ll), C.POINTER(ll)]
    L.bnbg_pass_profile.argtypes = [vp, dp, i]
    L.bnbg_pool_root.argtypes = [vp, i]
    L.bnbg_pool_relax.argtypes = [vp, C.POINTER(RelaxCfgC), i, ip, d, dp, ip, ip, ip, ip]
    L.bnbg_pool_branch.argtypes = [vp, i, dp, d, ip, C.POINTER(C.c_int32), ip, dp]
    L.bnbg_nccl_unique_id.argtypes = [C.c_char_p]
    L.bnbg_nccl_init.argtypes = [vp, C.c_char_p, i, i]
    L.bnbg_solve_sharded.argtypes = [vp, C.POINTER(SolverCfgC), C.POINTER(CommOpsC),
                                     C.POINTER(CertC)]
    i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
    L.bnbg_balance_plan.argtypes = [i, i64p, i64p]
    _lib = L
    return L
