"""ctypes view of libcosched.so (include/cosched.h). Argument marshalling only.

The library is built in-tree (paper_2405_03838_b200/build.py, called by
__graft_entry__.build()). If it is missing this module raises: there is no
Python or CPU fallback for any step of the search.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# COSCHED_LIB_PATH: an alternative build of the same library (compile-time
# variants for A/B timing, tools/build_variants.py); the default is the in-tree build
SO_PATH = os.environ.get("COSCHED_LIB_PATH") or os.path.join(HERE, "libcosched.so")

STATUS = {0: "OK", 2: "INFEASIBLE", 10: "E_ARG", 11: "E_INVALID_ALLOCATION", 12: "E_UNKNOWN_KEY",
          13: "E_DEGENERATE_PROFILE", 14: "E_RANGE", 15: "E_STATE", 20: "E_CUDA", 21: "E_NCCL", 22: "E_OOM"}
OK, INFEASIBLE = 0, 2


class Desc(ctypes.Structure):
    _fields_ = [
        ("n_slots", ctypes.c_int32), ("gpcs_total", ctypes.c_int32), ("n_states", ctypes.c_int32),
        ("state_gpcs", ctypes.c_void_p), ("state_mem", ctypes.c_void_p), ("state_slice", ctypes.c_void_p),
        ("n_slices", ctypes.c_int32), ("n_caps", ctypes.c_int32),
        ("caps_w", ctypes.c_void_p), ("coef_c", ctypes.c_void_p), ("coef_d", ctypes.c_void_p),
        ("objective", ctypes.c_int32), ("alpha", ctypes.c_float),
    ]


class Out(ctypes.Structure):
    _fields_ = [("obj", ctypes.c_void_p), ("cfg", ctypes.c_void_p),
                ("first_set", ctypes.c_int64), ("n_sets", ctypes.c_int64)]


class FitDesc(ctypes.Structure):
    _fields_ = [
        ("n_slices", ctypes.c_int32), ("n_caps", ctypes.c_int32), ("n_partners", ctypes.c_int32),
        ("n_apps", ctypes.c_int64), ("features", ctypes.c_void_p),
        ("n_solo", ctypes.c_int64), ("solo_app", ctypes.c_void_p), ("solo_key", ctypes.c_void_p),
        ("solo_rperf", ctypes.c_void_p),
        ("n_corun", ctypes.c_int64), ("co_app", ctypes.c_void_p), ("co_partners", ctypes.c_void_p),
        ("co_key", ctypes.c_void_p), ("co_rperf", ctypes.c_void_p),
    ]


class FitOut(ctypes.Structure):
    _fields_ = [("coef_c", ctypes.c_void_p), ("coef_d", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("count", ctypes.c_void_p), ("rms", ctypes.c_void_p)]


class TruthDesc(ctypes.Structure):
    _fields_ = [("g_full", ctypes.c_int32), ("n_modules", ctypes.c_int32), ("modules", ctypes.c_int32 * 17),
                ("w_base", ctypes.c_float), ("w_gpc", ctypes.c_float), ("kappa", ctypes.c_float),
                ("f_min", ctypes.c_float), ("p_max", ctypes.c_float)]


class EvalOut(ctypes.Structure):
    _fields_ = [("prop_obj", ctypes.c_void_p), ("prop_fair", ctypes.c_void_p), ("best_obj", ctypes.c_void_p),
                ("worst_obj", ctypes.c_void_p)]


class EvalSummary(ctypes.Structure):
    _fields_ = [("n_compared", ctypes.c_int64), ("n_violations", ctypes.c_int64),
                ("geomean_prop_over_best", ctypes.c_double), ("geomean_worst_over_best", ctypes.c_double)]


FIT_OK, FIT_NO_SAMPLES, FIT_INSUFFICIENT, FIT_RANK_DEFICIENT, FIT_MISSING_C = 0, 1, 2, 3, 4

# (name, restype, argtypes) for every symbol include/cosched.h declares
P = ctypes.c_void_p
I32, I64, U64, F32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
SIGNATURES = [
    ("cosched_create", I32, [ctypes.POINTER(Desc), ctypes.c_int, ctypes.POINTER(P)]),
    ("cosched_destroy", None, [P]),
    ("cosched_last_error", ctypes.c_char_p, [P]),
    ("cosched_last_create_error", ctypes.c_char_p, []),
    ("cosched_get_unique_id", I32, [P]),
    ("cosched_set_comm", I32, [P, P, ctypes.c_int, ctypes.c_int]),
    ("cosched_shard_range", I32, [P, I64, P, P]),
    ("cosched_shard_range_for", I32, [I64, I32, I32, I32, P, P]),
    ("cosched_n_sets", I64, [I64, I32]),
    ("cosched_unrank", I32, [I64, I32, I64, P]),
    ("cosched_pack_key", U64, [F32, I64]),
    ("cosched_unpack_key", None, [U64, P, P]),
    ("cosched_workspace_size", I32, [P, I64, P]),
    ("cosched_score_all", I32, [P, P, I64, P, I64, P, ctypes.c_size_t, ctypes.POINTER(Out), P]),
    ("cosched_local_best_key", I32, [P, P]),
    ("cosched_best_set", I32, [P, P, P, P]),
    ("cosched_best_set_begin", I32, [P]),
    ("cosched_last_step_ms", I32, [P, P]),
    ("cosched_set_timing", I32, [P, I32]),
    ("cosched_best_set_end", I32, [P, P, P, P]),
    ("cosched_best_config", I32, [P, I64, P, P, P, P, P]),
    ("cosched_best_allocation", I32, [P, I32, P, P, P, P]),
    ("cosched_set_variant", I32, [P, ctypes.c_int]),
    ("cosched_set_search", I32, [P, ctypes.c_int, I32, I32]),
    ("cosched_last_search_evals", I32, [P, P]),
    ("cosched_set_shard_view", I32, [P, ctypes.c_int, ctypes.c_int]),
    ("cosched_last_timings", I32, [P, P]),
    ("cosched_kernel_launches", I64, [P]),
    ("cosched_last_greedy_rounds", I64, [P]),
    ("cosched_last_rescored", I32, [P, P]),
    ("cosched_node_workspace_size", I32, [P, I64, I32, ctypes.c_double, P]),
    ("cosched_node_budget", I32, [P, I64, P, I32, ctypes.c_double, I32, P, ctypes.c_size_t, P, P, P, P]),
    ("cosched_evaluate_workspace_size", I32, [P, I64, P]),
    ("cosched_evaluate_truth", I32, [P, ctypes.POINTER(TruthDesc), P, I64, P, P, ctypes.c_size_t,
                                     ctypes.POINTER(EvalOut), ctypes.POINTER(EvalSummary), P]),
    ("cosched_fit_workspace_size", I32, [ctypes.POINTER(FitDesc), P]),
    ("cosched_fit", I32, [ctypes.POINTER(FitDesc), P, ctypes.c_size_t, ctypes.POINTER(FitOut), P]),
    ("cosched_fit_last_error", ctypes.c_char_p, []),
]

_lib = None


def load():
    """Load libcosched.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"{SO_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                               "There is no CPU fallback.")
        lib = ctypes.CDLL(SO_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
