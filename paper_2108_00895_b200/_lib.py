"""ctypes binding of the C-ABI in include/sskm_b200.h (libsskm_b200.so).

There is no CPU fallback: if the native library is missing and cannot be
built, importing the package fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _build

SSKM_OK, SSKM_EINVAL, SSKM_ERUNTIME = 0, 1, 2
MODES = {"baseline": 0, "ncc": 1, "ncc+index": 2}
STOP_REASONS = ("no_reassignments", "centroid_drift", "max_iterations")


class sskm_run_config(C.Structure):
    _fields_ = [
        ("k", C.c_uint32),
        ("mode", C.c_int32),
        ("lambdas", C.POINTER(C.c_double)),
        ("n_lambdas", C.c_uint32),
        ("conv_sq_dist", C.c_double),
        ("ncc_epsilon", C.c_double),
        ("index_activation_threshold", C.c_uint32),
        ("max_iters", C.c_uint32),
        ("seed", C.c_uint64),
        ("threads", C.c_uint32),
        ("device", C.c_int32),
    ]


class sskm_iteration_stats(C.Structure):
    _fields_ = [
        ("iteration", C.c_uint32),
        ("n_unchanged_centroids", C.c_uint32),
        ("n_reassigned", C.c_uint64),
        ("dot_products", C.c_uint64),
        ("index_queries", C.c_uint64),
        ("candidates_total", C.c_uint64),
        ("wall_seconds", C.c_double),
        ("index_build_seconds", C.c_double),
        ("max_sq_drift", C.c_double),
        ("objective", C.c_double),
        ("index_active", C.c_int32),
        ("n_repaired", C.c_int32),
        ("gpu_dot_products", C.c_uint64),
        ("n_moved", C.c_uint64),
        ("n_changed", C.c_uint32),
        ("n_recomputed", C.c_uint32),
        ("n_rescan", C.c_uint64),
        ("n_exact", C.c_uint64),
        ("update_ms", C.c_double),
        ("assign_ms", C.c_double),
        ("assign_kernel_ms", C.c_double),
        ("screen_ms", C.c_double),
        ("screen_launches", C.c_uint32),
        ("second_pass_docs", C.c_uint32),
        ("centroid_density", C.c_double),
        ("bound_docs", C.c_uint64),
        ("bound_pairs", C.c_uint64),
        ("bound_candidates", C.c_uint64),
        ("bound_doc_nnz", C.c_uint64),
        ("bound_cand_nnz", C.c_uint64),
        ("bound_theta", C.c_double),
        ("bound_visits", C.c_uint64),
        ("bound_own_dots", C.c_uint64),
        ("skip_docs", C.c_uint64),
        ("bound_own_nnz", C.c_uint64),
        ("reserved2", C.c_uint64),
        ("skip_ms", C.c_double),
    ]


_P = C.c_void_p
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_CFG = C.POINTER(sskm_run_config)
_ST = C.POINTER(sskm_iteration_stats)

# (name, restype, argtypes) for every symbol the header declares.
SIGNATURES = [
    ("sskm_last_error", C.c_char_p, []),
    ("sskm_validate", C.c_int, [_CFG, C.c_uint64]),
    ("sskm_open", C.c_int, [C.c_int32, C.POINTER(_P)]),
    ("sskm_close", C.c_int, [_P]),
    ("sskm_upload_csr", C.c_int, [_P, C.c_int64, C.c_uint32, _i64p, _i32p, _f32p, C.c_int64, C.c_int64]),
    ("sskm_configure", C.c_int, [_P, _CFG]),
    ("sskm_init_from_seeds", C.c_int, [_P, _u32p]),
    ("sskm_init_kmeanspp", C.c_int, [_P, C.c_uint64, _u32p]),
    ("sskm_update", C.c_int, [_P, _ST]),
    ("sskm_assign", C.c_int, [_P, _ST]),
    ("sskm_step", C.c_int, [_P, _ST]),
    ("sskm_step_n", C.c_int, [_P, C.c_uint32, _ST]),
    ("sskm_run", C.c_int, [_P, _ST, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_int32)]),
    ("sskm_get_state", C.c_int, [_P, _u32p, _f64p, _u8p]),
    ("sskm_set_state", C.c_int, [_P, _u32p, _f64p, C.c_uint32]),
    ("sskm_get_centroids", C.c_int, [_P, _f32p]),
    ("sskm_get_centroid_rows", C.c_int, [_P, C.c_uint32, _u32p, _f32p]),
    ("sskm_get_centroid_cols", C.c_int, [_P, C.c_uint32, _u32p, _f32p]),
    ("sskm_set_centroids", C.c_int, [_P, _f32p]),
    ("sskm_debug_check_postings", C.c_int, [_P, C.POINTER(C.c_int64)]),
    ("sskm_get_repaired", C.c_int, [_P, _u32p, C.POINTER(C.c_uint32)]),
    ("sskm_get_iteration", C.c_int, [_P, C.POINTER(C.c_uint32)]),
    ("sskm_cluster_csr", C.c_int, [_CFG, C.c_int64, C.c_uint32, _i64p, _i32p, _f32p, _P, _P, _P, _P,
                                   _ST, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_double)]),
    ("sskm_release_cache", C.c_int, []),
    # multi-device context (one host thread, several GPUs, peer-memory exchange)
    ("sskm_multi_open", C.c_int, [C.c_int32, _i32p, C.POINTER(_P)]),
    ("sskm_multi_close", C.c_int, [_P]),
    ("sskm_multi_upload_csr", C.c_int, [_P, C.c_int64, C.c_uint32, _i64p, _i32p, _f32p]),
    ("sskm_multi_configure", C.c_int, [_P, _CFG]),
    ("sskm_multi_init_from_seeds", C.c_int, [_P, _u32p]),
    ("sskm_multi_step", C.c_int, [_P, _ST]),
    ("sskm_multi_run", C.c_int, [_P, _ST, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_int32)]),
    ("sskm_multi_get_state", C.c_int, [_P, _P, _P]),
    ("sskm_multi_get_centroids", C.c_int, [_P, _f32p]),
    ("sskm_multi_launch_count", C.c_int, [_P, C.POINTER(C.c_uint64)]),
    ("sskm_cluster_csr_multi", C.c_int, [_CFG, C.c_int32, _i32p, C.c_int64, C.c_uint32, _i64p, _i32p, _f32p, _P,
                                         _P, _P, _P, _ST, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_int32),
                                         C.POINTER(C.c_double)]),
    ("sskm_local_counts", C.c_int, [_P, _i64p]),
    ("sskm_local_candidates", C.c_int, [_P, C.c_int64, _f64p, _i64p, _u32p, C.POINTER(C.c_int64)]),
    ("sskm_move_doc", C.c_int, [_P, C.c_int64, C.c_uint32]),
    ("sskm_moved_prepare", C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("sskm_moved_pack", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("sskm_init_from_rows", C.c_int, [_P, _i64p, _i32p, _f32p]),
    ("sskm_update_apply", C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _u32p, C.c_uint32, _ST]),
    ("sskm_local_sims_sum", C.c_int, [_P, C.POINTER(C.c_double)]),
    ("sskm_timer_record", C.c_int, [_P, C.c_int32]),
    ("sskm_timer_elapsed", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_double)]),
    ("sskm_launch_count", C.c_int, [_P, C.POINTER(C.c_uint64)]),
    ("sskm_synchronize", C.c_int, [_P]),
    ("sskm_postings_work", C.c_int, [_P, C.POINTER(C.c_uint64)]),
    # extension (not in the reference): teacher-forcing of the NCC flags
    ("sskm_set_unchanged", C.c_int, [_P, _u8p]),
    # GPU TF-IDF ingestion (vectorize_corpus, corpus.cpp:101-134)
    ("sskm_vectorize", C.c_int, [C.c_int32, C.c_int64, C.c_char_p, _i64p, C.c_int64, C.c_char_p, _i64p, C.c_double,
                                 C.POINTER(_P)]),
    ("sskm_vec_sizes", C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint32), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("sskm_vec_export", C.c_int, [_P, _i64p, _i32p, _f64p, _i64p, _i64p, _u32p, C.c_char_p, _i64p]),
    ("sskm_vec_stats", C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64)]),
    ("sskm_vec_free", C.c_int, [_P]),
    ("sskm_normalize_csr", C.c_int, [C.c_int32, C.c_int64, _i64p, _i32p, _f64p, _i64p, _i32p, _f64p]),
]

_lib = None


def lib_path() -> str:
    return _build.LIB


def load():
    """Load (building in-tree first if stale) the native library."""
    global _lib
    if _lib is not None:
        return _lib
    override = os.environ.get("SSKM_LIB")  # experiments: load a specific build
    if override:
        lib = C.CDLL(override)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name, None)  # an older build (A/B runs) may lack newer entry points
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib
    if _build.stale():
        try:
            _build.build()
        except Exception as e:  # no silent fallback, and never a stale binary
            raise ImportError(f"libsskm_b200.so is missing or out of date and could not be built: {e}") from e
    lib = C.CDLL(_build.LIB)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == SSKM_OK:
        return
    msg = load().sskm_last_error().decode()
    if rc == SSKM_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)
