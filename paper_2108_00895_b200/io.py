"""Corpus files and run reports.

* `load_matrix` / `write_matrix`: the reference's text matrix format with its
  `.ids` sidecar (corpus.cpp:182-272), parsed natively in parallel, same checks
  and error messages (`<path>:<line>: <what>` → RuntimeError).
* `save_csr` / `load_csr`: a binary CSR format ("SSKMCSR1") for fast reloads.
* `make_report` / `to_json` / `write_report`: the reference's RunReport JSON
  (report.cpp:10-86), same keys, nesting, totals and formatting.
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Optional

import numpy as np

from . import _lib
from .api import ClusteringResult, CorpusMatrix

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_bound = False


def _io():
    global _bound
    lib = _lib.load()
    if not _bound:
        sig = [
            ("sskm_io_last_error", C.c_char_p, []),
            ("sskm_io_load_matrix", C.c_void_p, [C.c_char_p, C.c_double, C.c_int]),
            ("sskm_io_sizes", None, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            ("sskm_io_export", None, [C.c_void_p, _i64p, _i32p, _f32p, C.c_void_p, C.c_void_p]),
            ("sskm_io_free", None, [C.c_void_p]),
            ("sskm_io_write_matrix", C.c_int, [C.c_char_p, C.c_int64, C.c_uint32, _i64p, _i32p, _f32p, C.c_char_p]),
            ("sskm_io_save_csr", C.c_int, [C.c_char_p, C.c_int64, C.c_uint32, _i64p, _i32p, _f32p]),
            ("sskm_io_csr_header", C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_uint32),
                                             C.POINTER(C.c_int64)]),
            ("sskm_io_csr_read", C.c_int, [C.c_char_p, _i64p, _i32p, _f32p]),
        ]
        for name, res, args in sig:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _bound = True
    return lib


def _err(lib, rc):
    msg = lib.sskm_io_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def load_matrix(path: str, norm_tol: float = 1e-9, threads: int = 0, keep_f64: bool = False) -> CorpusMatrix:
    """load_matrix (corpus.cpp:201-272). Rows must be unit length within
    `norm_tol` in fp64 (the reference uses 1e-9; files holding fp32-rounded
    rows need ~1e-6). Values are stored fp32; `keep_f64` also keeps the parsed
    doubles as `m.values_f64`."""
    lib = _io()
    h = lib.sskm_io_load_matrix(path.encode(), float(norm_tol), int(threads))
    if not h:
        raise RuntimeError(lib.sskm_io_last_error().decode())
    try:
        n, d, nnz, ib = C.c_int64(), C.c_uint32(), C.c_int64(), C.c_int64()
        lib.sskm_io_sizes(h, C.byref(n), C.byref(d), C.byref(nnz), C.byref(ib))
        indptr = np.zeros(n.value + 1, np.int64)
        idx = np.zeros(max(nnz.value, 1), np.int32)
        val = np.zeros(max(nnz.value, 1), np.float32)
        v64 = np.zeros(max(nnz.value, 1), np.float64) if keep_f64 else None
        ids = C.create_string_buffer(max(ib.value, 1))
        lib.sskm_io_export(h, indptr, idx, val, v64.ctypes.data if v64 is not None else None, ids)
    finally:
        lib.sskm_io_free(h)
    doc_ids = ids.raw[: ib.value].decode().split("\n")[:-1] if ib.value else []
    m = CorpusMatrix.from_csr(indptr, idx[: nnz.value], val[: nnz.value], d.value, doc_ids=doc_ids)
    if keep_f64:
        m.values_f64 = v64[: nnz.value]
    return m


def write_matrix(path: str, m: CorpusMatrix) -> None:
    """write_matrix (corpus.cpp:182-199): %.17g of the stored weights + `.ids`."""
    lib = _io()
    ids = None
    if m.doc_ids:
        ids = ("\n".join(m.doc_ids) + "\n").encode()
    rc = lib.sskm_io_write_matrix(path.encode(), m.n_docs, m.dims, m.indptr, m.indices, m.values, ids)
    if rc:
        _err(lib, rc)


def save_csr(path: str, m: CorpusMatrix) -> None:
    lib = _io()
    rc = lib.sskm_io_save_csr(path.encode(), m.n_docs, m.dims, m.indptr, m.indices, m.values)
    if rc:
        _err(lib, rc)


def load_csr(path: str) -> CorpusMatrix:
    lib = _io()
    n, d, nnz = C.c_int64(), C.c_uint32(), C.c_int64()
    rc = lib.sskm_io_csr_header(path.encode(), C.byref(n), C.byref(d), C.byref(nnz))
    if rc:
        _err(lib, rc)
    indptr = np.zeros(n.value + 1, np.int64)
    idx = np.zeros(max(nnz.value, 1), np.int32)
    val = np.zeros(max(nnz.value, 1), np.float32)
    rc = lib.sskm_io_csr_read(path.encode(), indptr, idx, val)
    if rc:
        _err(lib, rc)
    return CorpusMatrix.from_csr(indptr, idx[: nnz.value], val[: nnz.value], d.value)


# ------------------------------------------------------------------ report --
_ITER_KEYS = ("iteration", "n_reassigned", "n_unchanged_centroids", "dot_products", "index_queries",
              "candidates_total", "wall_seconds", "index_build_seconds", "index_active", "max_sq_drift", "objective")


def make_report(config: dict, data: CorpusMatrix, result: ClusteringResult,
                dropped_doc_ids: Optional[list] = None) -> dict:
    """make_report (report.cpp:10-22). `config` holds the RunConfig fields
    (k, mode, lambdas, conv_sq_dist, ncc_epsilon, index_activation_threshold,
    max_iters, seed, threads)."""
    defaults = dict(mode="baseline", lambdas=[0.1, 0.25, 0.4, 0.6], conv_sq_dist=0.0001, ncc_epsilon=0.0,
                    index_activation_threshold=100, max_iters=100, seed=0, threads=0)
    cfg = {**defaults, **config}
    iters = [{key: (bool(getattr(it, key)) if key == "index_active" else getattr(it, key)) for key in _ITER_KEYS}
             for it in result.iterations]
    sizes = np.bincount(np.asarray(result.assignments, np.int64), minlength=int(cfg["k"])).tolist()
    return {
        "config": {key: (list(cfg[key]) if key == "lambdas" else cfg[key])
                   for key in ("k", "mode", "lambdas", "conv_sq_dist", "ncc_epsilon", "index_activation_threshold",
                               "max_iters", "seed", "threads")},
        "n_docs": data.n_docs,
        "dims": data.dims,
        "iterations": iters,
        "totals": {
            "iterations": len(iters),
            "dot_products": sum(it["dot_products"] for it in iters),
            "index_queries": sum(it["index_queries"] for it in iters),
            "candidates_total": sum(it["candidates_total"] for it in iters),
            "n_reassigned": sum(it["n_reassigned"] for it in iters),
            "wall_seconds": sum(it["wall_seconds"] for it in iters),
            "index_build_seconds": sum(it["index_build_seconds"] for it in iters),
        },
        "objective": result.objective,
        "stop_reason": result.stop_reason,
        "dropped_doc_ids": list(dropped_doc_ids or []),
        "cluster_sizes": sizes,
    }


def to_json(report: dict) -> str:
    """to_json (report.cpp:24-79) exactly as the reference's nlohmann dump(2)
    prints it: sorted keys, 2-space indent, one array element per line — except
    `cluster_sizes` (a std::vector<uint64_t>), which that dump prints inline."""
    tmp = dict(report)
    sizes = tmp.pop("cluster_sizes", None)
    if sizes is not None:
        tmp["cluster_sizes"] = "@@CLUSTER_SIZES@@"
    out = json.dumps(tmp, indent=2, sort_keys=True, separators=(",", ": "))
    if sizes is not None:
        out = out.replace('"@@CLUSTER_SIZES@@"', "[" + ",".join(str(int(x)) for x in sizes) + "]")
    return out + "\n"


def write_report(path: str, report: dict) -> None:
    with open(path, "w") as f:
        f.write(to_json(report))
