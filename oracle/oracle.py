"""TEST INFRASTRUCTURE ONLY — ctypes front end for the CPU oracle.

Two interchangeable backends with one Python interface:

* ``"ref"``  — oracle/_ref/libsskm_ref.so: the UNMODIFIED reference C++ engine
  (/root/reference/proj/src/{engine,sparse_vector,parallel,prune_index,synthetic}.cpp)
  behind oracle/ref_shim.cpp, built by oracle/Makefile.
* ``"port"`` — oracle/libsskm_oracle.so: the plain-C restatement (oracle/sskm_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
legs may import this module; the product package never does.

The ``Stepper`` mirrors the reference tests' per-iteration driver
(proj/tests/test_engine.cpp:54-100): ``update()`` is compute_centroids + detect_unchanged
(engine.cpp:361-378) and ``assign()`` is assign + the objective sum (engine.cpp:394-405).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsskm_ref.so")
PORT_SO = os.path.join(HERE, "libsskm_oracle.so")

_P = C.c_void_p
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class CStats(C.Structure):
    # field order = engine.hpp:43-57 IterationStats (+ n_repaired)
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
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class OracleError(RuntimeError):
    pass


def build(ref: bool | None = None) -> None:
    """Build the oracle libraries (ref only when /root/reference is present)."""
    targets = ["port"]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/src")
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


_libs: dict = {}


def _load(kind: str):
    if kind in _libs:
        return _libs[kind]
    path = REF_SO if kind == "ref" else PORT_SO
    if not os.path.exists(path):
        if kind == "ref" and not os.path.isdir("/root/reference/proj/src"):
            raise OracleError(f"reference oracle not built ({path}) and /root/reference absent")
        build(ref=(kind == "ref"))
    lib = C.CDLL(path)
    if kind == "ref":
        lib.sref_last_error.restype = C.c_char_p
        lib.sref_corpus_from_csr.restype = _P
        lib.sref_corpus_from_csr.argtypes = [C.c_int64, C.c_uint32, _i64p, _i32p, _f64p]
        lib.sref_corpus_free.argtypes = [_P]
        lib.sref_corpus_nnz.restype = C.c_int64
        lib.sref_corpus_nnz.argtypes = [_P]
        lib.sref_corpus_n.restype = C.c_int64
        lib.sref_corpus_n.argtypes = [_P]
        lib.sref_corpus_dims.restype = C.c_uint32
        lib.sref_corpus_dims.argtypes = [_P]
        lib.sref_corpus_export.argtypes = [_P, _i64p, _u32p, _f64p]
        lib.sref_synthetic_zipf.restype = _P
        lib.sref_synthetic_zipf.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, C.c_uint64]
        lib.sref_dot.argtypes = [C.c_int64, _u32p, _f64p, C.c_int64, _u32p, _f64p, C.POINTER(C.c_double)]
        lib.sref_normalize.argtypes = [C.c_int64, _u32p, _f64p, C.POINTER(C.c_int64)]
        lib.sref_stepper_new.restype = _P
        lib.sref_stepper_new.argtypes = [_P, C.c_uint32, C.c_char_p, C.c_double, C.c_double,
                                         C.c_uint32, C.c_uint32, C.c_uint32]
        lib.sref_stepper_free.argtypes = [_P]
        lib.sref_stepper_new_sample.restype = _P
        lib.sref_stepper_new_sample.argtypes = [_P, C.c_uint32, C.c_char_p, C.c_double, C.c_uint32]
        lib.sref_stepper_cols_nnz.restype = C.c_int64
        lib.sref_stepper_cols_nnz.argtypes = [_P, C.c_int64, _u32p]
        lib.sref_stepper_get_cols.argtypes = [_P, C.c_int64, _u32p, _i64p, _u32p, _f64p]
        lib.sref_stepper_init_seeds.argtypes = [_P, _u32p, C.POINTER(CStats)]
        lib.sref_stepper_init_kmeanspp.argtypes = [_P, C.c_uint64, _u32p]
        lib.sref_stepper_step.argtypes = [_P, C.POINTER(CStats)]
        lib.sref_stepper_update.argtypes = [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
        lib.sref_stepper_assign.argtypes = [_P, C.c_uint32, C.c_double, C.POINTER(CStats)]
        lib.sref_stepper_iteration.restype = C.c_uint32
        lib.sref_stepper_iteration.argtypes = [_P]
        lib.sref_stepper_get_state.argtypes = [_P, _u32p, _f64p, _u8p]
        lib.sref_stepper_set_state.argtypes = [_P, _u32p, _f64p, _u8p, C.c_uint32]
        lib.sref_stepper_repaired.argtypes = [_P, _u32p, C.POINTER(C.c_int64)]
        lib.sref_stepper_centroids_nnz.restype = C.c_int64
        lib.sref_stepper_centroids_nnz.argtypes = [_P]
        lib.sref_stepper_get_centroids.argtypes = [_P, _i64p, _u32p, _f64p]
        lib.sref_stepper_set_centroids.argtypes = [_P, _i64p, _u32p, _f64p]
        lib.sref_compute_centroids.argtypes = [_P, _u32p, _f64p, _u32p, C.POINTER(C.c_int64)]
        lib.sref_run.argtypes = [_P, C.c_uint32, C.c_char_p, C.c_uint64, C.c_double, C.c_double,
                                 C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _f64p,
                                 C.POINTER(CStats), C.c_uint32, C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        lib.sref_seed_kmeanspp.argtypes = [_P, C.c_uint32, C.c_uint64, C.c_uint32, _u32p, _u32p, _f64p]
        lib.sref_validate.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, C.c_uint32,
                                      _f64p, C.c_uint32]
        lib.sref_vectorize.argtypes = [C.c_int64, C.c_char_p, _i64p, C.c_int64, C.c_char_p, _i64p, C.c_double,
                                       C.POINTER(_P)]
        lib.sref_vec_sizes.argtypes = [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint32), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_double)]
        lib.sref_vec_export.argtypes = [_P, _i64p, _u32p, _f64p, _i64p, _i64p, _u32p, C.c_char_p, _i64p]
        lib.sref_vec_free.argtypes = [_P]
        lib.sref_load_matrix.restype = _P
        lib.sref_load_matrix.argtypes = [C.c_char_p]
        lib.sref_write_matrix.argtypes = [C.c_char_p, _P]
        lib.sref_report_json.argtypes = [C.c_uint32, C.c_char_p, _f64p, C.c_uint32, C.c_double, C.c_double,
                                         C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32,
                                         C.POINTER(CStats), C.c_uint32, C.c_double, C.c_int32, _u32p,
                                         C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
    else:
        lib.o_last_error.restype = C.c_char_p
        lib.o_dot.restype = C.c_double
        lib.o_dot.argtypes = [C.c_int64, _u32p, _f64p, C.c_int64, _u32p, _f64p]
        lib.o_normalize.argtypes = [C.c_int64, _u32p, _f64p, C.POINTER(C.c_int64)]
        lib.o_normalize_capped.restype = C.c_uint64
        lib.o_mt64_draw.restype = C.c_uint64
        lib.o_mt64_draw.argtypes = [C.c_uint64, C.c_uint64]
        lib.o_validate.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, C.c_uint32,
                                   _f64p, C.c_uint32]
        lib.o_state_new.restype = _P
        lib.o_state_new.argtypes = [C.c_int64, C.c_uint32, _i64p, _i32p, _f64p, C.c_uint32,
                                    C.c_char_p, C.c_double, C.c_double, C.c_uint32, C.c_uint32]
        lib.o_state_free.argtypes = [_P]
        lib.o_assign.argtypes = [_P, C.POINTER(CStats)]
        lib.o_update.argtypes = [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
        lib.o_step.argtypes = [_P, C.POINTER(CStats)]
        lib.o_init_seeds.argtypes = [_P, _u32p, C.POINTER(CStats)]
        lib.o_seed_kmeanspp.argtypes = [_P, C.c_uint64, _u32p]
        lib.o_run.argtypes = [_P, C.POINTER(CStats), C.c_uint32, C.POINTER(C.c_uint32),
                              C.POINTER(C.c_int32)]
        lib.o_iteration.restype = C.c_uint32
        lib.o_iteration.argtypes = [_P]
        lib.o_get_state.argtypes = [_P, _u32p, _f64p, _u8p]
        lib.o_set_state.argtypes = [_P, _u32p, _f64p, _u8p, C.c_uint32]
        lib.o_centroids_nnz.restype = C.c_int64
        lib.o_centroids_nnz.argtypes = [_P]
        lib.o_get_centroids.argtypes = [_P, _i64p, _u32p, _f64p]
        lib.o_set_centroids.argtypes = [_P, _i64p, _u32p, _f64p]
        lib.o_repaired.restype = C.c_uint32
        lib.o_repaired.argtypes = [_P, _u32p]
        lib.o_compute_centroids.argtypes = [_P]
    _libs[kind] = lib
    return lib


def _check(lib, rc, kind):
    if rc != 0:
        msg = (lib.sref_last_error() if kind == "ref" else lib.o_last_error()).decode()
        if rc == 1:
            raise ValueError(msg)
        raise OracleError(msg)


STOP_REASONS = ("no_reassignments", "centroid_drift", "max_iterations")


class Corpus:
    """CSR corpus with fp64 values (fp32 product values widened)."""

    def __init__(self, indptr, indices, values, dims: int):
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.dims = int(dims)
        self.n = len(self.indptr) - 1
        self._ref = None

    def ref_handle(self):
        if self._ref is None:
            lib = _load("ref")
            h = lib.sref_corpus_from_csr(self.n, self.dims, self.indptr, self.indices, self.values)
            if not h:
                raise ValueError(lib.sref_last_error().decode())
            self._ref = h
        return self._ref

    def __del__(self):
        if self._ref is not None and "ref" in _libs:
            _libs["ref"].sref_corpus_free(self._ref)
            self._ref = None

    def row(self, i):
        b, e = self.indptr[i], self.indptr[i + 1]
        return self.indices[b:e].astype(np.uint32), self.values[b:e]


def reference_synthetic_zipf(n_docs, vocab, avg_nnz=10.0, zipf_s=1.1, seed=0):
    """The reference's own generator (synthetic.cpp:31-68) -> (indptr, indices, values f64, dims)."""
    lib = _load("ref")
    h = lib.sref_synthetic_zipf(n_docs, vocab, avg_nnz, zipf_s, seed)
    if not h:
        raise ValueError(lib.sref_last_error().decode())
    try:
        n = lib.sref_corpus_n(h)
        nnz = lib.sref_corpus_nnz(h)
        ptr = np.zeros(n + 1, np.int64)
        idx = np.zeros(max(nnz, 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float64)
        lib.sref_corpus_export(h, ptr, idx, val)
        return ptr, idx[:nnz].astype(np.int32), val[:nnz], int(lib.sref_corpus_dims(h))
    finally:
        lib.sref_corpus_free(h)


def dot(a_idx, a_val, b_idx, b_val, kind="ref") -> float:
    lib = _load(kind)
    ai = np.ascontiguousarray(a_idx, np.uint32)
    av = np.ascontiguousarray(a_val, np.float64)
    bi = np.ascontiguousarray(b_idx, np.uint32)
    bv = np.ascontiguousarray(b_val, np.float64)
    if kind == "ref":
        out = C.c_double()
        _check(lib, lib.sref_dot(len(ai), ai, av, len(bi), bi, bv, C.byref(out)), kind)
        return out.value
    return lib.o_dot(len(ai), ai, av, len(bi), bi, bv)


def normalize(idx, val, kind="ref"):
    lib = _load(kind)
    i = np.array(idx, np.uint32)
    v = np.array(val, np.float64)
    if len(i) == 0:
        i = np.zeros(1, np.uint32)
        v = np.zeros(1, np.float64)
        n = 0
    else:
        n = len(i)
    out = C.c_int64()
    fn = lib.sref_normalize if kind == "ref" else lib.o_normalize
    _check(lib, fn(n, i, v, C.byref(out)), kind)
    return i[: out.value], v[: out.value]


def validate(n_docs, k, conv_sq_dist=1e-4, ncc_epsilon=0.0, max_iters=100,
             lambdas=(0.1, 0.25, 0.4, 0.6), kind="ref"):
    lib = _load(kind)
    lam = np.ascontiguousarray(lambdas, np.float64) if len(lambdas) else np.zeros(1)
    fn = lib.sref_validate if kind == "ref" else lib.o_validate
    _check(lib, fn(n_docs, k, conv_sq_dist, ncc_epsilon, max_iters, lam, len(lambdas)), kind)


def dense_to_csr(ct: np.ndarray, k: int):
    """Cᵀ (d × ≥k, any float dtype) -> centroid CSR over k rows with fp64 values."""
    cols = np.ascontiguousarray(ct[:, :k].T)
    jj, tt = np.nonzero(cols)
    counts = np.bincount(jj, minlength=k)
    ptr = np.zeros(k + 1, np.int64)
    ptr[1:] = np.cumsum(counts)
    return ptr, tt.astype(np.uint32), cols[jj, tt].astype(np.float64)


def csr_to_dense(ptr, idx, val, k, dims):
    out = np.zeros((dims, k), np.float64)
    for j in range(k):
        b, e = ptr[j], ptr[j + 1]
        out[idx[b:e], j] = val[b:e]
    return out


class Stepper:
    """Per-iteration driver over either backend (test_engine.cpp:54-100)."""

    def __init__(self, corpus: Corpus, k: int, mode="baseline", ncc_epsilon=0.0,
                 conv_sq_dist=1e-4, max_iters=100, threads=0, index_activation_threshold=100,
                 kind="ref", sample=False):
        self.kind = kind
        self.lib = _load(kind)
        self.c = corpus
        self.k = k
        if sample and kind != "ref":
            raise ValueError("sample steppers (k > n) exist for the compiled reference only")
        if sample:  # assign-only stepper over a document sample; k may exceed its size
            h = self.lib.sref_stepper_new_sample(corpus.ref_handle(), k, mode.encode(), ncc_epsilon, threads)
            if not h:
                raise ValueError(self.lib.sref_last_error().decode())
        elif kind == "ref":
            h = self.lib.sref_stepper_new(corpus.ref_handle(), k, mode.encode(), ncc_epsilon,
                                          conv_sq_dist, max_iters, threads,
                                          index_activation_threshold)
            if not h:
                raise ValueError(self.lib.sref_last_error().decode())
        else:
            h = self.lib.o_state_new(corpus.n, corpus.dims, corpus.indptr, corpus.indices,
                                     corpus.values, k, mode.encode(), ncc_epsilon, conv_sq_dist,
                                     max_iters, threads)
            if not h:
                raise ValueError(self.lib.o_last_error().decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            (self.lib.sref_stepper_free if self.kind == "ref" else self.lib.o_state_free)(self.h)
            self.h = None

    def _ck(self, rc):
        _check(self.lib, rc, self.kind)

    def init_seeds(self, seeds):
        s = np.ascontiguousarray(seeds, np.uint32)
        st = CStats()
        fn = self.lib.sref_stepper_init_seeds if self.kind == "ref" else self.lib.o_init_seeds
        self._ck(fn(self.h, s, C.byref(st)))
        return st.as_dict()

    def init_kmeanspp(self, seed):
        out = np.zeros(self.k, np.uint32)
        fn = self.lib.sref_stepper_init_kmeanspp if self.kind == "ref" else self.lib.o_seed_kmeanspp
        self._ck(fn(self.h, seed, out))
        return out

    def step(self):
        st = CStats()
        fn = self.lib.sref_stepper_step if self.kind == "ref" else self.lib.o_step
        self._ck(fn(self.h, C.byref(st)))
        return st.as_dict()

    def update(self):
        nu = C.c_uint32()
        dr = C.c_double()
        fn = self.lib.sref_stepper_update if self.kind == "ref" else self.lib.o_update
        self._ck(fn(self.h, C.byref(nu), C.byref(dr)))
        return nu.value, dr.value

    def assign(self, n_unchanged=0, drift=0.0):
        st = CStats()
        if self.kind == "ref":
            self._ck(self.lib.sref_stepper_assign(self.h, n_unchanged, drift, C.byref(st)))
        else:
            self._ck(self.lib.o_assign(self.h, C.byref(st)))
            st.max_sq_drift = drift
        return st.as_dict()

    @property
    def iteration(self):
        fn = self.lib.sref_stepper_iteration if self.kind == "ref" else self.lib.o_iteration
        return int(fn(self.h))

    def get_state(self):
        a = np.zeros(self.c.n, np.uint32)
        s = np.zeros(self.c.n, np.float64)
        u = np.zeros(self.k, np.uint8)
        if self.kind == "ref":
            self._ck(self.lib.sref_stepper_get_state(self.h, a, s, u))
        else:
            self.lib.o_get_state(self.h, a, s, u)
        return a, s, u

    def set_state(self, a, sims, unchanged, iteration):
        a = np.ascontiguousarray(a, np.uint32)
        s = np.ascontiguousarray(sims, np.float64)
        u = np.ascontiguousarray(unchanged, np.uint8)
        if self.kind == "ref":
            self._ck(self.lib.sref_stepper_set_state(self.h, a, s, u, iteration))
        else:
            self.lib.o_set_state(self.h, a, s, u, iteration)

    def get_centroids_csr(self):
        nnz = (self.lib.sref_stepper_centroids_nnz if self.kind == "ref"
               else self.lib.o_centroids_nnz)(self.h)
        ptr = np.zeros(self.k + 1, np.int64)
        idx = np.zeros(max(nnz, 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float64)
        if self.kind == "ref":
            self._ck(self.lib.sref_stepper_get_centroids(self.h, ptr, idx, val))
        else:
            self.lib.o_get_centroids(self.h, ptr, idx, val)
        return ptr, idx[:nnz], val[:nnz]

    def get_cols_csr(self, cols):
        """CSR (ptr, idx, val) of the centroids `cols` only."""
        cols = np.ascontiguousarray(cols, np.uint32)
        if self.kind != "ref":
            ptr, idx, val = self.get_centroids_csr()
            parts = [(idx[ptr[j]:ptr[j + 1]], val[ptr[j]:ptr[j + 1]]) for j in cols]
            p = np.zeros(len(cols) + 1, np.int64)
            p[1:] = np.cumsum([len(a) for a, _ in parts])
            return (p, np.concatenate([a for a, _ in parts] + [np.zeros(0, np.uint32)]),
                    np.concatenate([b for _, b in parts] + [np.zeros(0)]))
        nnz = self.lib.sref_stepper_cols_nnz(self.h, len(cols), cols)
        ptr = np.zeros(len(cols) + 1, np.int64)
        idx = np.zeros(max(nnz, 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float64)
        self._ck(self.lib.sref_stepper_get_cols(self.h, len(cols), cols, ptr, idx, val))
        return ptr, idx[:nnz], val[:nnz]

    def get_centroids_dense(self):
        return csr_to_dense(*self.get_centroids_csr(), self.k, self.c.dims)

    def set_centroids_csr(self, ptr, idx, val):
        ptr = np.ascontiguousarray(ptr, np.int64)
        idx = np.ascontiguousarray(idx, np.uint32) if len(idx) else np.zeros(1, np.uint32)
        val = np.ascontiguousarray(val, np.float64) if len(val) else np.zeros(1, np.float64)
        if self.kind == "ref":
            self._ck(self.lib.sref_stepper_set_centroids(self.h, ptr, idx, val))
        else:
            self.lib.o_set_centroids(self.h, ptr, idx, val)

    def set_centroids_dense(self, ct):
        self.set_centroids_csr(*dense_to_csr(ct, self.k))

    def repaired(self):
        if self.kind == "ref":
            n = C.c_int64()
            out = np.zeros(self.k, np.uint32)
            self._ck(self.lib.sref_stepper_repaired(self.h, out, C.byref(n)))
            return out[: n.value]
        out = np.zeros(self.k, np.uint32)
        n = self.lib.o_repaired(self.h, out)
        return out[:n]

    def compute_centroids(self, a, sims):
        """compute_centroids on the given state; returns (new assignments, repaired)."""
        a = np.array(a, np.uint32)
        s = np.ascontiguousarray(sims, np.float64)
        if self.kind == "ref":
            rep = np.zeros(self.k, np.uint32)
            n = C.c_int64()
            self._ck(self.lib.sref_compute_centroids(self.h, a, s, rep, C.byref(n)))
            return a, rep[: n.value]
        self.set_state(a, s, self.get_state()[2], self.iteration)
        self._ck(self.lib.o_compute_centroids(self.h))
        a2, _, _ = self.get_state()
        return a2, self.repaired()


def run_seeded(corpus: Corpus, k, seeds, mode="baseline", ncc_epsilon=0.0, conv_sq_dist=1e-4,
               max_iters=100, threads=0, kind="ref", record=False):
    """run() from the BASELINE init (centroids = seed docs), engine.cpp:357-424.

    Returns dict(assignments, sims, centroids (dense d×k fp64), iterations, stop_reason,
    objective[, trace]) where trace holds per-iteration (assignments, sims) when record.
    """
    s = Stepper(corpus, k, mode, ncc_epsilon, conv_sq_dist, max_iters, threads, kind=kind)
    s.init_seeds(seeds)
    its, trace = [], []
    stop = 2
    for it in range(1, max_iters + 1):
        st = s.step()
        its.append(st)
        if record:
            a, sm, u = s.get_state()
            trace.append((a.copy(), sm.copy(), u.copy()))
        if st["n_reassigned"] == 0:
            stop = 0
            break
        if it > 1 and st["max_sq_drift"] < conv_sq_dist:
            stop = 1
            break
    a, sm, _ = s.get_state()
    out = dict(assignments=a, sims=sm, centroids=s.get_centroids_dense(), iterations=its,
               stop_reason=STOP_REASONS[stop], objective=its[-1]["objective"])
    if record:
        out["trace"] = trace
    return out


def run_kmeanspp(corpus: Corpus, k, mode="baseline", seed=0, conv_sq_dist=1e-4, ncc_epsilon=0.0,
                 index_activation_threshold=100, max_iters=100, threads=0):
    """The reference's own sskm::run (engine.cpp:345-425) via the shim."""
    lib = _load("ref")
    a = np.zeros(corpus.n, np.uint32)
    sm = np.zeros(corpus.n, np.float64)
    stats = (CStats * max_iters)()
    n_it = C.c_uint32()
    stop = C.c_int32()
    obj = C.c_double()
    _check(lib, lib.sref_run(corpus.ref_handle(), k, mode.encode(), seed, conv_sq_dist,
                             ncc_epsilon, index_activation_threshold, max_iters, threads, a, sm,
                             stats, max_iters, C.byref(n_it), C.byref(stop), C.byref(obj)), "ref")
    return dict(assignments=a, sims=sm, iterations=[stats[i].as_dict() for i in range(n_it.value)],
                stop_reason=STOP_REASONS[stop.value], objective=obj.value)


def seed_kmeanspp(corpus: Corpus, k, seed, threads=0):
    lib = _load("ref")
    seeds = np.zeros(k, np.uint32)
    a = np.zeros(corpus.n, np.uint32)
    sm = np.zeros(corpus.n, np.float64)
    _check(lib, lib.sref_seed_kmeanspp(corpus.ref_handle(), k, seed, threads, seeds, a, sm), "ref")
    return seeds, a, sm


# ------------------------------------------------------------- corpus IO ----
def ref_load_matrix(path):
    """The reference's load_matrix (corpus.cpp:201-272) -> (indptr, idx, val f64, dims, n)."""
    lib = _load("ref")
    h = lib.sref_load_matrix(path.encode())
    if not h:
        raise OracleError(lib.sref_last_error().decode())
    try:
        n = lib.sref_corpus_n(h)
        nnz = lib.sref_corpus_nnz(h)
        ptr = np.zeros(n + 1, np.int64)
        idx = np.zeros(max(nnz, 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float64)
        lib.sref_corpus_export(h, ptr, idx, val)
        return ptr, idx[:nnz].astype(np.int32), val[:nnz], int(lib.sref_corpus_dims(h))
    finally:
        lib.sref_corpus_free(h)


def ref_write_matrix(path, corpus: Corpus):
    """The reference's write_matrix (corpus.cpp:182-199) of a CSR corpus."""
    lib = _load("ref")
    _check(lib, lib.sref_write_matrix(path.encode(), corpus.ref_handle()), "ref")


def ref_report_json(cfg: dict, n_docs, dims, iterations, objective, stop_reason, assignments) -> str:
    """The reference's to_json(make_report(...)) (report.cpp:10-79)."""
    lib = _load("ref")
    its = (CStats * max(len(iterations), 1))()
    for t, it in enumerate(iterations):
        for f, _ in CStats._fields_:
            if f in it:
                setattr(its[t], f, it[f])
    lam = np.ascontiguousarray(cfg.get("lambdas", [0.1, 0.25, 0.4, 0.6]), np.float64)
    a = np.ascontiguousarray(assignments, np.uint32)
    n = C.c_uint64()
    args = [cfg["k"], cfg.get("mode", "baseline").encode(), lam if len(lam) else np.zeros(1), len(lam),
            cfg.get("conv_sq_dist", 1e-4), cfg.get("ncc_epsilon", 0.0), cfg.get("index_activation_threshold", 100),
            cfg.get("max_iters", 100), cfg.get("seed", 0), cfg.get("threads", 0), n_docs, dims, its, len(iterations),
            objective, STOP_REASONS.index(stop_reason), a]
    _check(lib, lib.sref_report_json(*args, None, 0, C.byref(n)), "ref")
    buf = C.create_string_buffer(n.value + 1)
    _check(lib, lib.sref_report_json(*args, buf, n.value + 1, C.byref(n)), "ref")
    return buf.value.decode()


# ------------------------------------------------------------- vectorize ----
def pack_texts(texts):
    """Strings (or bytes) -> one UTF-8 byte array + int64 offsets."""
    bs = [t.encode("utf-8") if isinstance(t, str) else bytes(t) for t in texts]
    offs = np.zeros(len(bs) + 1, np.int64)
    if bs:
        offs[1:] = np.cumsum([len(b) for b in bs])
    return b"".join(bs), offs


def ref_vectorize(texts, stop_words=(), max_df=0.5):
    """The reference's vectorize_corpus (corpus.cpp:101-134) on in-memory texts.

    Returns dict(indptr, indices, values f64, kept, dropped, doc_freq, vocab,
    n_docs, dims, seconds); kept / dropped are input positions (the shim uses
    the decimal positions as doc ids)."""
    lib = _load("ref")
    text, offs = pack_texts(texts)
    stext, soffs = pack_texts(list(stop_words))
    h = _P()
    _check(lib, lib.sref_vectorize(len(texts), text, offs, len(soffs) - 1, stext, soffs, float(max_df),
                                   C.byref(h)), "ref")
    try:
        n_rows, nnz, nd = C.c_int64(), C.c_int64(), C.c_int64()
        dims, n_docs = C.c_uint32(), C.c_uint32()
        vb, secs = C.c_int64(), C.c_double()
        lib.sref_vec_sizes(h, C.byref(n_rows), C.byref(nnz), C.byref(dims), C.byref(n_docs), C.byref(nd),
                           C.byref(vb), C.byref(secs))
        ptr = np.zeros(n_rows.value + 1, np.int64)
        idx = np.zeros(max(nnz.value, 1), np.uint32)
        val = np.zeros(max(nnz.value, 1), np.float64)
        kept = np.zeros(max(n_rows.value, 1), np.int64)
        dropped = np.zeros(max(nd.value, 1), np.int64)
        dfq = np.zeros(max(dims.value, 1), np.uint32)
        vt = C.create_string_buffer(max(vb.value, 1))
        voff = np.zeros(dims.value + 1, np.int64)
        lib.sref_vec_export(h, ptr, idx, val, kept, dropped, dfq, vt, voff)
        raw = vt.raw[:vb.value]
        vocab = [raw[voff[i]:voff[i + 1]].decode("utf-8", "surrogateescape") for i in range(dims.value)]
        return {"indptr": ptr, "indices": idx[:nnz.value].astype(np.int32), "values": val[:nnz.value],
                "kept": kept[:n_rows.value], "dropped": dropped[:nd.value], "doc_freq": dfq[:dims.value],
                "vocab": vocab, "n_docs": int(n_docs.value), "dims": int(dims.value), "seconds": float(secs.value)}
    finally:
        lib.sref_vec_free(h)
