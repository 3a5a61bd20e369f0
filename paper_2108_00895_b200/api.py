"""Python API mirroring the reference's `sskm` module (proj/src/bindings.cpp:23-136,
proj/python/sskm/__init__.py) on top of the C-ABI.

Same names, argument meaning and error behaviour as the reference: invalid
configs raise ValueError (std::invalid_argument, test_smoke.py:104-111), the
result exposes assignments / sims / iterations / objective / stop_reason /
n_clusters / total_dot_products(). Additions: CorpusMatrix.from_csr,
cluster(..., init_seeds=, device=), ClusteringResult.centroids, and the
per-phase Engine used by the parity tests and the multi-GPU driver.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import MODES, STOP_REASONS, check, sskm_iteration_stats, sskm_run_config


class SparseVector:
    """Read-only (dim, weight) view of a corpus row (sparse_vector.hpp:22-53)."""

    def __init__(self, dims_: np.ndarray, weights: np.ndarray, dims: int = 0):
        self._d = np.asarray(dims_, np.uint32)
        self._w = np.asarray(weights, np.float64)
        self.dims = int(dims)

    @property
    def nnz(self) -> int:
        return len(self._d)

    def entries(self):
        return [(int(d), float(w)) for d, w in zip(self._d, self._w)]

    def norm(self) -> float:
        return float(np.sqrt(np.sum(self._w * self._w)))

    def __eq__(self, other) -> bool:
        return isinstance(other, SparseVector) and np.array_equal(self._d, other._d) and np.array_equal(
            self._w, other._w)


class CorpusMatrix:
    """Unit-length document rows in CSR form (corpus.hpp:26-32).

    Values are fp32 (the device storage type); indices int32 sorted strictly
    ascending within each row; |x| <= 1.
    """

    def __init__(self):
        self.indptr = np.zeros(1, np.int64)
        self.indices = np.zeros(0, np.int32)
        self.values = np.zeros(0, np.float32)
        self.dims = 0
        self.doc_ids: list = []
        self.values64 = None  # exact fp64 weights when known (vectorize_corpus)

    @classmethod
    def from_csr(cls, indptr, indices, values, dims: int, doc_ids: Optional[Sequence[str]] = None):
        m = cls()
        m.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        m.indices = np.ascontiguousarray(indices, dtype=np.int32)
        m.values = np.ascontiguousarray(values, dtype=np.float32)
        m.dims = int(dims)
        if len(m.indptr) < 1 or m.indptr[0] != 0 or m.indptr[-1] != len(m.indices) or len(m.indices) != len(
                m.values):
            raise ValueError("malformed CSR arrays")
        n = len(m.indptr) - 1
        m.doc_ids = list(doc_ids) if doc_ids is not None else None
        if m.doc_ids is not None and len(m.doc_ids) != n:
            raise ValueError("doc_ids length mismatch")
        return m

    @property
    def n_docs(self) -> int:
        return len(self.indptr) - 1

    def size(self) -> int:
        return self.n_docs

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def row(self, i: int) -> SparseVector:
        if not 0 <= i < self.n_docs:
            raise IndexError(i)
        b, e = self.indptr[i], self.indptr[i + 1]
        vals = self.values64[b:e] if self.values64 is not None else self.values[b:e].astype(np.float64)
        return SparseVector(self.indices[b:e], vals, self.dims)


@dataclass
class IterationStats:
    """engine.hpp:43-57 plus the GPU extras of sskm_iteration_stats."""
    iteration: int = 0
    n_reassigned: int = 0
    n_unchanged_centroids: int = 0
    dot_products: int = 0
    index_queries: int = 0
    candidates_total: int = 0
    wall_seconds: float = 0.0
    index_build_seconds: float = 0.0
    index_active: bool = False
    max_sq_drift: float = 0.0
    objective: float = 0.0
    n_repaired: int = 0
    gpu_dot_products: int = 0
    n_moved: int = 0
    n_changed: int = 0
    n_recomputed: int = 0
    n_rescan: int = 0
    n_exact: int = 0
    update_ms: float = 0.0
    assign_ms: float = 0.0
    assign_kernel_ms: float = 0.0
    screen_ms: float = 0.0
    screen_launches: int = 0
    second_pass_docs: int = 0
    centroid_density: float = 0.0
    bound_docs: int = 0
    bound_pairs: int = 0
    bound_candidates: int = 0
    bound_doc_nnz: int = 0
    bound_cand_nnz: int = 0
    bound_theta: float = 0.0
    bound_visits: int = 0
    bound_own_dots: int = 0
    skip_docs: int = 0
    bound_own_nnz: int = 0
    reserved2: int = 0
    skip_ms: float = 0.0

    @classmethod
    def from_c(cls, s: sskm_iteration_stats) -> "IterationStats":
        d = {f: getattr(s, f) for f, _ in s._fields_}
        d["index_active"] = bool(d["index_active"])
        return cls(**d)


@dataclass
class ClusteringResult:
    """engine.hpp:132-142 (+ centroids exposed as Cᵀ, d × k fp32)."""
    assignments: np.ndarray
    sims: np.ndarray
    iterations: list
    objective: float
    stop_reason: str
    centroids: Optional[np.ndarray] = None
    seeds: Optional[np.ndarray] = None
    extra: dict = field(default_factory=dict)

    @property
    def n_clusters(self) -> int:
        return int(self.extra.get("k", 0))

    def total_dot_products(self) -> int:
        return int(sum(it.dot_products for it in self.iterations))

    def total_index_build_seconds(self) -> float:
        return float(sum(it.index_build_seconds for it in self.iterations))


def parse_mode(name: str) -> int:
    """engine.cpp:21-27."""
    if name not in MODES:
        raise ValueError(f"unknown mode '{name}' (expected baseline, ncc, or ncc+index)")
    return MODES[name]


def make_config(k, mode="baseline", seed=0, lambdas=(0.1, 0.25, 0.4, 0.6), conv_sq_dist=0.0001,
                ncc_epsilon=0.0, index_activation_threshold=100, max_iters=100, threads=0, device=0):
    cfg = sskm_run_config()
    if k < 0 or k >= 2 ** 32:
        raise ValueError("k must be at least 2")
    cfg.k = int(k)
    cfg.mode = parse_mode(mode)
    lam = np.ascontiguousarray(lambdas, dtype=np.float64)
    cfg._lam = lam  # keep alive
    cfg.lambdas = lam.ctypes.data_as(C.POINTER(C.c_double)) if len(lam) else None
    cfg.n_lambdas = len(lam)
    cfg.conv_sq_dist = float(conv_sq_dist)
    cfg.ncc_epsilon = float(ncc_epsilon)
    cfg.index_activation_threshold = int(index_activation_threshold)
    cfg.max_iters = int(max_iters)
    cfg.seed = int(seed)
    cfg.threads = int(threads)
    cfg.device = int(device)
    return cfg


class Engine:
    """Per-phase handle over one GPU (sskm_ctx). Device-resident corpus (shard),
    Cᵀ, fixed-point sums and state; calls map 1:1 onto the C-ABI."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        self.h = C.c_void_p()
        check(self.lib.sskm_open(int(device), C.byref(self.h)))
        self.n = 0
        self.k = 0
        self.dims = 0

    def close(self):
        if self.h:
            check(self.lib.sskm_close(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def upload(self, data: CorpusMatrix, doc_offset: int = 0, n_docs_total: int = 0):
        check(self.lib.sskm_upload_csr(self.h, data.n_docs, data.dims, data.indptr, data.indices, data.values,
                                       int(doc_offset), int(n_docs_total or data.n_docs)))
        self.n = data.n_docs
        self.dims = data.dims

    def configure(self, k, **kw):
        self.cfg = make_config(k, **kw)
        check(self.lib.sskm_configure(self.h, C.byref(self.cfg)))
        self.k = int(k)

    def init_from_seeds(self, seeds):
        s = np.ascontiguousarray(seeds, dtype=np.uint32)
        if len(s) != self.k:
            raise ValueError("need exactly k seeds")
        check(self.lib.sskm_init_from_seeds(self.h, s))

    def init_kmeanspp(self, seed: int) -> np.ndarray:
        out = np.zeros(self.k, np.uint32)
        check(self.lib.sskm_init_kmeanspp(self.h, int(seed), out))
        return out

    def _stats_call(self, fn) -> IterationStats:
        st = sskm_iteration_stats()
        check(fn(self.h, C.byref(st)))
        return IterationStats.from_c(st)

    def update(self) -> IterationStats:
        return self._stats_call(self.lib.sskm_update)

    def assign(self) -> IterationStats:
        return self._stats_call(self.lib.sskm_assign)

    def step(self) -> IterationStats:
        return self._stats_call(self.lib.sskm_step)

    def step_n(self, n: int):
        """n Lloyd iterations in one native call (no stop rules): [IterationStats]."""
        arr = (sskm_iteration_stats * max(int(n), 1))()
        check(self.lib.sskm_step_n(self.h, int(n), arr))
        return [IterationStats.from_c(arr[i]) for i in range(int(n))]

    def run(self, cap: Optional[int] = None):
        cap = cap or self.cfg.max_iters
        arr = (sskm_iteration_stats * cap)()
        n_it = C.c_uint32()
        stop = C.c_int32()
        check(self.lib.sskm_run(self.h, arr, cap, C.byref(n_it), C.byref(stop)))
        return [IterationStats.from_c(arr[i]) for i in range(min(n_it.value, cap))], STOP_REASONS[stop.value]

    def get_state(self):
        a = np.zeros(self.n, np.uint32)
        s = np.zeros(self.n, np.float64)
        u = np.zeros(self.k, np.uint8)
        check(self.lib.sskm_get_state(self.h, a, s, u))
        return a, s, u

    def set_state(self, assignments, sims, iteration: int):
        a = np.ascontiguousarray(assignments, np.uint32)
        s = np.ascontiguousarray(sims, np.float64)
        check(self.lib.sskm_set_state(self.h, a, s, int(iteration)))

    def set_unchanged(self, flags):
        check(self.lib.sskm_set_unchanged(self.h, np.ascontiguousarray(flags, np.uint8)))

    def get_centroids(self) -> np.ndarray:
        out = np.zeros((self.dims, self.k), np.float32)
        check(self.lib.sskm_get_centroids(self.h, out))
        return out

    def get_centroid_rows(self, rows) -> np.ndarray:
        """Rows of Cᵀ (terms) as a len(rows) × k array."""
        rows = np.ascontiguousarray(rows, np.uint32)
        out = np.zeros((len(rows), self.k), np.float32)
        if len(rows):
            check(self.lib.sskm_get_centroid_rows(self.h, len(rows), rows, out))
        return out

    def get_centroid_cols(self, cols) -> np.ndarray:
        """Columns of Cᵀ (clusters) as a d × len(cols) array."""
        cols = np.ascontiguousarray(cols, np.uint32)
        out = np.zeros((self.dims, len(cols)), np.float32)
        if len(cols):
            check(self.lib.sskm_get_centroid_cols(self.h, len(cols), cols, out))
        return out

    def debug_check_postings(self) -> int:
        """Rows where the kept high postings differ from a fresh build (-1: none kept)."""
        n = C.c_int64()
        check(self.lib.sskm_debug_check_postings(self.h, C.byref(n)))
        return int(n.value)

    def set_centroids(self, ct: np.ndarray):
        ct = np.ascontiguousarray(ct, np.float32)
        if ct.shape != (self.dims, self.k):
            raise ValueError(f"centroids must be d × k = {(self.dims, self.k)}")
        check(self.lib.sskm_set_centroids(self.h, ct))

    def repaired(self) -> np.ndarray:
        out = np.zeros(self.k, np.uint32)
        n = C.c_uint32()
        check(self.lib.sskm_get_repaired(self.h, out, C.byref(n)))
        return out[: n.value]

    def timer_record(self, slot: int):
        check(self.lib.sskm_timer_record(self.h, int(slot)))

    def timer_elapsed(self, a: int, b: int) -> float:
        ms = C.c_double()
        check(self.lib.sskm_timer_elapsed(self.h, int(a), int(b), C.byref(ms)))
        return ms.value

    def launch_count(self) -> int:
        n = C.c_uint64()
        check(self.lib.sskm_launch_count(self.h, C.byref(n)))
        return int(n.value)

    def postings_work(self) -> int:
        n = C.c_uint64()
        check(self.lib.sskm_postings_work(self.h, C.byref(n)))
        return int(n.value)

    def synchronize(self):
        check(self.lib.sskm_synchronize(self.h))

    @property
    def iteration(self) -> int:
        it = C.c_uint32()
        check(self.lib.sskm_get_iteration(self.h, C.byref(it)))
        return int(it.value)


class MultiEngine:
    """Several GPUs of one node driven from this thread (sskm_multi_*): the
    corpus is sharded over `devices` in contiguous equal ranges; every device
    applies every shard's moved rows to its own exact sums through peer memory,
    so assignments, sims and centroids equal a single-GPU run bit for bit."""

    def __init__(self, devices: Sequence[int]):
        self.lib = _lib.load()
        self.devices = [int(d) for d in devices]
        self.h = C.c_void_p()
        check(self.lib.sskm_multi_open(len(self.devices), np.asarray(self.devices, np.int32), C.byref(self.h)))
        self.n = self.k = self.dims = 0

    def close(self):
        if self.h:
            check(self.lib.sskm_multi_close(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, data: CorpusMatrix):
        check(self.lib.sskm_multi_upload_csr(self.h, data.n_docs, data.dims, data.indptr, data.indices, data.values))
        self.n, self.dims = data.n_docs, data.dims

    def configure(self, k, **kw):
        self.cfg = make_config(k, **kw)
        check(self.lib.sskm_multi_configure(self.h, C.byref(self.cfg)))
        self.k = int(k)

    def init_from_seeds(self, seeds):
        s = np.ascontiguousarray(seeds, dtype=np.uint32)
        if len(s) != self.k:
            raise ValueError("need exactly k seeds")
        check(self.lib.sskm_multi_init_from_seeds(self.h, s))

    def step(self) -> IterationStats:
        st = sskm_iteration_stats()
        check(self.lib.sskm_multi_step(self.h, C.byref(st)))
        return IterationStats.from_c(st)

    def run(self):
        cap = int(self.cfg.max_iters)
        stats = (sskm_iteration_stats * cap)()
        n_it, stop = C.c_uint32(), C.c_int32()
        check(self.lib.sskm_multi_run(self.h, stats, cap, C.byref(n_it), C.byref(stop)))
        return [IterationStats.from_c(stats[i]) for i in range(n_it.value)], STOP_REASONS[stop.value]

    def get_state(self):
        a = np.zeros(self.n, np.uint32)
        s = np.zeros(self.n, np.float64)
        check(self.lib.sskm_multi_get_state(self.h, a.ctypes.data, s.ctypes.data))
        return a, s

    def get_centroids(self) -> np.ndarray:
        out = np.zeros((self.dims, self.k), np.float32)
        check(self.lib.sskm_multi_get_centroids(self.h, out))
        return out

    def launch_count(self) -> int:
        n = C.c_uint64()
        check(self.lib.sskm_multi_launch_count(self.h, C.byref(n)))
        return int(n.value)


def validate(n_docs: int, k: int, **kw) -> None:
    """RunConfig::validate (engine.cpp:47-64)."""
    cfg = make_config(k, **{x: y for x, y in kw.items() if x != "threads"})
    check(_lib.load().sskm_validate(C.byref(cfg), int(n_docs)))


def cluster(data: CorpusMatrix, k: int, mode: str = "baseline", seed: int = 0,
            lambdas: Sequence[float] = (0.1, 0.25, 0.4, 0.6), conv_sq_dist: float = 0.0001,
            ncc_epsilon: float = 0.0, index_activation_threshold: int = 100, max_iters: int = 100,
            threads: int = 0, init_seeds=None, device: int = 0, devices: Optional[Sequence[int]] = None,
            return_centroids: bool = False) -> ClusteringResult:
    """sskm.cluster (bindings.cpp:113-135) on the GPU: the one-shot C-ABI entry
    sskm_cluster_csr = sskm::run (engine.hpp:148). With init_seeds=None the seeds
    come from k-means++ (engine.cpp:66-130) exactly like the reference.
    devices=[...] shards the documents over several GPUs of this node
    (sskm_cluster_csr_multi; needs init_seeds); the result is bitwise the
    single-GPU one."""
    if not isinstance(data, CorpusMatrix):
        raise TypeError("data must be a CorpusMatrix")
    lib = _lib.load()
    if not isinstance(k, (int, np.integer)) or k < 0:
        raise ValueError("k must be at least 2")
    cfg = make_config(k, mode=mode, seed=seed, lambdas=lambdas, conv_sq_dist=conv_sq_dist,
                      ncc_epsilon=ncc_epsilon, index_activation_threshold=index_activation_threshold,
                      max_iters=max_iters, threads=threads, device=device)
    check(lib.sskm_validate(C.byref(cfg), data.n_docs))
    n = data.n_docs
    a = np.zeros(n, np.uint32)
    s = np.zeros(n, np.float64)
    ct = np.zeros((data.dims, k), np.float32) if return_centroids else None
    stats = (sskm_iteration_stats * max_iters)()
    n_it = C.c_uint32()
    stop = C.c_int32()
    obj = C.c_double()
    seeds = None
    if init_seeds is not None:
        seeds = np.ascontiguousarray(init_seeds, np.uint32)
        if len(seeds) != k:
            raise ValueError("init_seeds must hold exactly k document ids")
    if devices is not None:
        devs = np.ascontiguousarray([int(x) for x in devices], np.int32)
        if seeds is None:
            raise ValueError("a multi-device run needs init_seeds (k-means++ runs on one device)")
        check(lib.sskm_cluster_csr_multi(C.byref(cfg), len(devs), devs, n, data.dims, data.indptr, data.indices,
                                         data.values, seeds.ctypes.data, a.ctypes.data, s.ctypes.data,
                                         ct.ctypes.data if ct is not None else None, stats, max_iters,
                                         C.byref(n_it), C.byref(stop), C.byref(obj)))
    else:
        check(lib.sskm_cluster_csr(C.byref(cfg), n, data.dims, data.indptr, data.indices, data.values,
                                   seeds.ctypes.data if seeds is not None else None, a.ctypes.data,
                                   s.ctypes.data, ct.ctypes.data if ct is not None else None, stats, max_iters,
                                   C.byref(n_it), C.byref(stop), C.byref(obj)))
    its = [IterationStats.from_c(stats[i]) for i in range(n_it.value)]
    return ClusteringResult(assignments=a, sims=s, iterations=its, objective=obj.value,
                            stop_reason=STOP_REASONS[stop.value], centroids=ct, seeds=seeds,
                            extra={"k": int(k)})
