"""BASELINE.json synthetic corpora (configs 0-4) and the seed-document init.

The generator is native (csrc/synth.cpp, pinned in its header and DESIGN.md);
this module wraps it and names the five configurations. These corpora stand in
for the paper's private datasets (BASELINE.json names no public one).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .api import CorpusMatrix


@dataclass(frozen=True)
class CorpusConfig:
    name: str
    n_docs: int
    dims: int
    k_true: int
    mean_len: float
    sigma: float
    k: int
    iterations: int
    zipf_s: float = 1.1
    seed: int = 0


# BASELINE.json "configs"
CONFIGS = {
    "c0": CorpusConfig("c0", 20_000, 16_384, 50, 60.0, 0.5, 100, 20),
    "c1": CorpusConfig("c1", 1_000_000, 262_144, 500, 100.0, 0.5, 1_000, 30),
    "c2": CorpusConfig("c2", 4_000_000, 262_144, 5_000, 100.0, 0.5, 10_000, 30),
    "c3": CorpusConfig("c3", 500_000, 131_072, 200, 1_500.0, 0.7, 2_000, 20),
    "c4": CorpusConfig("c4", 16_000_000, 131_072, 20_000, 80.0, 0.5, 50_000, 25),
}


def generate(n_docs: int, dims: int, k_true: int, mean_len: float, sigma: float = 0.5,
             zipf_s: float = 1.1, seed: int = 0, threads: int = 0) -> CorpusMatrix:
    lib = _lib.load()
    h = lib.sskm_synth_generate(int(n_docs), int(dims), int(k_true), float(mean_len), float(sigma),
                                float(zipf_s), int(seed), int(threads))
    if not h:
        raise ValueError(lib.sskm_synth_last_error().decode())
    try:
        n, nnz, d, dropped = C.c_int64(), C.c_int64(), C.c_uint32(), C.c_int64()
        lib.sskm_synth_sizes(h, C.byref(n), C.byref(nnz), C.byref(d), C.byref(dropped))
        indptr = np.zeros(n.value + 1, np.int64)
        idx = np.zeros(max(nnz.value, 1), np.int32)
        val = np.zeros(max(nnz.value, 1), np.float32)
        lib.sskm_synth_export(h, indptr, idx, val)
    finally:
        lib.sskm_synth_free(h)
    m = CorpusMatrix.from_csr(indptr, idx[: nnz.value], val[: nnz.value], d.value)
    m.dropped = int(dropped.value)
    return m


def corpus(cfg: "CorpusConfig | str", threads: int = 0, n_docs: int | None = None) -> CorpusMatrix:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return generate(n_docs or cfg.n_docs, cfg.dims, cfg.k_true, cfg.mean_len, cfg.sigma, cfg.zipf_s,
                    cfg.seed, threads)


def init_seeds(n_docs: int, k: int, seed: int = 0) -> np.ndarray:
    """k distinct documents from seed 0, order = cluster ids:
    numpy.random.default_rng(seed).choice(n_docs, k, replace=False)."""
    return np.random.default_rng(seed).choice(n_docs, k, replace=False).astype(np.uint32)
