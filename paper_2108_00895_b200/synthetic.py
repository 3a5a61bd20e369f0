"""BASELINE.json synthetic corpora (configs 0-4) as CorpusMatrix.

The generator itself lives in the repo-level `corpora` package (its own g++
library, shared with the reference arm of bench.py); this module only wraps its
CSR arrays in the package's CorpusMatrix.
"""
from __future__ import annotations

import corpora as _C
from corpora import CONFIGS, CorpusConfig, init_seeds  # noqa: F401

from .api import CorpusMatrix


def _wrap(c: "_C.CSR") -> CorpusMatrix:
    m = CorpusMatrix.from_csr(c.indptr, c.indices, c.values, c.dims)
    m.dropped = c.dropped
    return m


def generate(n_docs: int, dims: int, k_true: int, mean_len: float, sigma: float = 0.5,
             zipf_s: float = 1.1, seed: int = 0, threads: int = 0) -> CorpusMatrix:
    return _wrap(_C.generate(n_docs, dims, k_true, mean_len, sigma, zipf_s, seed, threads))


def corpus(cfg: "CorpusConfig | str", threads: int = 0, n_docs: int | None = None) -> CorpusMatrix:
    return _wrap(_C.corpus(cfg, threads, n_docs))
