"""B200-native data-parallel core of sparse spherical k-means (arXiv 2108.00895).

Drop-in for the reference `sskm` hot path (proj/python/sskm/__init__.py):
`cluster`, `CorpusMatrix`, `ClusteringResult`, `IterationStats`, backed by the
sm_100a kernels in csrc/ behind the C-ABI in include/sskm_b200.h.
"""
from ._lib import load as _load_native
from .io import load_csr, load_matrix, make_report, save_csr, to_json, write_matrix, write_report
from .api import (
    ClusteringResult,
    CorpusMatrix,
    Engine,
    IterationStats,
    MultiEngine,
    SparseVector,
    cluster,
    parse_mode,
    validate,
)

from .vectorize import VectorizeResult, vectorize_corpus, vectorize_texts

_load_native()  # fail loudly at import if the native library is unusable

__all__ = [
    "load_csr",
    "load_matrix",
    "make_report",
    "save_csr",
    "to_json",
    "write_matrix",
    "write_report",
    "ClusteringResult",
    "CorpusMatrix",
    "Engine",
    "IterationStats",
    "MultiEngine",
    "SparseVector",
    "cluster",
    "parse_mode",
    "validate",
    "VectorizeResult",
    "vectorize_corpus",
    "vectorize_texts",
]
