"""GPU TF-IDF ingestion: the reference's `vectorize_corpus` (corpus.cpp:101-134,
Python binding bindings.cpp:53-63) on the device through the C-ABI
(`sskm_vectorize`, csrc/vectorize.cu). Bit-identical to the reference:
same dims (first-occurrence order), doc frequencies, fp64 weights after the
reference's iterated normalize, dropped ids in the reference's order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from . import _lib
from .api import CorpusMatrix


def _pack(texts) -> Tuple[bytes, np.ndarray]:
    bs = [t.encode("utf-8") if isinstance(t, str) else bytes(t) for t in texts]
    offs = np.zeros(len(bs) + 1, np.int64)
    if bs:
        offs[1:] = np.cumsum([len(b) for b in bs])
    return b"".join(bs), offs


@dataclass
class VectorizeResult:
    """corpus.hpp:74-78: matrix + vocabulary + dropped ids (plus GPU stats)."""
    matrix: CorpusMatrix
    vocab: List[str]                 # terms by dim
    doc_freq: np.ndarray             # uint32 by dim
    n_docs: int                      # Vocabulary::n_docs (documents after the stop-word pre-pass)
    dropped_doc_ids: list
    kept_positions: np.ndarray       # input position of each matrix row
    dropped_positions: np.ndarray
    stats: dict = field(default_factory=dict)

    @property
    def term_to_dim(self) -> dict:
        return {t: i for i, t in enumerate(self.vocab)}


def vectorize_texts(texts: Sequence, ids: Sequence | None = None, stop_words: Sequence[str] = (),
                    max_df: float = 0.5, device: int = 0) -> VectorizeResult:
    """vectorize_corpus over `texts` (ids default to the positions as strings)."""
    lib = _lib.load()
    text, offs = _pack(texts)
    stext, soffs = _pack(list(stop_words))
    h = C.c_void_p()
    _lib.check(lib.sskm_vectorize(int(device), len(texts), text, offs, len(soffs) - 1, stext, soffs, float(max_df),
                                  C.byref(h)))
    try:
        n_rows, nnz, nd, vb = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        dims, n_docs = C.c_uint32(), C.c_uint32()
        _lib.check(lib.sskm_vec_sizes(h, C.byref(n_rows), C.byref(nnz), C.byref(dims), C.byref(n_docs), C.byref(nd),
                                      C.byref(vb)))
        ptr = np.zeros(n_rows.value + 1, np.int64)
        idx = np.zeros(max(nnz.value, 1), np.int32)
        val = np.zeros(max(nnz.value, 1), np.float64)
        kept = np.zeros(max(n_rows.value, 1), np.int64)
        dropped = np.zeros(max(nd.value, 1), np.int64)
        dfq = np.zeros(max(dims.value, 1), np.uint32)
        vt = C.create_string_buffer(max(vb.value, 1))
        voff = np.zeros(dims.value + 1, np.int64)
        _lib.check(lib.sskm_vec_export(h, ptr, idx, val, kept, dropped, dfq, vt, voff))
        ms, launches, ntok, nbrent = C.c_double(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _lib.check(lib.sskm_vec_stats(h, C.byref(ms), C.byref(launches), C.byref(ntok), C.byref(nbrent)))
    finally:
        lib.sskm_vec_free(h)
    raw = vt.raw[:vb.value]
    vocab = [raw[voff[i]:voff[i + 1]].decode("utf-8", "surrogateescape") for i in range(dims.value)]
    ids = [str(i) for i in range(len(texts))] if ids is None else list(ids)
    kept = kept[:n_rows.value]
    dropped = dropped[:nd.value]
    m = CorpusMatrix.from_csr(ptr, idx[:nnz.value], val[:nnz.value].astype(np.float32), dims.value,
                              doc_ids=[ids[i] for i in kept])
    m.values64 = val[:nnz.value]
    return VectorizeResult(matrix=m, vocab=vocab, doc_freq=dfq[:dims.value], n_docs=int(n_docs.value),
                           dropped_doc_ids=[ids[i] for i in dropped], kept_positions=kept,
                           dropped_positions=dropped,
                           stats={"gpu_ms": ms.value, "launches": launches.value, "tokens": ntok.value,
                                  "brent_rows": nbrent.value, "text_bytes": len(text)})


def vectorize_corpus(docs: Sequence[Tuple[str, str]], stop_words: Sequence[str] = (), max_df: float = 0.5,
                     device: int = 0):
    """sskm.vectorize_corpus (bindings.cpp:53-63): docs = [(id, text)] ->
    (CorpusMatrix, vocabulary size, dropped doc ids)."""
    docs = list(docs)
    r = vectorize_texts([t for _, t in docs], ids=[i for i, _ in docs], stop_words=stop_words, max_df=max_df,
                        device=device)
    return r.matrix, len(r.vocab), r.dropped_doc_ids
