"""Shared helpers for the tests (test-only; may use the oracle)."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def csr_from_rows(rows, dims=None, dtype=np.float64):
    """rows: list of list[(dim, weight)] (sorted, as SparseVector) -> CSR."""
    ptr = np.zeros(len(rows) + 1, np.int64)
    idx, val = [], []
    for i, r in enumerate(rows):
        r = sorted(r)
        ptr[i + 1] = ptr[i] + len(r)
        idx += [d for d, _ in r]
        val += [w for _, w in r]
    if dims is None:
        dims = max([d for r in rows for d, _ in r] + [-1]) + 1
    return ptr, np.array(idx, np.int32), np.array(val, dtype), int(dims)


def unit(pairs):
    """normalize(SparseVector(pairs)) with the reference's own normalize."""
    idx, val = O.normalize([d for d, _ in pairs], [w for _, w in pairs], kind="port")
    return list(zip(idx.tolist(), val.tolist()))


def e(dim):
    return [(dim, 1.0)]


def random_unit_rows(rng: np.random.Generator, n, dims, max_nnz, allow_negative=False):
    """Like oracle.hpp:59-71 random_unit (our own RNG), normalized by the reference's normalize."""
    rows = []
    for _ in range(n):
        nnz = 1 + int(rng.integers(0, max_nnz))
        d = np.sort(rng.choice(dims, nnz, replace=False))
        w = 1.0 - rng.random(nnz)
        if allow_negative:
            w = np.where(rng.random(nnz) < 0.5, -w, w)
        rows.append(unit(list(zip(d.tolist(), w.tolist()))))
    return rows


def f32_rows(rows):
    """Round weights to fp32 (the GPU storage type) and back to float."""
    return [[(d, float(np.float32(w))) for d, w in r] for r in rows]


def oracle_corpus(ptr, idx, val, dims):
    return O.Corpus(ptr, idx, np.asarray(val, np.float64), dims)
