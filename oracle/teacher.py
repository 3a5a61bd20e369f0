"""TEST INFRASTRUCTURE ONLY — teacher-forced parity of the GPU engine against the oracle.

SURVEY §8c protocol, one Lloyd iteration at a time (the Stepper of the reference tests,
proj/tests/test_engine.cpp:54-100):

* update: the oracle's ``compute_centroids`` (engine.cpp:137-195) runs over ALL documents on the
  GPU's pre-update state; the repaired list and post-repair assignments must be equal and the GPU's
  centroids within 1e-5 (relative per column and absolute per entry), checked on a column sample at
  large k;
* assign: given the GPU's fp32 centroids and its pre-assign state, the oracle's ``assign``
  (engine.cpp:218-322) must reproduce the GPU's assignments and sims on a document sample. The
  centroids handed to the oracle are restricted to the terms the sample uses: ``dot`` visits only
  shared dims, in ascending order, with either strategy (sparse_vector.cpp:72-108), so dropping terms
  no sampled document has — and renumbering the kept ones monotonically — changes no bit of any dot.
  That keeps config 4 (Cᵀ is 26 GB dense) checkable.

Used by tests/ and by bench.py's cpu_baseline leg (its ``parity`` block). Never by the product.
"""
from __future__ import annotations

import numpy as np

from . import oracle as O

REL_TOL = 1e-5     # north_star: centroids within 1e-5 relative
NEAR_TIE = 1e-5    # north_star: assignments equal except at near-ties |Δcos| ≤ 1e-5


def gather_rows(m, docs):
    """CSR of the documents `docs` (sorted) of a CorpusMatrix-like m."""
    docs = np.asarray(docs, np.int64)
    lens = (m.indptr[docs + 1] - m.indptr[docs]).astype(np.int64)
    ptr = np.zeros(len(docs) + 1, np.int64)
    ptr[1:] = np.cumsum(lens)
    pos = np.repeat(m.indptr[docs] - ptr[:-1], lens) + np.arange(int(ptr[-1]), dtype=np.int64)
    return ptr, m.indices[pos], m.values[pos]


def columns_csr(rows_block: np.ndarray, chunk: int = 4096):
    """Column-wise CSR (ptr, idx, val) of a dense |T| × k block; idx are row numbers."""
    nrows, k = rows_block.shape
    ptr = np.zeros(k + 1, np.int64)
    idx_parts, val_parts = [], []
    for j0 in range(0, k, chunk):
        b = np.ascontiguousarray(rows_block[:, j0:j0 + chunk].T)  # columns as rows, terms ascending
        c, r = np.nonzero(b)
        ptr[j0 + 1:j0 + b.shape[0] + 1] = np.bincount(c, minlength=b.shape[0])
        idx_parts.append(r.astype(np.uint32))
        val_parts.append(b[c, r].astype(np.float64))
    ptr = np.cumsum(ptr)
    return ptr, np.concatenate(idx_parts), np.concatenate(val_parts)


class TeacherForcing:
    """Oracle side of a teacher-forced run: ``check_update`` after ``eng.update()``,
    ``check_assign`` after ``eng.assign()``."""

    def __init__(self, m, k, mode="baseline", kind="ref", docs=None, ncc_epsilon=0.0, threads=0,
                 full_update=True):
        self.m, self.k, self.mode, self.kind = m, int(k), mode, kind
        self.full_update = full_update
        if full_update:
            c_full = O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), m.dims)
            self.c_full = c_full
            self.upd = O.Stepper(c_full, k, mode, kind=kind, ncc_epsilon=ncc_epsilon, threads=threads)
        self.docs = None if docs is None else np.sort(np.asarray(docs, np.int64))
        if self.docs is None:
            if not full_update:
                raise ValueError("a full-corpus assign check needs the full-corpus stepper")
            self.terms = None
            self.asg = self.upd
        else:
            ptr, idx, val = gather_rows(m, self.docs)
            self.terms = np.unique(idx).astype(np.uint32)
            ridx = np.searchsorted(self.terms, idx).astype(np.int32)
            self.c_samp = O.Corpus(ptr, ridx, val.astype(np.float64), max(1, len(self.terms)))
            sample = kind == "ref"
            if not sample and k > len(self.docs):
                raise ValueError("the C port needs k <= sample size")
            self.asg = O.Stepper(self.c_samp, k, mode, kind=kind, ncc_epsilon=ncc_epsilon, threads=threads,
                                 sample=sample)

    # ------------------------------------------------------------------ update --
    def check_update(self, eng, a_pre, s_pre, cols=None):
        """Reference compute_centroids on the GPU's pre-update state (all documents)."""
        a_rep, rep = self.upd.compute_centroids(a_pre, s_pre)
        a_mid, s_mid, unch = eng.get_state()
        out = {"repaired_equal": bool(np.array_equal(rep, eng.repaired())),
               "assignments_equal": bool(np.array_equal(a_rep, a_mid)),
               "n_repaired": int(len(rep))}
        cols = np.arange(self.k, dtype=np.uint32) if cols is None else np.asarray(sorted(set(cols)), np.uint32)
        gpu = eng.get_centroid_cols(cols)
        ptr, idx, val = self.upd.get_cols_csr(cols)
        worst_rel, worst_abs = 0.0, 0.0
        for q in range(len(cols)):
            ref = np.zeros(gpu.shape[0])
            ref[idx[ptr[q]:ptr[q + 1]]] = val[ptr[q]:ptr[q + 1]]
            d = gpu[:, q].astype(np.float64) - ref
            nr = np.linalg.norm(ref)
            worst_rel = max(worst_rel, float(np.linalg.norm(d) / nr) if nr > 0 else float(np.linalg.norm(d)))
            worst_abs = max(worst_abs, float(np.max(np.abs(d))) if len(d) else 0.0)
        out.update(cols=int(len(cols)), max_centroid_rel=worst_rel, max_centroid_abs=worst_abs,
                   ok=out["repaired_equal"] and out["assignments_equal"] and worst_rel <= REL_TOL
                   and worst_abs <= REL_TOL)
        return out, (a_mid, s_mid, unch)

    # ------------------------------------------------------------------ assign --
    def check_assign(self, eng, a_mid, s_mid, unch, iteration, a_post, s_post):
        """Reference assign with the GPU's fp32 centroids on the (sampled) documents."""
        if self.terms is None:
            self.asg.set_centroids_dense(eng.get_centroids().astype(np.float64))
            docs = np.arange(self.m.n_docs)
        else:
            rows = eng.get_centroid_rows(self.terms)
            self.asg.set_centroids_csr(*columns_csr(rows))
            docs = self.docs
        self.asg.set_state(a_mid[docs], s_mid[docs], unch, iteration)
        r = self.asg.assign()
        ra, rs, _ = self.asg.get_state()
        ga, gs = a_post[docs], s_post[docs]
        diff = np.nonzero(ra != ga)[0]
        near = int(np.sum(np.abs(rs[diff] - gs[diff]) <= NEAR_TIE))
        sims_diff = int(np.sum((rs != gs) & (ra == ga)))  # same argmax: the sims must be bitwise equal
        return {"docs": int(len(docs)), "mismatches": int(len(diff)), "near_ties": near,
                "sims_not_bitwise": sims_diff, "max_sim_abs_diff": float(np.max(np.abs(rs - gs))) if len(docs) else 0.0,
                "dot_products": int(r["dot_products"]), "n_reassigned": int(r["n_reassigned"]),
                "objective": float(r["objective"]), "ok": len(diff) == near and sims_diff == 0}
