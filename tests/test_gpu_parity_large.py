"""Teacher-forced parity at BASELINE.json's full sizes (configs 1-4), against the
compiled reference (oracle/_ref) whenever it is present.

Every checked iteration feeds the GPU's state to the reference (oracle/teacher.py):
compute_centroids over ALL documents (repairs and post-repair assignments equal,
centroids within 1e-5 on a column sample), then assign on a uniform document
sample with the GPU's fp32 centroids (assignments equal except near-ties, sims
bitwise). SURVEY §8c; engine.cpp:137-195, 218-322; test_engine.cpp:54-100.
"""
import numpy as np
import pytest

import paper_2108_00895_b200 as P
from oracle import oracle as O
from oracle.teacher import TeacherForcing
from paper_2108_00895_b200 import synthetic as S

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def run_checked(cfg_name, mode, free_iters, checked_iters, n_sample, n_cols, seed=1):
    cfg = S.CONFIGS[cfg_name]
    m = S.corpus(cfg)
    k = cfg.k
    seeds = S.init_seeds(m.n_docs, k, 0)
    kind = "ref" if O.ref_available() else "port"
    docs = np.random.default_rng(seed).choice(m.n_docs, n_sample, replace=False)
    tf = TeacherForcing(m, k, mode, kind=kind, docs=docs)
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(k, mode=mode, conv_sq_dist=1e-300, max_iters=10 ** 6)
    eng.init_from_seeds(seeds)
    for _ in range(free_iters):
        eng.step()
    report = []
    for q in range(checked_iters):
        a_pre, s_pre, _ = eng.get_state()
        eng.update()
        it = eng.iteration
        cols = sorted(set(np.random.default_rng(100 + it).choice(k, n_cols, replace=False).tolist())
                      | set(eng.repaired().tolist()))
        up, (a_mid, s_mid, unch) = tf.check_update(eng, a_pre, s_pre, cols=cols)
        assert up["repaired_equal"] and up["assignments_equal"], (it, up)
        assert up["max_centroid_rel"] <= 1e-5 and up["max_centroid_abs"] <= 1e-5, (it, up)
        st = eng.assign()
        a_post, s_post, _ = eng.get_state()
        asg = tf.check_assign(eng, a_mid, s_mid, unch, it, a_post, s_post)
        assert asg["ok"], (it, asg)
        assert asg["sims_not_bitwise"] == 0, (it, asg)  # identical centroids: exact fp64 dots
        report.append((it, st.n_changed, st.n_reassigned, up["max_centroid_rel"], asg["mismatches"]))
    return report, kind


def test_c1_baseline_operating_point():
    """The bench's operating point: c1, baseline mode, iterations 6-10 (adaptive
    θ, cached own similarities for bit-identical columns)."""
    rep, kind = run_checked("c1", "baseline", free_iters=5, checked_iters=5, n_sample=3000, n_cols=200)
    assert [r[0] for r in rep] == [6, 7, 8, 9, 10]


def test_c1_ncc():
    rep, _ = run_checked("c1", "ncc", free_iters=0, checked_iters=4, n_sample=2000, n_cols=200)
    assert len(rep) == 4


def test_c2_baseline():
    """k = 10,000: five 2048-cluster tiles per document pass."""
    rep, _ = run_checked("c2", "baseline", free_iters=1, checked_iters=2, n_sample=2000, n_cols=128)
    assert len(rep) == 2


def test_c3_ncc():
    """Long documents (mean 1,500 terms)."""
    rep, _ = run_checked("c3", "ncc", free_iters=1, checked_iters=2, n_sample=1500, n_cols=128)
    assert len(rep) == 2


def test_c4_baseline():
    """N = 16e6, k = 50,000: 25 cluster tiles, 8.9e8 nonzeros, the 26 GB Cᵀ."""
    rep, _ = run_checked("c4", "baseline", free_iters=0, checked_iters=2, n_sample=1000, n_cols=64)
    assert len(rep) == 2
