"""ncc+index on the GPU against the compiled reference, teacher-forced per
iteration (SURVEY §8c protocol): the reference's MultiIndex is built from the
GPU's centroids and queried from the GPU's pre-assign state; assignments, sims
and the index counters (index_active, index_queries, candidates_total,
dot_products — engine.cpp:277-298, 384-386) must be equal."""
import numpy as np
import pytest

import paper_2108_00895_b200 as P
from oracle import oracle as O
from paper_2108_00895_b200 import synthetic as S
from tests._util import csr_from_rows, random_unit_rows

pytestmark = pytest.mark.gpu

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="compiled reference (oracle/_ref) not built")


def index_teacher_check(m, k, seeds, iters, threshold, ncc_epsilon=0.0):
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(k, mode="ncc+index", conv_sq_dist=1e-300, ncc_epsilon=ncc_epsilon,
                  index_activation_threshold=threshold)
    eng.init_from_seeds(seeds)
    c = O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), m.dims)
    ref = O.Stepper(c, k, "ncc+index", ncc_epsilon=ncc_epsilon, conv_sq_dist=1e-300,
                    index_activation_threshold=threshold, kind="ref")
    active = 0
    for it in range(1, iters + 1):
        eng.update()
        a_mid, s_mid, unch = eng.get_state()
        ct = eng.get_centroids()
        st = eng.assign()
        a, s, _ = eng.get_state()
        ref.set_centroids_dense(ct)
        ref.set_state(a_mid, s_mid, unch, it)
        r = ref.assign(n_unchanged=int(np.count_nonzero(unch)) if it > 1 else 0)
        ra, rs, _ = ref.get_state()
        assert np.array_equal(ra, a) and np.array_equal(rs, s), it
        assert bool(r["index_active"]) == bool(st.index_active), it
        assert r["index_queries"] == st.index_queries, (it, r["index_queries"], st.index_queries)
        assert r["candidates_total"] == st.candidates_total, (it, r["candidates_total"], st.candidates_total)
        assert r["dot_products"] == st.dot_products, (it, r["dot_products"], st.dot_products)
        active += int(st.index_active)
        if st.n_reassigned == 0:
            break
    return active


@needs_ref
def test_index_counters_nonnegative_corpus():
    m = S.generate(3000, 2000, 12, 40.0, seed=21)
    seeds = np.random.default_rng(0).choice(m.n_docs, 40, replace=False)
    assert index_teacher_check(m, 40, seeds, 10, threshold=3) >= 2


@needs_ref
def test_index_counters_rescan_list_path():
    # ncc_epsilon > 0 takes the changed-list pass A + rescan list (no full-scan shortcut)
    m = S.generate(2500, 1500, 10, 30.0, seed=5)
    seeds = np.random.default_rng(1).choice(m.n_docs, 32, replace=False)
    assert index_teacher_check(m, 32, seeds, 8, threshold=2, ncc_epsilon=1e-12) >= 1


@needs_ref
def test_index_counters_signed_corpus():
    rows = random_unit_rows(np.random.default_rng(8), 1500, 400, 20, allow_negative=True)
    rows = [[(d, float(np.float32(w))) for d, w in r] for r in rows]
    m = P.CorpusMatrix.from_csr(*csr_from_rows(rows, dims=400, dtype=np.float32))
    seeds = np.random.default_rng(2).choice(m.n_docs, 24, replace=False)
    index_teacher_check(m, 24, seeds, 6, threshold=1)


@needs_ref
def test_index_counters_two_cluster_tiles():
    # k > 1024: the query runs over two cluster tiles
    m = S.generate(6000, 3000, 40, 25.0, seed=13)
    seeds = np.random.default_rng(3).choice(m.n_docs, 1100, replace=False)
    assert index_teacher_check(m, 1100, seeds, 4, threshold=10) >= 1


def test_index_inactive_below_threshold():
    m = S.generate(1500, 800, 6, 20.0, seed=2)
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(16, mode="ncc+index", conv_sq_dist=1e-300)  # default threshold 100 > k
    eng.init_from_seeds(np.arange(16))
    for _ in range(4):
        st = eng.step()
        assert not st.index_active and st.index_queries == 0 and st.candidates_total == 0


def test_index_counters_reported_through_step_and_cluster():
    m = S.generate(2000, 1200, 10, 30.0, seed=17)
    res = P.cluster(m, k=30, mode="ncc+index", index_activation_threshold=2, init_seeds=np.arange(30),
                    conv_sq_dist=1e-300, max_iters=6)
    act = [it for it in res.iterations if it.index_active]
    assert act and all(it.index_queries > 0 and it.candidates_total > 0 for it in act)
    assert all(it.index_build_seconds > 0 for it in act)
    base = P.cluster(m, k=30, mode="ncc", init_seeds=np.arange(30), conv_sq_dist=1e-300, max_iters=6)
    assert np.array_equal(res.assignments, base.assignments)
