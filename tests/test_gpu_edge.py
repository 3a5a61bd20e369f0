"""GPU edge cases, each against the oracle through the C-ABI:
signed weights (absolute certification bound), k = N, empty document rows,
a cluster of only empty rows (the reference's zero-vector error), k = 2."""
import numpy as np
import pytest

import paper_2108_00895_b200 as P
from oracle import oracle as O
from paper_2108_00895_b200 import synthetic as S
from tests._util import csr_from_rows, random_unit_rows

pytestmark = pytest.mark.gpu


def f32_corpus(rows, dims):
    rows = [[(d, float(np.float32(w))) for d, w in r] for r in rows]
    return P.CorpusMatrix.from_csr(*csr_from_rows(rows, dims=dims, dtype=np.float32))


def gpu_run(m, k, seeds, mode="ncc", iters=12):
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(k, mode=mode, conv_sq_dist=1e-300, max_iters=iters)
    eng.init_from_seeds(seeds)
    trace = []
    for _ in range(iters):
        st = eng.step()
        a, s, u = eng.get_state()
        trace.append((a, s, st))
        if st.n_reassigned == 0:
            break
    return eng, trace


def oracle_teacher_check(m, k, seeds, mode="ncc", iters=12):
    """GPU steps; the oracle's assign on the GPU's centroids/state must agree bitwise."""
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(k, mode=mode, conv_sq_dist=1e-300, max_iters=iters)
    eng.init_from_seeds(seeds)
    c = O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), m.dims)
    ref = O.Stepper(c, k, mode, kind="port")
    for it in range(1, iters + 1):
        eng.update()
        a_mid, s_mid, unch = eng.get_state()
        ct = eng.get_centroids()
        st = eng.assign()
        a, s, _ = eng.get_state()
        ref.set_centroids_dense(ct)
        ref.set_state(a_mid, s_mid, unch, it)
        r = ref.assign()
        ra, rs, _ = ref.get_state()
        assert np.array_equal(ra, a) and np.array_equal(rs, s), it
        assert r["dot_products"] == st.dot_products
        if st.n_reassigned == 0:
            break


def test_signed_weights_absolute_bound():
    # allow_negative: centroids have mixed signs; the screen uses the absolute δ bound
    rows = random_unit_rows(np.random.default_rng(3), 1500, 300, 25, allow_negative=True)
    m = f32_corpus(rows, 300)
    seeds = np.random.default_rng(0).choice(m.n_docs, 24, replace=False)
    oracle_teacher_check(m, 24, seeds, "ncc", 10)
    oracle_teacher_check(m, 24, seeds, "baseline", 4)


def test_k_equals_n():
    m = S.generate(64, 500, 4, 20.0, seed=9)
    eng, trace = gpu_run(m, m.n_docs, np.arange(m.n_docs), iters=3)
    a, s, st = trace[0]
    assert np.array_equal(a, np.arange(m.n_docs))  # every document its own singleton cluster
    assert st.n_reassigned == 0
    np.testing.assert_allclose(s, 1.0, atol=1e-6)


def test_empty_rows():
    base = S.generate(400, 600, 6, 20.0, seed=4)
    rows = [list(zip(base.indices[base.indptr[i]:base.indptr[i + 1]].tolist(),
                     base.values[base.indptr[i]:base.indptr[i + 1]].tolist())) for i in range(base.n_docs)]
    for i in (5, 77, 200, 399):
        rows[i] = []  # documents with no terms: dot 0 with everything
    m = P.CorpusMatrix.from_csr(*csr_from_rows(rows, dims=600, dtype=np.float32))
    seeds = np.array([0, 10, 20, 30, 40, 50, 60, 70], np.uint32)
    oracle_teacher_check(m, 8, seeds, "ncc", 8)
    eng, trace = gpu_run(m, 8, seeds, iters=8)
    a, s, _ = trace[-1]
    assert all(s[i] == 0.0 for i in (5, 77, 200, 399))


def test_cluster_of_only_empty_rows_raises_like_reference():
    rows = [[], [], [(0, 1.0)], [(1, 1.0)], [(0, 0.6), (1, 0.8)]]
    m = P.CorpusMatrix.from_csr(*csr_from_rows(rows, dims=2, dtype=np.float32))
    seeds = np.array([0, 2, 3], np.uint32)  # cluster 0 = the two empty documents
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(3, conv_sq_dist=1e-300)
    eng.init_from_seeds(seeds)
    with pytest.raises(ValueError, match="cannot normalize zero vector"):
        eng.update()
    c = O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), 2)
    s = O.Stepper(c, 3, kind="ref" if O.ref_available() else "port")
    s.init_seeds(seeds)
    with pytest.raises(ValueError, match="cannot normalize zero vector"):
        s.step()


def test_minimum_k_and_tiny_corpus():
    m = S.generate(5, 40, 2, 6.0, seed=1)
    eng, trace = gpu_run(m, 2, [0, 1], mode="baseline", iters=5)
    oracle_teacher_check(m, 2, [0, 1], "baseline", 5)
    with pytest.raises(ValueError):
        P.cluster(m, k=6, init_seeds=list(range(6)))  # k > N
