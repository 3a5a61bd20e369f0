"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

Protocol (BASELINE north_star):
* teacher-forced assign: given the GPU's fp32 centroids and pre-assign state,
  the reference's assign must produce the GPU's assignments and sims — bitwise
  (fp64 accumulation of exact fp32 products in ascending term order);
* teacher-forced update: the reference's compute_centroids on the GPU's
  pre-update state must give the GPU's centroids within 1e-5 relative, and the
  same repaired clusters;
* free-running trajectories equal the reference's golden trajectory except at
  near-ties (|Δcos| ≤ 1e-5), objective within 1e-6 relative;
* mode equivalence holds bitwise on the GPU.
"""
import numpy as np
import pytest

import paper_2108_00895_b200 as P
from oracle import oracle as O
from paper_2108_00895_b200 import synthetic as S
from tests._util import csr_from_rows, e, random_unit_rows, unit
from tests.conftest import golden_names

pytestmark = pytest.mark.gpu

NEAR_TIE = 1e-5


def engine_for(m, k, mode="baseline", **kw):
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(k, mode=mode, **kw)
    return eng


def corpus_from_golden(g):
    return P.CorpusMatrix.from_csr(g["indptr"], g["indices"], g["values"], int(g["dims"]))


def ref_corpus(m, rows=None):
    if rows is None:
        return O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), m.dims)
    lens = np.diff(m.indptr)[rows]
    ptr = np.zeros(len(rows) + 1, np.int64)
    ptr[1:] = np.cumsum(lens)
    idx = np.concatenate([m.indices[m.indptr[i]:m.indptr[i + 1]] for i in rows])
    val = np.concatenate([m.values[m.indptr[i]:m.indptr[i + 1]] for i in rows])
    return O.Corpus(ptr, idx, val.astype(np.float64), m.dims)


def near_tie_ok(ref_stepper_centroids_dense, m, docs, a_gpu, a_ref):
    """Every differing assignment must be a near-tie under the reference's dots."""
    for i in np.nonzero(a_gpu != a_ref)[0]:
        d = docs[i]
        b, e_ = m.indptr[d], m.indptr[d + 1]
        x = np.zeros(m.dims)
        x[m.indices[b:e_]] = m.values[b:e_]
        s_gpu = float(x @ ref_stepper_centroids_dense[:, a_gpu[i]])
        s_ref = float(x @ ref_stepper_centroids_dense[:, a_ref[i]])
        assert abs(s_gpu - s_ref) <= NEAR_TIE, (d, s_gpu, s_ref)


# ------------------------------------------------------------- KATs on GPU --
def test_gpu_mixed_centroid_assignment():
    # test_engine.cpp:362-381 with fp32 storage
    x = [(d, float(np.float32(w))) for d, w in unit([(0, 1.0), (1, 0.9)])]
    m = P.CorpusMatrix.from_csr(*csr_from_rows([x, e(0), e(1)], dims=2, dtype=np.float32))
    eng = engine_for(m, 3)
    eng.init_from_seeds([1, 2, 0])
    ct = np.zeros((2, 3), np.float32)
    ct[0, 0] = 1.0
    ct[1, 1] = 1.0
    mixed = unit([(0, 1.0), (1, 1.0)])
    ct[0, 2], ct[1, 2] = mixed[0][1], mixed[1][1]
    eng.set_centroids(ct)
    eng.set_state([0, 0, 0], [-2.0] * 3, 1)
    st = eng.assign()
    a, s, _ = eng.get_state()
    assert a[0] == 2
    assert s[0] == pytest.approx(1.9 / np.sqrt(3.62), rel=1e-6)
    assert st.dot_products == 9
    # bitwise vs the reference fed the same fp32 values
    c = O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), 2)
    r = O.Stepper(c, 3, kind="port")
    r.init_seeds([1, 2, 0])
    r.set_centroids_dense(ct.astype(np.float64))
    r.set_state([0, 0, 0], [-2.0] * 3, [0, 0, 0], 1)
    r.assign()
    ra, rs, _ = r.get_state()
    assert np.array_equal(ra, a) and np.array_equal(rs, s)


@pytest.mark.parametrize("case", ["lowest", "ties", "multiple", "donor_size"])
def test_gpu_empty_cluster_repair(case):
    # test_engine.cpp:283-313
    m = P.CorpusMatrix.from_csr(*csr_from_rows([e(0), e(1), e(2), e(3)], dtype=np.float32))
    k = {"multiple": 3, "donor_size": 3}.get(case, 2)
    a, sims, exp_a, exp_rep = {
        "lowest": ([0, 0, 0, 0], [0.9, 0.2, 0.5, 0.8], [0, 1, 0, 0], [1]),
        "ties": ([0, 0, 0, 0], [0.5] * 4, [1, 0, 0, 0], [1]),
        "multiple": ([0, 0, 0, 0], [0.9, 0.2, 0.5, 0.8], [0, 1, 2, 0], [1, 2]),
        "donor_size": ([0, 0, 1, 1], [0.1, 0.9, 0.2, 0.3], [2, 0, 1, 1], [2]),
    }[case]
    eng = engine_for(m, k)
    eng.init_from_seeds(list(range(k)))
    eng.set_state(a, sims, 0)
    st = eng.update()
    assert eng.repaired().tolist() == exp_rep
    assert st.n_repaired == len(exp_rep)
    assert eng.get_state()[0].tolist() == exp_a
    ct = eng.get_centroids()
    for j in range(k):  # every centroid is the unit axis of its (single or merged) members
        members = [i for i in range(4) if exp_a[i] == j]
        expect = np.zeros(4, np.float32)
        expect[members] = np.float32(1.0 / np.sqrt(len(members)))
        np.testing.assert_allclose(ct[:, j], expect, rtol=1e-6)


def test_gpu_ncc_all_unchanged_does_no_work_and_baseline_counts_kn():
    # test_engine.cpp:383-415
    rows = [[(d, float(np.float32(w))) for d, w in r] for r in random_unit_rows(np.random.default_rng(13), 25, 20, 4)]
    m = P.CorpusMatrix.from_csr(*csr_from_rows(rows, dims=20, dtype=np.float32))
    eng = engine_for(m, 4, mode="ncc")
    eng.init_from_seeds([0, 5, 10, 15])
    st = eng.step()
    assert st.dot_products == 4 * 25
    a, s, _ = eng.get_state()
    eng.set_unchanged(np.ones(4, np.uint8))
    eng.set_state(a, s, 2)
    st2 = eng.assign()
    assert st2.dot_products == 0 and st2.n_reassigned == 0 and st2.n_unchanged_centroids == 4
    eng_b = engine_for(m, 4, mode="baseline")
    eng_b.init_from_seeds([0, 5, 10, 15])
    for _ in range(3):
        assert eng_b.step().dot_products == 4 * 25


# --------------------------------------------------- golden trajectories ----
@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("mode", ["baseline", "ncc"])
def test_gpu_trajectory_vs_reference_golden(golden, name, mode):
    g = golden(name)
    m = corpus_from_golden(g)
    k = int(g["k"])
    eng = engine_for(m, k, mode=mode, conv_sq_dist=float(g["conv_sq_dist"]), max_iters=int(g["max_iters"]))
    eng.init_from_seeds(g["seeds"])
    a0, s0, _ = eng.get_state()
    np.testing.assert_array_equal(a0, g["seed_assignments"])
    np.testing.assert_array_equal(s0, g["seed_sims"])  # seed docs are fp32 already: bitwise
    its, stop = eng.run()
    n_ref = len(g[f"{mode}_stats_iteration"])
    ref_final = O.csr_to_dense(g[f"{mode}_centroid_ptr"], g[f"{mode}_centroid_idx"],
                               g[f"{mode}_centroid_val"], k, m.dims)
    a, s, _ = eng.get_state()
    diff = np.nonzero(a != g[f"{mode}_assignments"])[0]
    assert len(diff) <= max(1, m.n_docs // 1000)
    if len(diff) == 0:
        assert len(its) == n_ref and stop == str(g[f"{mode}_stop_reason"])
        np.testing.assert_allclose(s, g[f"{mode}_sims"], rtol=0, atol=1e-6)
        for key in ["n_reassigned", "dot_products", "n_repaired", "n_unchanged_centroids"]:
            np.testing.assert_array_equal([getattr(it, key) for it in its], g[f"{mode}_stats_{key}"])
        np.testing.assert_allclose([it.objective for it in its], g[f"{mode}_stats_objective"], rtol=1e-6)
        ct = eng.get_centroids().astype(np.float64)
        nrm = np.linalg.norm(ref_final, axis=0)
        assert np.max(np.linalg.norm(ct - ref_final, axis=0) / nrm) <= 1e-5
    else:
        near_tie_ok(ref_final, m, diff, a[diff], g[f"{mode}_assignments"][diff])


# ---------------------------------------------------- teacher forcing -------
def centroid_rel_err(ct, ptr, idx, val, cols=None):
    """max_j ||c_gpu_j - c_ref_j|| / ||c_ref_j|| and max elementwise |Δ|, column by column."""
    worst_rel, worst_abs = 0.0, 0.0
    for j in (range(ct.shape[1]) if cols is None else cols):
        ref = np.zeros(ct.shape[0])
        ref[idx[ptr[j]:ptr[j + 1]]] = val[ptr[j]:ptr[j + 1]]
        d = ct[:, j].astype(np.float64) - ref
        worst_rel = max(worst_rel, float(np.linalg.norm(d) / np.linalg.norm(ref)))
        worst_abs = max(worst_abs, float(np.max(np.abs(d))))
    return worst_rel, worst_abs


def teacher_forced(m, k, seeds, mode, iters, sample=None, kind=None, n_cols=None, ncc_epsilon=0.0):
    """Run the GPU; at every iteration feed its state/centroids to the oracle
    (the compiled reference when present)."""
    if kind is None:
        kind = "ref" if O.ref_available() else "port"
    eng = engine_for(m, k, mode=mode, conv_sq_dist=1e-300, max_iters=iters, ncc_epsilon=ncc_epsilon)
    eng.init_from_seeds(seeds)
    docs = np.arange(m.n_docs) if sample is None else np.sort(sample)
    c_full = ref_corpus(m)
    c_samp = c_full if sample is None else ref_corpus(m, docs)
    upd = O.Stepper(c_full, k, mode, kind=kind, ncc_epsilon=ncc_epsilon)
    asg = upd if sample is None else O.Stepper(c_samp, min(k, c_samp.n), mode, kind=kind, ncc_epsilon=ncc_epsilon)
    if sample is not None:
        assert k <= c_samp.n
    report = []
    for it in range(1, iters + 1):
        a_pre, s_pre, _ = eng.get_state()
        st_u = eng.update()
        # --- update parity: reference compute_centroids on the GPU's pre-update state
        a_rep, rep = upd.compute_centroids(a_pre, s_pre)
        a_mid, s_mid, unch = eng.get_state()
        np.testing.assert_array_equal(rep, eng.repaired())
        np.testing.assert_array_equal(a_rep, a_mid)
        ct = eng.get_centroids()
        cols = None
        if n_cols is not None:  # large k: a seeded sample of columns plus every repaired one
            cols = sorted(set(np.random.default_rng(it).choice(k, n_cols, replace=False).tolist())
                          | set(eng.repaired().tolist()))
        rel, ab = centroid_rel_err(ct, *upd.get_centroids_csr(), cols=cols)
        assert rel <= 1e-5 and ab <= 1e-5, (it, rel, ab)
        # --- assign parity: reference assign with the GPU's fp32 centroids and state
        st_a = eng.assign()
        a_post, s_post, _ = eng.get_state()
        asg.set_centroids_dense(ct)
        asg.set_state(a_mid[docs], s_mid[docs], unch, it)
        r = asg.assign()
        ra, rs, _ = asg.get_state()
        np.testing.assert_array_equal(ra, a_post[docs])
        np.testing.assert_array_equal(rs, s_post[docs])  # bitwise
        if sample is None:
            assert r["dot_products"] == st_a.dot_products
            assert r["n_reassigned"] == st_a.n_reassigned
            assert st_a.objective == pytest.approx(r["objective"], rel=1e-12)
        report.append((it, st_u.n_recomputed, st_a.n_changed, st_a.n_reassigned, rel))
    return report


@pytest.mark.parametrize("mode", ["baseline", "ncc"])
def test_gpu_teacher_forced_c0(mode):
    cfg = S.CONFIGS["c0"]
    m = S.corpus(cfg)
    seeds = S.init_seeds(m.n_docs, cfg.k, 0)
    rep = teacher_forced(m, cfg.k, seeds, mode, cfg.iterations)
    assert len(rep) == cfg.iterations


def test_gpu_teacher_forced_approximate_ncc():
    """ncc_epsilon > 0: centroids that moved by less than epsilon
    are treated as unchanged; the GPU must follow the reference's NCC literally
    (no full-scan shortcut) and still match it bitwise given the same state."""
    m = S.generate(8000, 4096, 20, 60.0, seed=8)
    seeds = S.init_seeds(m.n_docs, 40, 0)
    rep = teacher_forced(m, 40, seeds, "ncc", 10, ncc_epsilon=2e-3)
    assert len(rep) == 10


def test_gpu_modes_bitwise_equivalent_c0():
    cfg = S.CONFIGS["c0"]
    m = S.corpus(cfg)
    seeds = S.init_seeds(m.n_docs, cfg.k, 0)
    engs = {md: engine_for(m, cfg.k, mode=md, conv_sq_dist=1e-300) for md in ("baseline", "ncc", "ncc+index")}
    for eng in engs.values():
        eng.init_from_seeds(seeds)
    total = {md: 0 for md in engs}
    for it in range(cfg.iterations):
        out = {}
        for md, eng in engs.items():
            st = eng.step()
            total[md] += st.dot_products
            out[md] = (eng.get_state(), eng.get_centroids(), st)
        for md in ("ncc", "ncc+index"):
            assert np.array_equal(out[md][0][0], out["baseline"][0][0])
            assert np.array_equal(out[md][0][1], out["baseline"][0][1])
            assert np.array_equal(out[md][1], out["baseline"][1])
            assert out[md][2].n_reassigned == out["baseline"][2].n_reassigned
            assert out[md][2].objective == out["baseline"][2].objective
            assert out[md][2].dot_products <= out["baseline"][2].dot_products
    assert total["ncc"] < total["baseline"]


# ------------------------------------------------- public API (test_smoke) --
def test_gpu_cluster_runs_and_is_deterministic():
    # test_smoke.py:74-101
    data = S.generate(200, 500, 5, 8.0, seed=7)
    runs = [P.cluster(data, k=6, mode="ncc+index", seed=11, index_activation_threshold=0, threads=t)
            for t in (1, 2)]
    first = runs[0]
    assert len(first.assignments) == data.n_docs
    assert first.n_clusters == 6
    assert first.stop_reason in ("no_reassignments", "centroid_drift", "max_iterations")
    assert first.iterations[0].dot_products == 6 * data.n_docs
    assert 0.0 < first.objective <= data.n_docs + 1e-9
    for other in runs[1:]:
        assert np.array_equal(other.assignments, first.assignments)
        assert other.objective == first.objective
    results = {md: P.cluster(data, k=5, mode=md, seed=4, index_activation_threshold=0)
               for md in ("baseline", "ncc", "ncc+index")}
    base = results["baseline"]
    assert np.array_equal(results["ncc"].assignments, base.assignments)
    assert np.array_equal(results["ncc+index"].assignments, base.assignments)
    assert results["ncc"].total_dot_products() <= base.total_dot_products()


def test_gpu_kmeanspp_matches_reference(golden):
    g = golden("kmeanspp_600_k10")
    m = corpus_from_golden(g)
    eng = engine_for(m, 10)
    seeds = eng.init_kmeanspp(3)
    np.testing.assert_array_equal(seeds, g["kpp_seeds"])
    a, s, _ = eng.get_state()
    np.testing.assert_array_equal(a, g["kpp_assignments"])
    np.testing.assert_array_equal(s, g["kpp_sims"])
    for mode in ("baseline", "ncc"):
        r = P.cluster(m, 10, mode=mode, seed=3)
        same = np.mean(r.assignments == g[f"run_{mode}_assignments"])
        assert same >= 0.995
        assert r.objective == pytest.approx(float(g[f"run_{mode}_objective"]), rel=1e-6)


def test_gpu_sims_are_live_dots_and_objective_monotone():
    # test_engine.cpp:481-563: cached sims = dots vs final centroids; objective non-decreasing
    m = S.generate(5000, 4096, 30, 50.0, seed=21)
    seeds = S.init_seeds(m.n_docs, 40, 0)
    r = P.cluster(m, 40, mode="ncc", init_seeds=seeds, conv_sq_dist=1e-300, return_centroids=True)
    objs = [it.objective for it in r.iterations]
    assert all(b >= a - 1e-12 for a, b in zip(objs, objs[1:]))
    ct = r.centroids.astype(np.float64)
    for i in range(0, m.n_docs, 50):
        b, e_ = m.indptr[i], m.indptr[i + 1]
        dots = m.values[b:e_].astype(np.float64) @ ct[m.indices[b:e_], :]
        assert r.sims[i] == pytest.approx(dots[r.assignments[i]], abs=1e-12)
        assert dots.max() - dots[r.assignments[i]] <= 1e-12


def test_gpu_cluster_cached_engine_reshapes():
    """cluster() reuses one engine per device: a larger vocabulary with the same
    k, then a smaller corpus, must give the same results as fresh engines."""
    import ctypes  # noqa: F401
    from paper_2108_00895_b200 import _lib

    small = S.generate(3000, 2048, 8, 40.0, seed=3)
    big = S.generate(5000, 8192, 8, 40.0, seed=4)
    out = []
    for m in (small, big, small):
        seeds = S.init_seeds(m.n_docs, 16, 0)
        r = P.cluster(m, 16, mode="ncc", init_seeds=seeds, conv_sq_dist=1e-300, max_iters=8,
                      return_centroids=True)
        eng = engine_for(m, 16, mode="ncc", conv_sq_dist=1e-300, max_iters=8)
        eng.init_from_seeds(seeds)
        its, _ = eng.run()
        a, s, _ = eng.get_state()
        assert np.array_equal(r.assignments, a) and np.array_equal(r.sims, s)
        assert np.array_equal(r.centroids, eng.get_centroids())
        eng.close()
        out.append(r.objective)
    assert out[0] == out[2]
    _lib.check(_lib.load().sskm_release_cache())


@pytest.mark.parametrize("k", [100, 400])
def test_gpu_kmeanspp_device_rounds_match_reference(k, monkeypatch):
    """Device-resident k-means++ rounds (bracketed sequential sums, exact pick)
    give the reference's seeds, the host-replayed rounds' seeds, and the same
    nearest-seed state, on config 0."""
    m = S.corpus(S.CONFIGS["c0"])
    eng = engine_for(m, k)
    seeds = eng.init_kmeanspp(5)
    a, s, _ = eng.get_state()
    monkeypatch.setenv("SSKM_KPP_HOST", "1")
    eng2 = engine_for(m, k)
    seeds2 = eng2.init_kmeanspp(5)
    a2, s2, _ = eng2.get_state()
    np.testing.assert_array_equal(seeds, seeds2)
    np.testing.assert_array_equal(a, a2)
    np.testing.assert_array_equal(s, s2)
    if O.ref_available():
        c = O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), m.dims)
        rs, ra, rsims = O.seed_kmeanspp(c, k, 5)
        np.testing.assert_array_equal(seeds, rs)
        np.testing.assert_array_equal(a, ra)
        np.testing.assert_array_equal(s, rsims)


@pytest.mark.parametrize("mode", ["baseline", "ncc"])
def test_gpu_step_n_equals_steps(mode):
    """sskm_step_n: n iterations in one native call = n sskm_step calls, bit for
    bit (state and per-iteration counters)."""
    m = S.generate(5000, 4096, 24, 50.0, seed=21)
    k = 48
    seeds = S.init_seeds(m.n_docs, k, 0)
    a = engine_for(m, k, mode, conv_sq_dist=1e-300, max_iters=100)
    b = engine_for(m, k, mode, conv_sq_dist=1e-300, max_iters=100)
    a.init_from_seeds(seeds)
    b.init_from_seeds(seeds)
    sa = [a.step() for _ in range(6)]
    sb = b.step_n(6)
    assert len(sb) == 6
    for x, y in zip(sa, sb):
        assert (x.iteration, x.dot_products, x.n_reassigned, x.n_unchanged_centroids, x.objective) == \
               (y.iteration, y.dot_products, y.n_reassigned, y.n_unchanged_centroids, y.objective)
    (aa, asim, _), (ba, bsim, _) = a.get_state(), b.get_state()
    assert np.array_equal(aa, ba) and np.array_equal(asim, bsim)
