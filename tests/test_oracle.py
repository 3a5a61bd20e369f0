"""CPU: pin the oracle.

1. The plain-C restatement (oracle "port") reproduces the committed golden
   vectors that the UNMODIFIED reference produced (tests/golden/make_golden.py),
   bit for bit: per-iteration assignments, sims, stats, final centroids.
2. The reference's own known-answer tests for the hot path
   (proj/tests/test_engine.cpp, test_sparsevec.cpp, test_smoke.py), re-expressed
   against the oracle API, pass on the port — and on the compiled reference
   when oracle/_ref is built.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests._util import csr_from_rows, e, oracle_corpus, random_unit_rows, unit
from tests.conftest import golden_names

KINDS = ["port", "ref"]


def _kind(kind, ref_available):
    if kind == "ref" and not ref_available:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return kind


# ------------------------------------------------------------- golden pins --
@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("mode", ["baseline", "ncc"])
@pytest.mark.parametrize("kind", KINDS)
def test_trajectory_matches_golden(golden, name, mode, kind, ref_available):
    _kind(kind, ref_available)
    g = golden(name)
    c = O.Corpus(g["indptr"], g["indices"], g["values"].astype(np.float64), int(g["dims"]))
    r = O.run_seeded(c, int(g["k"]), g["seeds"], mode=mode, conv_sq_dist=float(g["conv_sq_dist"]),
                     max_iters=int(g["max_iters"]), kind=kind, record=True)
    n_it = len(g[f"{mode}_stats_iteration"])
    assert len(r["iterations"]) == n_it
    for t in range(n_it):
        a, s, u = r["trace"][t]
        np.testing.assert_array_equal(a, g[f"{mode}_trace_assignments"][t])
        np.testing.assert_array_equal(s, g[f"{mode}_trace_sims"][t])  # bitwise
        np.testing.assert_array_equal(u, g[f"{mode}_trace_unchanged"][t])
    for key in ["n_unchanged_centroids", "n_reassigned", "dot_products", "n_repaired"]:
        np.testing.assert_array_equal([it[key] for it in r["iterations"]], g[f"{mode}_stats_{key}"])
    for key in ["max_sq_drift", "objective"]:
        np.testing.assert_array_equal([it[key] for it in r["iterations"]], g[f"{mode}_stats_{key}"])
    assert r["stop_reason"] == str(g[f"{mode}_stop_reason"])
    ptr, idx, val = O.dense_to_csr(r["centroids"], int(g["k"]))
    np.testing.assert_array_equal(ptr, g[f"{mode}_centroid_ptr"])
    np.testing.assert_array_equal(idx, g[f"{mode}_centroid_idx"])
    np.testing.assert_array_equal(val, g[f"{mode}_centroid_val"])


def test_repair_fixture_exercises_repair(golden):
    g = golden("repair_400_k6")
    assert g["baseline_stats_n_repaired"][0] == 2


def test_port_kmeanspp_matches_golden(golden):
    g = golden("kmeanspp_600_k10")
    c = O.Corpus(g["indptr"], g["indices"], g["values"].astype(np.float64), int(g["dims"]))
    s = O.Stepper(c, 10, "baseline", kind="port")
    seeds = s.init_kmeanspp(3)
    np.testing.assert_array_equal(seeds, g["kpp_seeds"])
    a, sm, _ = s.get_state()
    np.testing.assert_array_equal(a, g["kpp_assignments"])
    np.testing.assert_array_equal(sm, g["kpp_sims"])


def test_mt19937_64_known_answer():
    # std::mt19937_64 default-seed (5489) 10000th output, C++11 [rand.predef]
    assert O._load("port").o_mt64_draw(5489, 9999) == 9981545732273789042


# ------------------------------------------------------- sparse-vector KATs --
@pytest.mark.parametrize("kind", KINDS)
def test_dot_kats(kind, ref_available):
    # test_sparsevec.cpp:29-38
    _kind(kind, ref_available)
    assert O.dot([0, 1], [0.6, 0.8], [1, 2], [0.8, 0.6], kind) == pytest.approx(0.64, abs=1e-12)
    assert O.dot([0], [1.0], [1], [1.0], kind) == 0.0
    i, v = O.normalize([0, 4, 9], [1.0, 2.0, 2.0], kind)
    assert O.dot(i, v, i, v, kind) == pytest.approx(1.0, abs=1e-9)


@pytest.mark.parametrize("kind", KINDS)
def test_dot_symmetric_and_gallop(kind, ref_available):
    # test_sparsevec.cpp:40-64: bitwise symmetry; gallop agrees with a dense oracle
    _kind(kind, ref_available)
    rng = np.random.default_rng(41)
    for trial in range(100):
        a = unit(list(zip(np.sort(rng.choice(60, 1 + trial % 12, replace=False)).tolist(),
                          (1 - rng.random(1 + trial % 12)).tolist())))
        b = unit(list(zip(np.sort(rng.choice(60, 1 + (trial * 7) % 12, replace=False)).tolist(),
                          (1 - rng.random(1 + (trial * 7) % 12)).tolist())))
        ai, av = zip(*a)
        bi, bv = zip(*b)
        ab = O.dot(ai, av, bi, bv, kind)
        assert ab == O.dot(bi, bv, ai, av, kind)
        da, db = np.zeros(60), np.zeros(60)
        da[list(ai)] = av
        db[list(bi)] = bv
        assert ab == pytest.approx(float(da @ db), abs=1e-12)
    big_i = np.arange(4000) * 2
    big_v = 0.01 + (np.arange(4000) % 7)
    bi, bv = O.normalize(big_i, big_v, kind)
    si, sv = O.normalize([0, 3998, 7300], [1.0, 2.0, 3.0], kind)
    got = O.dot(bi, bv, si, sv, kind)
    dense_b, dense_s = np.zeros(8000), np.zeros(8000)
    dense_b[bi] = bv
    dense_s[si] = sv
    assert got == pytest.approx(float(dense_b @ dense_s), abs=1e-12)
    assert got == O.dot(si, sv, bi, bv, kind)


@pytest.mark.parametrize("kind", KINDS)
def test_normalize_kats(kind, ref_available):
    # test_sparsevec.cpp:66-92
    _kind(kind, ref_available)
    i, v = O.normalize([0, 1], [3.0, 4.0], kind)
    assert v.tolist() == [0.6, 0.8]
    i, v = O.normalize([7], [5.0], kind)
    assert i.tolist() == [7] and v.tolist() == [1.0]
    with pytest.raises(ValueError, match="cannot normalize zero vector"):
        O.normalize([], [], kind)
    for trial in range(60):
        i, v = O.normalize([trial, 1000 + trial * 3, 5000], [0.3, 1e-7, 17.0 + trial], kind)
        assert abs(math.sqrt(float(np.sum(v * v))) - 1.0) <= 1e-9
        i2, v2 = O.normalize(i, v, kind)
        assert np.array_equal(i2, i) and np.array_equal(v2, v)  # bitwise idempotent


def test_port_normalize_matches_ref_bitwise(ref_available):
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(2, 40))
        i = np.sort(rng.choice(1000, n, replace=False))
        v = rng.standard_normal(n) * 10 ** rng.uniform(-3, 3, n)
        a = O.normalize(i, v, "ref")
        b = O.normalize(i, v, "port")
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ------------------------------------------------------------- engine KATs --
def stepper_from_rows(rows, k, mode="baseline", kind="port", **kw):
    c = oracle_corpus(*csr_from_rows(rows))
    return c, O.Stepper(c, k, mode, kind=kind, **kw)


@pytest.mark.parametrize("kind", KINDS)
def test_assignment_picks_mixed_centroid(kind, ref_available):
    # test_engine.cpp:362-381
    _kind(kind, ref_available)
    x = unit([(0, 1.0), (1, 0.9)])
    c, s = stepper_from_rows([x, e(0), e(1)], 3, kind=kind)
    cents = [e(0), e(1), unit([(0, 1.0), (1, 1.0)])]
    ptr, idx, val, _ = csr_from_rows(cents, dims=2)
    s.init_seeds([1, 2, 0])  # any state; overwritten below
    s.set_centroids_csr(ptr, idx.astype(np.uint32), val)
    s.set_state([0, 0, 0], [-2.0] * 3, [0, 0, 0], 1)
    st = s.assign()
    a, sm, _ = s.get_state()
    assert a[0] == 2
    assert sm[0] == pytest.approx(1.9 / math.sqrt(3.62), rel=1e-12)
    assert st["dot_products"] == 3 * 3


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("case", ["lowest", "ties", "multiple", "donor_size"])
def test_empty_cluster_repair(kind, case, ref_available):
    # test_engine.cpp:283-313
    _kind(kind, ref_available)
    c, s = stepper_from_rows([e(0), e(1), e(2), e(3)], {"multiple": 3, "donor_size": 3}.get(case, 2),
                             kind=kind)
    a, sims, exp_a, exp_rep = {
        "lowest": ([0, 0, 0, 0], [0.9, 0.2, 0.5, 0.8], [0, 1, 0, 0], [1]),
        "ties": ([0, 0, 0, 0], [0.5] * 4, [1, 0, 0, 0], [1]),
        "multiple": ([0, 0, 0, 0], [0.9, 0.2, 0.5, 0.8], [0, 1, 2, 0], [1, 2]),
        "donor_size": ([0, 0, 1, 1], [0.1, 0.9, 0.2, 0.3], [2, 0, 1, 1], [2]),
    }[case]
    new_a, rep = s.compute_centroids(a, sims)
    assert new_a.tolist() == exp_a
    assert rep.tolist() == exp_rep


@pytest.mark.parametrize("kind", KINDS)
def test_compute_centroids_examples(kind, ref_available):
    # test_engine.cpp:210-281
    _kind(kind, ref_available)
    c, s = stepper_from_rows([e(0), e(1), e(7)], 2, kind=kind)
    new_a, rep = s.compute_centroids([0, 0, 1], [1.0, 1.0, 1.0])
    assert rep.tolist() == []
    ptr, idx, val = s.get_centroids_csr()
    assert idx[ptr[0]:ptr[1]].tolist() == [0, 1]
    np.testing.assert_allclose(val[ptr[0]:ptr[1]], [0.70710678118654752] * 2, rtol=1e-12)
    # singletons reproduce their member bitwise
    rows = random_unit_rows(np.random.default_rng(21), 6, 25, 5)
    c, s = stepper_from_rows(rows, 6, kind=kind)
    s.compute_centroids(list(range(6)), [1.0] * 6)
    ptr, idx, val = s.get_centroids_csr()
    for j in range(6):
        assert list(zip(idx[ptr[j]:ptr[j + 1]].tolist(), val[ptr[j]:ptr[j + 1]].tolist())) == rows[j]


@pytest.mark.parametrize("kind", KINDS)
def test_ncc_all_unchanged_does_no_work(kind, ref_available):
    # test_engine.cpp:383-402
    _kind(kind, ref_available)
    rows = random_unit_rows(np.random.default_rng(13), 25, 20, 4)
    c, s = stepper_from_rows(rows, 4, mode="ncc", kind=kind)
    s.init_seeds([0, 5, 10, 15])
    st = s.step()
    assert st["dot_products"] == 4 * 25
    a, sm, _ = s.get_state()
    s.set_state(a, sm, np.ones(4, np.uint8), 2)
    st2 = s.assign()
    assert st2["dot_products"] == 0 and st2["n_reassigned"] == 0
    assert st2["n_unchanged_centroids"] == 4


@pytest.mark.parametrize("kind", KINDS)
def test_modes_equivalent_and_baseline_dot_count(kind, ref_available):
    # test_engine.cpp:404-461 (mode equivalence per iteration; baseline k·N dots)
    _kind(kind, ref_available)
    rng = np.random.default_rng(23)
    for inst in range(3):
        rows = random_unit_rows(rng, 120, 50, 8)
        c = oracle_corpus(*csr_from_rows(rows, dims=50))
        seeds = rng.choice(120, 10, replace=False)
        rb = O.run_seeded(c, 10, seeds, "baseline", kind=kind, record=True)
        rn = O.run_seeded(c, 10, seeds, "ncc", kind=kind, record=True)
        assert len(rb["trace"]) == len(rn["trace"])
        for tb, tn in zip(rb["trace"], rn["trace"]):
            assert np.array_equal(tb[0], tn[0]) and np.array_equal(tb[1], tn[1])
        for sb, sn in zip(rb["iterations"], rn["iterations"]):
            assert sb["dot_products"] == 10 * 120
            assert sn["dot_products"] <= sb["dot_products"]
            assert sb["n_reassigned"] == sn["n_reassigned"]


@pytest.mark.parametrize("kind", KINDS)
def test_objective_monotone_and_stop_reasons(kind, ref_available):
    # test_engine.cpp:549-602
    _kind(kind, ref_available)
    rng = np.random.default_rng(47)
    for inst in range(4):
        rows = random_unit_rows(rng, 100, 40, 6)
        c = oracle_corpus(*csr_from_rows(rows, dims=40))
        seeds = rng.choice(100, 8, replace=False)
        r = O.run_seeded(c, 8, seeds, "baseline" if inst % 2 == 0 else "ncc", kind=kind)
        objs = [it["objective"] for it in r["iterations"]]
        assert all(b >= a for a, b in zip(objs, objs[1:]))
    rows = random_unit_rows(rng, 60, 30, 5)
    c = oracle_corpus(*csr_from_rows(rows, dims=30))
    seeds = rng.choice(60, 6, replace=False)
    r = O.run_seeded(c, 6, seeds, max_iters=1, kind=kind)
    assert len(r["iterations"]) == 1
    if r["iterations"][0]["n_reassigned"] > 0:
        assert r["stop_reason"] == "max_iterations"
    r = O.run_seeded(c, 6, seeds, conv_sq_dist=1e9, kind=kind)
    assert len(r["iterations"]) <= 2
    if len(r["iterations"]) == 2 and r["iterations"][-1]["n_reassigned"] > 0:
        assert r["stop_reason"] == "centroid_drift"
    r = O.run_seeded(c, 4, seeds[:4], conv_sq_dist=1e-300, kind=kind)
    assert r["stop_reason"] == "no_reassignments"


@pytest.mark.parametrize("kind", KINDS)
def test_validation_messages(kind, ref_available):
    # engine.cpp:47-64, test_engine.cpp:128-149
    _kind(kind, ref_available)
    O.validate(10, 3, kind=kind)
    for kw in [dict(k=1), dict(k=11), dict(lambdas=(0.4, 0.2)), dict(lambdas=(0.0, 0.4)),
               dict(lambdas=(0.4, 1.0)), dict(conv_sq_dist=0.0), dict(ncc_epsilon=-1.0),
               dict(max_iters=0)]:
        args = dict(n_docs=10, k=3)
        args.update(kw)
        with pytest.raises(ValueError):
            O.validate(**args, kind=kind)
    O.validate(10, 3, lambdas=(), kind=kind)
