"""The bound screen's result does not depend on θ (bound_kernels.cuh header).

θ only moves work between the high pairs, the candidate dots and the exact
scan, so every θ — including the degenerate ones (θ tiny: nearly every weight
high, dense touched sweeps; θ huge: no high pairs, every document falls
through to the exact tile scan) — and the postings screen (SSKM_BOUND=0) must
produce bit-identical trajectories. Checked on one cluster tile and on two
(k > 2048), on nonnegative and signed corpora, in baseline and NCC modes;
the default run is also teacher-forced against the oracle.
"""
import numpy as np
import pytest

import paper_2108_00895_b200 as P
from oracle import oracle as O
from paper_2108_00895_b200 import synthetic as S
from tests._util import csr_from_rows, random_unit_rows

pytestmark = pytest.mark.gpu


def trajectory(m, k, seeds, mode, iters):
    thetas = []
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(k, mode=mode, conv_sq_dist=1e-300, max_iters=iters)
    eng.init_from_seeds(seeds)
    out = []
    for _ in range(iters):
        st = eng.step()
        a, s, _ = eng.get_state()
        out.append((a.copy(), s.copy(), st.dot_products, st.n_reassigned))
        thetas.append(st.bound_theta)
    return out, thetas


def assert_same(t0, t1, label):
    assert len(t0) == len(t1)
    for it, (x, y) in enumerate(zip(t0, t1)):
        assert np.array_equal(x[0], y[0]), f"{label}: assignments differ at iteration {it + 1}"
        assert np.array_equal(x[1], y[1]), f"{label}: sims differ at iteration {it + 1}"
        assert x[2:] == y[2:], f"{label}: counters differ at iteration {it + 1}"


def signed_corpus(n, dims, seed):
    rows = random_unit_rows(np.random.default_rng(seed), n, dims, 30, allow_negative=True)
    rows = [[(d, float(np.float32(w))) for d, w in r] for r in rows]
    return P.CorpusMatrix.from_csr(*csr_from_rows(rows, dims=dims, dtype=np.float32))


CASES = {
    "one_tile": lambda: (S.generate(3000, 4096, 24, 60.0, seed=11), 64),
    "two_tiles": lambda: (S.generate(6000, 8192, 300, 50.0, seed=12), 2100),
    "signed": lambda: (signed_corpus(2500, 800, 5), 40),
    "five_tiles": lambda: (S.generate(12000, 8192, 600, 40.0, seed=13), 9000),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("mode", ["baseline", "ncc"])
def test_theta_and_screen_invariance(case, mode, monkeypatch):
    m, k = CASES[case]()
    seeds = np.random.default_rng(0).choice(m.n_docs, k, replace=False)
    iters = 5
    ref, _ = trajectory(m, k, seeds, mode, iters)
    for theta in ("1e-5", "0.02", "0.3"):
        monkeypatch.setenv("SSKM_THETA", theta)
        t, th = trajectory(m, k, seeds, mode, iters)
        assert_same(ref, t, f"theta={theta}")
        # the fixed split was the one used (passes that ran the bound screen)
        assert any(x > 0 for x in th) and all(x == 0 or x == pytest.approx(float(theta), rel=1e-6) for x in th)
    monkeypatch.delenv("SSKM_THETA")
    if k > 2048:  # one hash-accumulator pass by default; a pass per 2048-cluster tile without
        monkeypatch.setenv("SSKM_HASH", "0")
        t, _ = trajectory(m, k, seeds, mode, iters)
        assert_same(ref, t, "tile passes")
        monkeypatch.delenv("SSKM_HASH")
    if mode == "ncc":
        # by default an exact-NCC step runs as the (bit-identical) full screened scan with the
        # drift bound; the passes over the changed list (pass A, rescan) must give the same
        for frac in ("2.0", "0.25"):
            monkeypatch.setenv("SSKM_NCC_FULL_FRAC", frac)
            t, _ = trajectory(m, k, seeds, mode, iters)
            assert_same(ref, t, f"NCC changed-list passes (full frac {frac})")
        monkeypatch.delenv("SSKM_NCC_FULL_FRAC")
    monkeypatch.setenv("SSKM_BOUND", "0")
    t, th = trajectory(m, k, seeds, mode, iters)
    assert_same(ref, t, "postings screen")
    assert all(x == 0 for x in th)  # no bound-screen pass ran


def test_bound_default_teacher_forced_against_oracle():
    """Default (adaptive θ) bound screen vs the oracle's assign on the GPU's
    centroids and state, bitwise, on two cluster tiles."""
    m, k = CASES["two_tiles"]()
    seeds = np.random.default_rng(0).choice(m.n_docs, k, replace=False)
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(k, mode="baseline", conv_sq_dist=1e-300, max_iters=10)
    eng.init_from_seeds(seeds)
    c = O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), m.dims)
    ref = O.Stepper(c, k, "baseline", kind="ref" if O.ref_available() else "port")
    for it in range(1, 5):
        eng.update()
        a_mid, s_mid, unch = eng.get_state()
        ct = eng.get_centroids()
        st = eng.assign()
        assert st.bound_docs > 0 or it == 1
        a, s, _ = eng.get_state()
        ref.set_centroids_dense(ct)
        ref.set_state(a_mid, s_mid, unch, it)
        ref.assign()
        ra, rs, _ = ref.get_state()
        assert np.array_equal(ra, a), it
        assert np.array_equal(rs, s), it


@pytest.mark.parametrize("case", ["two_tiles", "five_tiles"])
@pytest.mark.parametrize("mode", ["baseline", "ncc"])
def test_hash_second_pass_is_exact(case, mode, monkeypatch):
    """Hash-accumulator passes (k > 2048): documents the first pass cannot settle
    are screened again at a lower θ with larger tables before the exact scan
    (bound_second_pass); with or without that pass, and for any θ ratio, the
    trajectory is the same bit for bit. θ = 0.1 makes many documents fall
    through; the leftovers take the span-parallel exact scan."""
    m, k = CASES[case]()
    seeds = np.random.default_rng(0).choice(m.n_docs, k, replace=False)
    monkeypatch.setenv("SSKM_THETA", "0.1")
    monkeypatch.setenv("SSKM_SECOND_PASS", "0")
    ref, _ = trajectory(m, k, seeds, mode, 4)
    monkeypatch.setenv("SSKM_SECOND_PASS", "1")
    monkeypatch.setenv("SSKM_SECOND_MIN", "1")
    ran = 0
    for ratio in ("0.5", "0.05"):
        monkeypatch.setenv("SSKM_SECOND_RATIO", ratio)
        eng = P.Engine(0)
        eng.upload(m)
        eng.configure(k, mode=mode, conv_sq_dist=1e-300, max_iters=4)
        eng.init_from_seeds(seeds)
        out = []
        for _ in range(4):
            st = eng.step()
            ran += st.second_pass_docs
            a, s, _ = eng.get_state()
            out.append((a.copy(), s.copy(), st.dot_products, st.n_reassigned))
        assert_same(ref, out, f"second pass ratio={ratio}")
    if mode == "baseline":
        assert ran > 0  # the second pass did run


@pytest.mark.parametrize("case", sorted(CASES))
def test_postings_overflow_stays_exact(case, monkeypatch):
    """A high-postings buffer too small for the first bound pass: single-tile
    passes drop the overflowing lists and bound those terms by their largest
    weight (looser, still exact); multi-tile passes grow and rebuild."""
    m, k = CASES[case]()
    seeds = np.random.default_rng(0).choice(m.n_docs, k, replace=False)
    ref, _ = trajectory(m, k, seeds, "baseline", 4)
    monkeypatch.setenv("SSKM_PAIRS_CAP", "64")
    t, _ = trajectory(m, k, seeds, "baseline", 4)
    assert_same(ref, t, "pairs cap 64")


@pytest.mark.parametrize("case", ["one_tile", "two_tiles", "signed", "five_tiles"])
def test_drift_bound_skip_is_exact(case, monkeypatch):
    """Documents kept in their cluster by the drift bound (skip_test_kernel)
    must leave exactly the trajectory of screening every document
    (SSKM_SKIP=0), and the bound must actually keep documents once the
    centroids settle."""
    m, k = CASES[case]()
    seeds = S.init_seeds(m.n_docs, k, 0)
    iters = 16

    def run():
        eng = P.Engine(0)
        eng.upload(m)
        eng.configure(k, mode="baseline", conv_sq_dist=1e-300, max_iters=iters)
        eng.init_from_seeds(seeds)
        out, skipped = [], 0
        for _ in range(iters):
            st = eng.step()
            a, s, _ = eng.get_state()
            out.append((a.copy(), s.copy(), st.dot_products, st.n_reassigned))
            skipped += st.skip_docs
        return out, skipped

    monkeypatch.setenv("SSKM_SKIP", "0")
    ref, s0 = run()
    monkeypatch.setenv("SSKM_SKIP", "1")
    got, s1 = run()
    assert s0 == 0
    assert s1 > 0
    assert_same(ref, got, f"skip {case}")


@pytest.mark.parametrize("case", ["one_tile", "signed", "two_tiles"])
def test_kept_postings_equal_a_rebuild(case):
    """The high postings kept across iterations and maintained in place by the
    column rewrite (hipost_maintain) hold exactly the entries a fresh build at
    the same θ would, after every update and assign."""
    m, k = CASES[case]()
    eng = P.Engine(0)
    eng.upload(m)
    eng.configure(k, mode="baseline", conv_sq_dist=1e-300, max_iters=20)
    eng.init_from_seeds(S.init_seeds(m.n_docs, k, 0))
    checked = 0
    for _ in range(14):
        eng.update()
        bad = eng.debug_check_postings()
        assert bad in (-1, 0), bad
        checked += bad == 0
        eng.assign()
        bad = eng.debug_check_postings()
        assert bad in (-1, 0), bad
    assert checked >= 5  # the lists were kept (not rebuilt) on most updates
