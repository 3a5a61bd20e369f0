"""GPU TF-IDF ingestion (csrc/vectorize.cu) against the reference's
vectorize_corpus (corpus.cpp:101-134) compiled in oracle/_ref: vocabulary
(dims in first-occurrence order), doc frequencies, n_docs, fp64 weights after
normalize, kept and dropped ids — all bitwise. Cases follow the reference's
test_corpus.cpp:45-177 and test_smoke.py:29-49, plus seeded synthetic texts
(tests/textgen.py) and normalize's long orbits (sparse_vector.cpp:184-208)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import textgen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "vectorize_golden.npz")

KAT_DOCS = [  # test_corpus.cpp:154-161
    ("d0", "alpha beta shared"),
    ("d1", "the of the"),
    ("d2", "beta gamma shared"),
    ("d3", "shared shared"),
    ("d4", "shared delta"),
    ("d5", "shared epsilon"),
]
SMOKE_DOCS = [  # test_smoke.py:35-40
    ("d1", "apple banana apple"),
    ("d2", "banana cherry"),
    ("d3", "the the"),
    ("d4", "apple cherry durian"),
]
EDGE_TEXTS = ["Sparse K-Means!", "", "the the the", "a1-b2 3c", "café, bar", "  \t\n", "CAFÉ Café",
              "x", "X x X", "end."]


def ref(texts, stop=(), max_df=0.5):
    return O.ref_vectorize(texts, stop, max_df)


def assert_same(g, r):
    m = g.matrix
    assert g.vocab == r["vocab"]
    assert np.array_equal(g.doc_freq, r["doc_freq"])
    assert g.n_docs == r["n_docs"]
    assert np.array_equal(g.kept_positions, r["kept"])
    assert np.array_equal(g.dropped_positions, r["dropped"])
    assert np.array_equal(m.indptr, r["indptr"])
    assert np.array_equal(m.indices, r["indices"])
    assert np.array_equal(m.values64.view(np.uint64), r["values"].view(np.uint64)), "weights not bitwise"
    assert m.dims == r["dims"] == len(g.vocab)


# ------------------------------------------------------------------ CPU ----
@pytest.mark.skipif(not O.ref_available(), reason="reference oracle not built")
def test_reference_kat_as_its_tests_state():
    """The shim drives the unmodified reference: its own test's expectations hold."""
    r = ref([t for _, t in KAT_DOCS], ["the", "of"], 1.0)
    assert list(r["dropped"]) == [1, 3]
    assert list(r["kept"]) == [0, 2, 4, 5]
    assert r["n_docs"] == 5
    assert r["vocab"][:2] == ["alpha", "beta"]


@pytest.mark.skipif(not O.ref_available(), reason="reference oracle not built")
def test_reference_matches_committed_golden():
    """Pins the oracle: the compiled reference reproduces the committed fixture
    (tests/golden/make_golden_vectorize.py)."""
    z = np.load(GOLDEN, allow_pickle=False)
    texts = textgen.corpus(int(z["n_docs"]), n_vocab=int(z["n_vocab"]), seed=int(z["seed"]))
    r = ref(texts, textgen.STOP, float(z["max_df"]))
    assert np.array_equal(r["indptr"], z["indptr"])
    assert np.array_equal(r["indices"], z["indices"])
    assert np.array_equal(r["values"].view(np.uint64), z["values"].view(np.uint64))
    assert np.array_equal(r["kept"], z["kept"]) and np.array_equal(r["dropped"], z["dropped"])
    assert np.array_equal(r["doc_freq"], z["doc_freq"])
    assert "\n".join(r["vocab"]) == str(z["vocab"])


def test_textgen_is_seeded():
    assert textgen.corpus(50, seed=3) == textgen.corpus(50, seed=3)


# ------------------------------------------------------------------ GPU ----
def gpu_vec(texts, stop=(), max_df=0.5, ids=None):
    from paper_2108_00895_b200 import vectorize_texts

    return vectorize_texts(texts, ids=ids, stop_words=stop, max_df=max_df)


@pytest.mark.gpu
def test_kat_drops_and_ids():
    from paper_2108_00895_b200 import vectorize_corpus

    m, vs, dropped = vectorize_corpus(KAT_DOCS, ["the", "of"], 1.0)
    assert dropped == ["d1", "d3"]
    assert m.n_docs == 4 and m.doc_ids == ["d0", "d2", "d4", "d5"]
    assert m.dims == vs
    for i in range(m.n_docs):
        assert abs(m.row(i).norm() - 1.0) <= 1e-9
    g = gpu_vec([t for _, t in KAT_DOCS], ["the", "of"], 1.0)
    assert g.n_docs == 5
    assert_same(g, ref([t for _, t in KAT_DOCS], ["the", "of"], 1.0))


@pytest.mark.gpu
def test_smoke_case():
    from paper_2108_00895_b200 import vectorize_corpus

    m, vs, dropped = vectorize_corpus(SMOKE_DOCS, stop_words=["the"], max_df=1.0)
    assert dropped == ["d3"] and m.n_docs == 3 and vs == 4 and m.doc_ids == ["d1", "d2", "d4"]
    assert_same(gpu_vec([t for _, t in SMOKE_DOCS], ["the"], 1.0), ref([t for _, t in SMOKE_DOCS], ["the"], 1.0))


@pytest.mark.gpu
@pytest.mark.parametrize("max_df", [1.0, 0.5, 0.3, 1e-3])
def test_edge_texts(max_df):
    texts = EDGE_TEXTS * 3 + ["shared"] * 2
    try:
        r = ref(texts, ["the"], max_df)
    except O.OracleError as e:
        with pytest.raises(RuntimeError, match=str(e)):
            gpu_vec(texts, ["the"], max_df)
        return
    assert_same(gpu_vec(texts, ["the"], max_df), r)


@pytest.mark.gpu
def test_errors_like_the_reference():
    with pytest.raises(RuntimeError, match="empty corpus"):
        gpu_vec([])
    with pytest.raises(RuntimeError, match="empty corpus"):
        gpu_vec(["the"], ["the", "of"], 1.0)  # test_corpus.cpp:175
    with pytest.raises(RuntimeError, match="empty corpus"):
        gpu_vec(["", " ,. "], [], 1.0)
    for bad in (0.0, 1.5, -1.0, float("nan")):
        with pytest.raises(ValueError, match=r"max_df_ratio must be in \(0, 1\]"):
            gpu_vec(["a b"], [], bad)
        with pytest.raises(ValueError):
            ref(["a b"], [], bad)
    with pytest.raises(RuntimeError, match="empty vocabulary"):
        gpu_vec(["a b", "a b"], [], 0.5)  # every term in every document: df/N = 1 > 0.5
    with pytest.raises(RuntimeError, match="empty corpus"):
        gpu_vec(["a b", "a b"], [], 1.0)  # idf 0: every row vectorises to zero
    with pytest.raises(O.OracleError, match="empty corpus"):
        ref(["a b", "a b"], [], 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed,max_df", [(300, 1, 1.0), (5000, 2, 0.5), (40000, 3, 0.2)])
def test_synthetic_texts_bitwise(n, seed, max_df):
    texts = textgen.corpus(n, n_vocab=20000, seed=seed)
    g = gpu_vec(texts, textgen.STOP, max_df)
    assert_same(g, ref(texts, textgen.STOP, max_df))
    assert g.stats["launches"] > 0


@pytest.mark.gpu
def test_golden_fixture():
    z = np.load(GOLDEN, allow_pickle=False)
    texts = textgen.corpus(int(z["n_docs"]), n_vocab=int(z["n_vocab"]), seed=int(z["seed"]))
    g = gpu_vec(texts, textgen.STOP, float(z["max_df"]))
    assert np.array_equal(g.matrix.indptr, z["indptr"])
    assert np.array_equal(g.matrix.values64.view(np.uint64), z["values"].view(np.uint64))
    assert "\n".join(g.vocab) == str(z["vocab"])


def gpu_normalize(ptr, idx, val):
    import ctypes as C

    from paper_2108_00895_b200 import _lib

    lib = _lib.load()
    optr = np.zeros_like(ptr)
    oidx = np.zeros(max(len(idx), 1), np.int32)
    oval = np.zeros(max(len(idx), 1), np.float64)
    _lib.check(lib.sskm_normalize_csr(0, len(ptr) - 1, ptr, idx.astype(np.int32), val, optr, oidx, oval))
    return optr, oidx[:optr[-1]], oval[:optr[-1]]


@pytest.mark.gpu
def test_normalize_rows_bitwise_including_long_orbits():
    """normalize (sparse_vector.cpp:158-209) on rows built to need the period-2
    rule and Brent's search (a weight orders of magnitude below its siblings),
    plus ±1 singletons, tiny and huge magnitudes."""
    rng = np.random.default_rng(7)
    rows = []
    for q in range(3000):
        n = int(rng.integers(1, 40))
        v = rng.lognormal(0, 1, n) * rng.choice([-1.0, 1.0], n)
        kind = q % 6
        if kind == 1 and n > 1:
            v[0] *= 1e-9  # slow drift through a finer ulp grid
        elif kind == 2:
            v *= 1e-200
        elif kind == 3:
            v *= 1e200
        elif kind == 4 and n > 2:
            v[1] = v[0]
        rows.append((np.sort(rng.choice(1 << 20, n, replace=False)).astype(np.int32), v))
    ptr = np.zeros(len(rows) + 1, np.int64)
    ptr[1:] = np.cumsum([len(r[0]) for r in rows])
    idx = np.concatenate([r[0] for r in rows])
    val = np.concatenate([r[1] for r in rows])
    optr, oidx, oval = gpu_normalize(ptr, idx, val)
    for r, (ri, rv) in enumerate(rows):
        ei, ev = O.normalize(ri.astype(np.uint32), rv.copy(), kind="ref")
        b, e = optr[r], optr[r + 1]
        assert np.array_equal(oidx[b:e], np.asarray(ei).astype(np.int32)), r
        assert np.array_equal(oval[b:e].view(np.uint64), np.asarray(ev, np.float64).view(np.uint64)), r
