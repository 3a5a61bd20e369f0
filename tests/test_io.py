"""CPU: corpus IO and the run report against the reference's own
load_matrix / write_matrix / to_json (oracle/_ref, compiled from corpus.cpp and
report.cpp)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2108_00895_b200 import io as IO
from paper_2108_00895_b200 import synthetic as S
from paper_2108_00895_b200.api import ClusteringResult, IterationStats

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref_corpus():
    ptr, idx, val, dims = O.reference_synthetic_zipf(300, 800, 8.0, 1.1, 3)
    return O.Corpus(ptr, idx, val, dims)


def test_load_reference_written_matrix(tmp_path, ref_corpus):
    path = str(tmp_path / "m.mtx")
    O.ref_write_matrix(path, ref_corpus)
    m = IO.load_matrix(path, keep_f64=True)
    assert m.n_docs == ref_corpus.n and m.dims == ref_corpus.dims
    np.testing.assert_array_equal(m.indptr, ref_corpus.indptr)
    np.testing.assert_array_equal(m.indices, ref_corpus.indices)
    np.testing.assert_array_equal(m.values_f64, ref_corpus.values)  # %.17g round-trips bitwise
    np.testing.assert_array_equal(m.values, ref_corpus.values.astype(np.float32))
    assert m.doc_ids == [str(i) for i in range(ref_corpus.n)]


def test_write_then_reference_load(tmp_path):
    m = S.generate(200, 500, 4, 10.0, seed=2)
    path = str(tmp_path / "ours.mtx")
    IO.write_matrix(path, m)
    # fp32-valued rows are ~1e-8 off unit length: the reference's 1e-9 check rejects them
    # (corpus.cpp:256-262, SURVEY finding 5) ...
    with pytest.raises(O.OracleError, match="is not unit length"):
        O.ref_load_matrix(path)
    with pytest.raises(RuntimeError, match="is not unit length"):
        IO.load_matrix(path)
    # ... and both read them with the values bit-exact when the tolerance allows fp32 rows
    back = IO.load_matrix(path, norm_tol=1e-6)
    np.testing.assert_array_equal(back.indptr, m.indptr)
    np.testing.assert_array_equal(back.indices, m.indices)
    np.testing.assert_array_equal(back.values, m.values)


@pytest.mark.parametrize("body,what", [
    ("%%sparse-unit-matrix 2 5\n", "bad header"),
    ("%%sparse-unit-matrix 2 5 2\n1 0 1\n0 1 1\n", "rows out of order"),
    ("%%sparse-unit-matrix 2 5 3\n0 3 0.6\n0 1 0.8\n1 0 1\n", "dims out of order within row"),
    ("%%sparse-unit-matrix 2 5 2\n0 0 0\n1 0 1\n", "zero weight"),
    ("%%sparse-unit-matrix 2 5 2\n0 7 1\n1 0 1\n", "dim index out of bounds"),
    ("%%sparse-unit-matrix 2 5 2\n3 0 1\n1 0 1\n", "row index out of bounds"),
    ("%%sparse-unit-matrix 2 5 2\n0 0 1\nbad line\n", "expected '<row> <dim> <weight>'"),
    ("%%sparse-unit-matrix 2 5 3\n0 0 1\n1 0 1\n", "header declares 3 entries but file has 2"),
    ("%%sparse-unit-matrix 2 5 2\n0 0 0.5\n1 0 1\n", "row 0 is not unit length"),
])
def test_errors_match_reference(tmp_path, body, what):
    path = str(tmp_path / "bad.mtx")
    with open(path, "w") as f:
        f.write(body)
    with open(path + ".ids", "w") as f:
        f.write("a\nb\n")
    with pytest.raises(O.OracleError) as ref:
        O.ref_load_matrix(path)
    with pytest.raises(RuntimeError) as ours:
        IO.load_matrix(path)
    assert what in str(ref.value)
    assert str(ours.value) == str(ref.value)


def test_binary_csr_roundtrip(tmp_path):
    m = S.generate(500, 1000, 6, 20.0, seed=5)
    path = str(tmp_path / "m.sskmb")
    IO.save_csr(path, m)
    back = IO.load_csr(path)
    assert back.dims == m.dims
    for a, b in [(back.indptr, m.indptr), (back.indices, m.indices), (back.values, m.values)]:
        np.testing.assert_array_equal(a, b)
    with open(path, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(ValueError, match="not an SSKMCSR1 file"):
        IO.load_csr(path)


def test_report_json_matches_reference(ref_corpus):
    r = O.run_seeded(ref_corpus, 6, [0, 10, 20, 30, 40, 50], mode="ncc", kind="port")
    its = [IterationStats(**{k: v for k, v in it.items() if k in IterationStats.__dataclass_fields__})
           for it in r["iterations"]]
    res = ClusteringResult(assignments=r["assignments"], sims=r["sims"], iterations=its,
                           objective=r["objective"], stop_reason=r["stop_reason"], extra={"k": 6})
    cfg = dict(k=6, mode="ncc", seed=3, max_iters=100)

    class D:
        n_docs, dims = ref_corpus.n, ref_corpus.dims

    ours = IO.to_json(IO.make_report(cfg, D, res))
    ref = O.ref_report_json(cfg, ref_corpus.n, ref_corpus.dims, r["iterations"], r["objective"], r["stop_reason"],
                            r["assignments"])
    assert ours == ref
