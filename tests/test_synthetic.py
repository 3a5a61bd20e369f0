"""CPU: the BASELINE corpus generator is deterministic (any thread count),
produces valid unit-length CSR rows, and matches the realized shapes SURVEY
§8d measured for its generator description."""
import numpy as np
import pytest

from paper_2108_00895_b200 import synthetic as S


def test_deterministic_across_threads():
    a = S.generate(3000, 4096, 20, 60.0, seed=3, threads=1)
    b = S.generate(3000, 4096, 20, 60.0, seed=3, threads=7)
    assert np.array_equal(a.indptr, b.indptr)
    assert np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.values, b.values)
    c = S.generate(3000, 4096, 20, 60.0, seed=4, threads=2)
    assert not np.array_equal(a.indices[:100], c.indices[:100])


def test_rows_are_valid_unit_vectors():
    m = S.generate(2000, 5000, 10, 40.0, sigma=0.7, seed=9)  # non power-of-two vocab
    assert m.indices.min() >= 0 and m.indices.max() < 5000
    for i in range(0, m.n_docs, 97):
        b, e = m.indptr[i], m.indptr[i + 1]
        assert e > b
        assert np.all(np.diff(m.indices[b:e]) > 0)
        assert np.all(m.values[b:e] > 0)
        assert abs(np.sum(m.values[b:e].astype(np.float64) ** 2) - 1.0) < 1e-6


def test_c0_shape_matches_survey():
    m = S.corpus("c0")
    assert m.n_docs == 20_000 and m.dims == 16_384
    lens = np.diff(m.indptr)
    # c0 distinct nnz/doc mean 40.8 (p50 37, p99 96)
    assert 38 < lens.mean() < 44
    assert 34 <= np.percentile(lens, 50) <= 41
    assert 85 <= np.percentile(lens, 99) <= 110


def test_init_seeds_distinct_and_pinned():
    s = S.init_seeds(20_000, 100, 0)
    assert len(set(s.tolist())) == 100
    assert np.array_equal(s, np.random.default_rng(0).choice(20_000, 100, replace=False))
