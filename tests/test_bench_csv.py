"""The GPU bench CSV keeps the reference CLI's columns and statistics
(cmd_bench, sskm_main.cpp:180-262) and appends the B200 columns."""
import numpy as np
import pytest

from paper_2108_00895_b200 import bench_csv as B


def test_header_and_format():
    rows = [{"mode": "ncc+index", "k": 10, "median_seconds": 0.5, "iqr_seconds": 0.25, "dot_products": 12345,
             "iterations": 7, "index_build_seconds": 0.001, "comparisons_per_s": 1.5e9, "exact_dots": 99,
             "screen_gbs": 1234.5, "roofline_frac": 0.19}]
    text = B.to_csv(rows)
    head, line = text.splitlines()
    assert head.startswith("mode,k,median_seconds,iqr_seconds,dot_products,iterations,index_build_seconds,")
    assert line.startswith("ncc+index,10,0.500000,0.250000,12345,7,0.001000,")


def test_median_is_the_references():
    assert B._median([3.0, 1.0, 2.0]) == 2.0
    assert B._median([4.0, 1.0, 2.0, 3.0]) == 2.5
    with pytest.raises(ValueError):
        B.bench_rows(None, [2], ["baseline"], repeats=0)


@pytest.mark.gpu
def test_gpu_bench_counts_equal_the_references_run():
    from oracle import oracle as O
    from paper_2108_00895_b200 import synthetic as S

    if not O.ref_available():
        pytest.skip("compiled reference not present")
    m = S.generate(600, 1024, 6, 30.0, seed=4)
    rows = B.bench_rows(m, [8], ["baseline", "ncc"], repeats=2, seed=7)
    c = O.Corpus(m.indptr, m.indices, m.values.astype(np.float64), m.dims)
    for r in rows:
        ref = O.run_kmeanspp(c, 8, mode=r["mode"], seed=7)
        assert r["iterations"] == len(ref["iterations"])
        assert r["dot_products"] == sum(it["dot_products"] for it in ref["iterations"])
        assert r["median_seconds"] > 0 and r["comparisons_per_s"] > 0
