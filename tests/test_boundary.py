"""CPU: the C-ABI library loads, exports every symbol the headers declare, and
fails loudly (no CPU fallback) when no GPU is present. Config validation runs
host-side and matches the reference's messages (engine.cpp:47-64)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import _build, _lib
from tests.conftest import ROOT, gpu_available


def header_symbols():
    syms = set()
    for h in ["sskm_b200.h", "sskm_io.h"]:
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        syms |= set(re.findall(r"\b(sskm_[a-z0-9_]+)\s*\(", src))
    return syms


def test_library_built_for_sm100a_only():
    assert os.path.exists(_build.LIB)
    assert "arch=compute_100a,code=sm_100a" in " ".join(_build.NVCC_FLAGS)


def test_exports_every_header_symbol():
    lib = C.CDLL(_lib.lib_path())
    missing = [s for s in sorted(header_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _lib.SIGNATURES}
    from paper_2108_00895_b200 import io as IO

    IO._io()
    io_bound = {s for s in header_symbols() if s.startswith("sskm_io_") and getattr(lib, s, None) is not None}
    assert header_symbols() <= bound | io_bound, header_symbols() - bound - io_bound


def test_validate_matches_reference_messages():
    P.validate(10, 3)
    with pytest.raises(ValueError, match="k must be at least 2"):
        P.validate(10, 1)
    with pytest.raises(ValueError, match=r"k \(11\) exceeds the number of documents \(10\)"):
        P.validate(10, 11)
    with pytest.raises(ValueError, match="lambdas must be strictly ascending"):
        P.validate(10, 3, lambdas=(0.4, 0.2))
    with pytest.raises(ValueError, match=r"lambda must be in \(0, 1\)"):
        P.validate(10, 3, lambdas=(0.0, 0.4))
    with pytest.raises(ValueError, match="conv_sq_dist must be positive"):
        P.validate(10, 3, conv_sq_dist=0.0)
    with pytest.raises(ValueError, match="ncc_epsilon must be nonnegative"):
        P.validate(10, 3, ncc_epsilon=-1.0)
    with pytest.raises(ValueError, match="max_iters must be at least 1"):
        P.validate(10, 3, max_iters=0)
    with pytest.raises(ValueError, match="unknown mode"):
        P.validate(10, 3, mode="nope")


def test_cluster_bad_arguments_raise_value_error_before_touching_the_gpu():
    # test_smoke.py:104-111
    from paper_2108_00895_b200 import synthetic as S

    data = S.generate(20, 50, 2, 5.0, seed=1)
    with pytest.raises(ValueError):
        P.cluster(data, k=0)
    with pytest.raises(ValueError):
        P.cluster(data, k=30)
    with pytest.raises(ValueError):
        P.cluster(data, k=3, mode="nope")


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(RuntimeError):
        P.Engine(0)
    from paper_2108_00895_b200 import synthetic as S

    data = S.generate(50, 64, 2, 5.0, seed=1)
    with pytest.raises(RuntimeError):
        P.cluster(data, k=3, init_seeds=[0, 1, 2])


def test_corpus_matrix_api():
    m = P.CorpusMatrix.from_csr([0, 2, 3], [3, 7, 1], [0.6, 0.8, 1.0], 10)
    assert m.n_docs == 2 and m.dims == 10 and m.nnz == 3
    assert m.row(0).entries() == [(3, pytest.approx(0.6)), (7, pytest.approx(0.8))]
    assert m.row(0).norm() == pytest.approx(1.0, abs=1e-7)
    with pytest.raises(ValueError):
        P.CorpusMatrix.from_csr([0, 2], [1], [1.0], 4)
