"""BASELINE.json synthetic corpora — benchmark and test INPUT, not the product.

The seeded generator (synth.cpp, pinned in its header and DESIGN.md §7) is its
own small C++ library, libsskm_synth.so, built with g++ and loaded here with
ctypes, so that both arms of bench.py (ours and the reference's) can build the
same corpus without loading anything of the other arm: the reference arm
imports this module and oracle/ only. These corpora stand in for the paper's
private datasets (BASELINE.json names no public one).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "synth.cpp")
LIB = os.path.join(HERE, "libsskm_synth.so")


@dataclass(frozen=True)
class CorpusConfig:
    name: str
    n_docs: int
    dims: int
    k_true: int
    mean_len: float
    sigma: float
    k: int
    iterations: int
    zipf_s: float = 1.1
    seed: int = 0


# BASELINE.json "configs"
CONFIGS = {
    "c0": CorpusConfig("c0", 20_000, 16_384, 50, 60.0, 0.5, 100, 20),
    "c1": CorpusConfig("c1", 1_000_000, 262_144, 500, 100.0, 0.5, 1_000, 30),
    "c2": CorpusConfig("c2", 4_000_000, 262_144, 5_000, 100.0, 0.5, 10_000, 30),
    "c3": CorpusConfig("c3", 500_000, 131_072, 200, 1_500.0, 0.7, 2_000, 20),
    "c4": CorpusConfig("c4", 16_000_000, 131_072, 20_000, 80.0, 0.5, 50_000, 25),
}


@dataclass
class CSR:
    """Plain CSR arrays (int64 indptr, int32 sorted indices, fp32 values)."""
    indptr: np.ndarray
    indices: np.ndarray
    values: np.ndarray
    dims: int
    dropped: int = 0

    @property
    def n_docs(self) -> int:
        return len(self.indptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["g++", "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", "-o", LIB + ".tmp", SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("g++ failed building libsskm_synth.so:\n" + r.stderr)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(LIB)
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        lib.sskm_synth_last_error.restype = C.c_char_p
        lib.sskm_synth_generate.restype = C.c_void_p
        lib.sskm_synth_generate.argtypes = [C.c_int64, C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                            C.c_double, C.c_uint64, C.c_int]
        lib.sskm_synth_sizes.restype = None
        lib.sskm_synth_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_uint32), C.POINTER(C.c_int64)]
        lib.sskm_synth_export.restype = None
        lib.sskm_synth_export.argtypes = [C.c_void_p, i64p, i32p, f32p]
        lib.sskm_synth_free.restype = None
        lib.sskm_synth_free.argtypes = [C.c_void_p]
        _lib = lib
    return _lib


def generate(n_docs: int, dims: int, k_true: int, mean_len: float, sigma: float = 0.5,
             zipf_s: float = 1.1, seed: int = 0, threads: int = 0) -> CSR:
    lib = _load()
    h = lib.sskm_synth_generate(int(n_docs), int(dims), int(k_true), float(mean_len), float(sigma),
                                float(zipf_s), int(seed), int(threads))
    if not h:
        raise ValueError(lib.sskm_synth_last_error().decode())
    try:
        n, nnz, d, dropped = C.c_int64(), C.c_int64(), C.c_uint32(), C.c_int64()
        lib.sskm_synth_sizes(h, C.byref(n), C.byref(nnz), C.byref(d), C.byref(dropped))
        indptr = np.zeros(n.value + 1, np.int64)
        idx = np.zeros(max(nnz.value, 1), np.int32)
        val = np.zeros(max(nnz.value, 1), np.float32)
        lib.sskm_synth_export(h, indptr, idx, val)
    finally:
        lib.sskm_synth_free(h)
    return CSR(indptr, idx[: nnz.value], val[: nnz.value], int(d.value), int(dropped.value))


def corpus(cfg: "CorpusConfig | str", threads: int = 0, n_docs: int | None = None) -> CSR:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return generate(n_docs or cfg.n_docs, cfg.dims, cfg.k_true, cfg.mean_len, cfg.sigma, cfg.zipf_s,
                    cfg.seed, threads)


def init_seeds(n_docs: int, k: int, seed: int = 0) -> np.ndarray:
    """k distinct documents from seed 0, order = cluster ids:
    numpy.random.default_rng(seed).choice(n_docs, k, replace=False)."""
    return np.random.default_rng(seed).choice(n_docs, k, replace=False).astype(np.uint32)
