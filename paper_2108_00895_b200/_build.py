"""In-tree build of the native library (sm_100a only).

`python -m paper_2108_00895_b200._build` compiles csrc/ into
paper_2108_00895_b200/libsskm_b200.so with nvcc (cross-compiles without a GPU).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsskm_b200.so")
SOURCES = ["engine.cu", "vectorize.cu", "io.cpp"]
DEPS = SOURCES + sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp")))
HEADER = os.path.join(os.path.dirname(PKG), "include", "sskm_b200.h")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-fopenmp",
    "-Xptxas", "-v",
] + [f for f in os.environ.get("SSKM_NVCC_EXTRA", "").split() if f]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-lgomp"]
OBJ = os.path.join(PKG, "build")  # objects (git-ignored): one per source, rebuilt when it or a header changed
# headers each source includes (a source is recompiled only when one of its own changed)
SRC_DEPS = {
    "engine.cu": [f for f in DEPS if f.endswith(".cuh")],
    "vectorize.cu": ["common.cuh"],
    "io.cpp": [],
}


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [HEADER]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src: str) -> str:
        obj = os.path.join(OBJ, src + ".o")
        deps = [os.path.join(CSRC, src), HEADER] + [os.path.join(CSRC, h) for h in SRC_DEPS.get(src, [])]
        if not force and os.path.exists(obj) and all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in deps):
            return obj
        r = subprocess.run([_nvcc(), *NVCC_FLAGS, "-c", "-o", obj, os.path.join(CSRC, src)], capture_output=True,
                           text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed compiling {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    r = subprocess.run([_nvcc(), *LINK_FLAGS, "-o", LIB + ".tmp", *objs], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libsskm_b200.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
