"""The C++ host API (include/sskm_b200.hpp) compiles against the C-ABI, keeps
the reference's exception types, and (on a GPU) runs the clustering."""
import os
import subprocess

import pytest

from paper_2108_00895_b200 import _build
from tests.conftest import ROOT, gpu_available

EXE = os.path.join(ROOT, "tests", "cpp", "run_example")


@pytest.fixture(scope="module")
def exe():
    _build.build()
    libdir = os.path.dirname(_build.LIB)
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp",
           "run_example.cpp"), "-o", EXE, "-L", libdir, "-l:libsskm_b200.so", f"-Wl,-rpath,{libdir}"]
    subprocess.run(cmd, check=True)
    return EXE


def test_invalid_config_throws_invalid_argument(exe):
    r = subprocess.run([exe, "validate"], capture_output=True, text=True)
    assert r.returncode == 2
    assert "k must be at least 2" in r.stdout


@pytest.mark.skipif(gpu_available(), reason="no-GPU failure path")
def test_no_gpu_is_runtime_error(exe):
    r = subprocess.run([exe, "run"], capture_output=True, text=True)
    assert r.returncode == 1 and "runtime_error" in r.stdout


@pytest.mark.gpu
def test_cpp_run_matches_python_api(exe):
    r = subprocess.run([exe, "run", "4"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "stop=no_reassignments" in r.stdout
    assert "a0=0 a1=1 a2=2 a3=3" in r.stdout  # 4 orthogonal groups, seeds 0..3 one per group


@pytest.mark.gpu
def test_cpp_multi_device_run_equals_single(exe):
    """RunConfig::devices (sskm_cluster_csr_multi): the same result line."""
    one = subprocess.run([exe, "run", "4"], capture_output=True, text=True)
    two = subprocess.run([exe, "multi", "4"], capture_output=True, text=True)
    assert two.returncode == 0, two.stdout + two.stderr
    assert two.stdout == one.stdout
