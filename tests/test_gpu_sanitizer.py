"""compute-sanitizer over every kernel family (scripts/sanitize_run.py):
memcheck (out-of-bounds and misaligned accesses, leaks) and racecheck (shared
memory hazards; the screens' warp-private accumulators are updated with shared
atomics and read after __syncwarp)."""
import os
import shutil
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, f"--tool={tool}", "--error-exitcode=99", sys.executable, os.path.join(ROOT, "scripts", "sanitize_run.py")]
    if tool == "memcheck":
        cmd[1:1] = ["--leak-check=full"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr, tail
