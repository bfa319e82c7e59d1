"""compute-sanitizer racecheck / synccheck / memcheck over the fused ZipGEMM kernel (mbarrier
rings, hand-rolled stage hand-offs, named barriers, split-K fixup) and the decompress kernel,
on a small problem (tests/sanitize_target.py).  The tool must report 0 errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "memcheck"])
def test_sanitizer_clean(tool):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "99", "--kernel-name", "regex=zipgemm|decompress",
           sys.executable, os.path.join(HERE, "sanitize_target.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed" in out:
        # the GPU pool disables the tool (runs under it left GPUs needing a reset); the kernels'
        # own guards (mbarrier watchdogs, host-side shape / capacity checks) and the exact parity
        # tests are what remain
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert "sanitize target ok" in out, out[-4000:]
    # memcheck / synccheck print "ERROR SUMMARY: 0 errors", racecheck "RACECHECK SUMMARY: 0 hazards
    # displayed (0 errors, 0 warnings)"
    clean = "ERROR SUMMARY: 0 errors" in out or "(0 errors, 0 warnings)" in out
    assert r.returncode == 0 and clean, out[-4000:]
