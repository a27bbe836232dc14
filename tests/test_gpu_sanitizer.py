"""compute-sanitizer memcheck over the tiny case of every kernel family (memcheck / racecheck /
synccheck / initcheck on tiny and ragged configs).  The full four-tool sweep over scripts/sanitize_case.py is
recorded in profiles/r02_sanitizer.md; this test keeps memcheck in the GPU suite."""
import os
import shutil
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    return None


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
def test_memcheck_tiny_all_kernel_families():
    cs = _sanitizer()
    if cs is None:
        pytest.skip("compute-sanitizer not installed")
    cmd = [cs, "--tool", "memcheck", "--error-exitcode", "17", "--print-limit", "20", sys.executable,
           os.path.join(ROOT, "scripts", "sanitize_case.py"), "tiny"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = p.stdout + p.stderr
    if "closed on this pool" in out:
        # the GPU pool's wrapper refuses compute-sanitizer (earlier runs under it left GPUs needing a reset); the
        # four-tool sweep run while it was open is recorded in profiles/r02_sanitizer.md
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert p.returncode == 0, out[-4000:]
    assert "SANITIZE_CASE_DONE" in out, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
