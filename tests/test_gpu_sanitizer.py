"""compute-sanitizer memcheck and synccheck over one small call of every
kernel path (scripts/sanitize.py): no errors, and every option still gives
the default path's bits under the tool."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_kernels_clean_under_compute_sanitizer(tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    proc = subprocess.run([exe, "--tool", tool, "--error-exitcode", "3", sys.executable,
                           os.path.join(ROOT, "scripts", "sanitize.py")],
                          capture_output=True, text=True, timeout=600)
    out = proc.stdout + proc.stderr
    assert proc.returncode == 0, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
    assert "ALL_EQUAL True" in out, out[-3000:]
