"""compute-sanitizer memcheck over tiny launches of every kernel family."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck"])
def test_sanitizer_clean(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not found")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "17", sys.executable,
                        os.path.join(ROOT, "tools", "run_small.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
