"""compute-sanitizer over tiny launches of every kernel family and
instantiation class (tools/run_small.py: 1-D/2-D/3-D, fp16/bf16 (both variants)/fp32, D 16-128, small-tile forward, strided layouts,
tensor-core and CUDA-core paths): memcheck (out-of-bounds / misaligned
accesses), racecheck (shared-memory hazards across the hand-written mbarrier
and TMEM pipelines), synccheck (illegal barrier use) and initcheck (reads of
uninitialised device memory)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not found")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "17", sys.executable,
                        os.path.join(ROOT, "tools", "run_small.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    if r.returncode != 0 and "closed on this pool" in out:
        # the GPU pool's wrapper refuses sanitizer runs; the last clean run on
        # this pool is recorded in profiles/r02_sanitizers_v2.md
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0, out[-4000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, out[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
