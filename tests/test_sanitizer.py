"""compute-sanitizer memcheck / racecheck / synccheck over one small run of
every kernel (decode, both GEMVs, tcgen05 GEMM, grouped experts, split paths),
SURVEY.md §5 "race detection".  GPU only."""
import os
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(cuda, tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    if os.environ.get("CCQ_RUN_SANITIZER") != "1":
        # The GPU pool this suite runs on has closed compute-sanitizer (its
        # wrapper refuses with exit code 86); the committed run is
        # profiles/r02_compute_sanitizer.txt.  Opt in where it is allowed.
        pytest.skip("compute-sanitizer is opt-in (CCQ_RUN_SANITIZER=1)")
    out = subprocess.run([exe, "--tool", tool, "--error-exitcode", "3", sys.executable,
                          os.path.join(ROOT, "tools", "sanitize_case.py")],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    text = out.stdout + out.stderr
    if out.returncode == 86 and "closed" in text:
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert out.returncode == 0, text[-4000:]
    assert "sanitize case ok" in text
