"""compute-sanitizer (memcheck, racecheck, synccheck) over a small pass of
every kernel family (tools/sanitize_driver.py): SURVEY §5 race detection."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool, dev):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not available")
    out = subprocess.run([exe, "--tool", tool, "--error-exitcode", "9", sys.executable,
                          os.path.join(ROOT, "tools", "sanitize_driver.py")], cwd=ROOT, capture_output=True,
                         text=True, timeout=1200)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]
    assert "sanitize driver done" in out.stdout
