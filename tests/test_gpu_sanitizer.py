"""compute-sanitizer over one forward + backward of a 2000-convex frame
(SURVEY.md 5): memcheck (out-of-bounds / misaligned accesses), synccheck
(barrier misuse) and initcheck (reads of uninitialised device memory) must
report no error.  racecheck is not run: it does not model the mbarrier
phase ordering of the blend kernels' producer/consumer ring (every shared
stage is written by the producer warp before its release arrive on `full`
and read by consumers after their acquire wait on it) and reports those
accesses as hazards; the protocol itself is exercised by every parity test
(a wait that stalls 2 s traps and fails the launch)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool,mode", [("memcheck", "depth"), ("synccheck", "depth"), ("initcheck", "depth"),
                                       ("memcheck", "depth2")])   # depth2: the float64-line kernels
def test_sanitizer_clean(tool, mode):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not available")
    out = subprocess.run([exe, "--tool", tool, "--error-exitcode", "9", sys.executable,
                          os.path.join(ROOT, "tools", "fwd_small.py"), "2000", "320", "200", mode],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, (out.stdout + out.stderr)[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out.stdout + out.stderr
