"""compute-sanitizer over every engine kernel: out-of-bounds and
misaligned accesses (memcheck), shared-memory hazards between the warps of
the compute_Y groups and the reduction buffers (racecheck), barrier misuse
of the named per-group barriers (synccheck), and reads of uninitialised
device memory (initcheck), on small problems (tools/sanitize_step.py:
2J = 5, 8, 14; staged and graph runs, descriptors, virial, device neighbor
lists, the one-call path)."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    cmd = [cs, "--tool", tool, "--error-exitcode", "9"]
    if tool == "memcheck":
        cmd += ["--leak-check", "full"]
    out = subprocess.run(cmd + ["python", "tools/sanitize_step.py"], cwd=ROOT,
                         capture_output=True, text=True, timeout=1800)
    tail = (out.stdout + out.stderr)[-4000:]
    assert out.returncode == 0, tail
    assert "sanitize_step: done" in out.stdout, tail
    text = out.stdout + out.stderr
    # memcheck / synccheck / initcheck: "ERROR SUMMARY: 0 errors";
    # racecheck: "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    assert "ERROR SUMMARY: 0 errors" in text or "SUMMARY: 0 hazards displayed (0 errors" in text, tail
