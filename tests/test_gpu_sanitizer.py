"""compute-sanitizer memcheck and synccheck over the operator kernels and the
SSB SF=1 suite (tools/sanitize_workload.py checks every result itself), as
SURVEY section 5 asks.  racecheck is recorded in profiles/r02_sanitizer.txt:
it cannot order cp.async.bulk (async-proxy) writes through mbarrier
complete_tx, so every TMA ring reports false WAR hazards.

Opt-in (CRYS_SANITIZE=1): the GPU pool this build is measured on has closed
compute-sanitizer (its wrapper exits 86 without running the tool, as runs
under it left GPUs needing a reset), so by default these tests skip; the
committed runs are profiles/r02_sanitizer.txt."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,parts", [("memcheck", "select,join,sort,block,project"),
                                        ("memcheck", "ssb"),
                                        ("synccheck", "select,join,sort,block,ssb")])
def test_sanitizer_clean(tool, parts):
    if os.environ.get("CRYS_SANITIZE") != "1":
        pytest.skip("opt-in: CRYS_SANITIZE=1 (compute-sanitizer is closed on the measurement pool)")
    if not os.path.exists(SANITIZER):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, CRYS_GRAPHS="0")
    r = subprocess.run([SANITIZER, "--tool", tool, "--error-exitcode", "17", "--print-limit", "20",
                        sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py"), parts],
                       env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "closed" in out:
        pytest.skip("compute-sanitizer closed on this pool: " + out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-4000:]
    assert "workload ok" in out and "ERROR SUMMARY: 0 errors" in out, out[-4000:]
