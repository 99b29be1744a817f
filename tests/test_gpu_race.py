"""compute-sanitizer on the fast engine: racecheck
and synccheck report no hazard on the shipped kernels, and racecheck DOES
flag the broken-barrier negative control (WL_BREAK_BARRIER=1), mirroring
the reference's acceptance criterion 6 (acceptance.cpp:283-296)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
PKG = os.path.join(ROOT, "paper_1605_00561_b200")


def sanitize(tool, lib):
    env = dict(os.environ, WL_LIB=lib)
    r = subprocess.run([SAN, "--tool", tool, sys.executable,
                        os.path.join(ROOT, "tools", "race_workload.py")],
                       capture_output=True, text=True, env=env, timeout=600)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (the pool
        # operators closed it); the committed sanitizer logs of earlier runs
        # stay the evidence (profiles/, DESIGN.md f3)
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip()[:120])
    return r.returncode, out


def hazards(out):
    m = re.search(r"RACECHECK SUMMARY: (\d+) hazard", out)
    return int(m.group(1)) if m else (0 if "0 errors" in out else -1)


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not available")
def test_racecheck_and_synccheck_clean():
    lib = os.path.join(PKG, "libwavelift_b200.so")
    rc, out = sanitize("racecheck", lib)
    assert "workload done" in out and rc == 0, out[-2000:]
    assert hazards(out) == 0, out[-2000:]
    rc, out = sanitize("synccheck", lib)
    assert "workload done" in out and rc == 0 and "ERROR SUMMARY: 0 errors" in out, out[-2000:]


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not available")
def test_racecheck_flags_broken_barrier():
    lib = os.path.join(PKG, "libwavelift_b200_brk1.so")
    if not os.path.exists(lib):
        env = dict(os.environ, WL_VARIANT="brk1", WL_DEFS="-DWL_BREAK_BARRIER=1")
        subprocess.run([sys.executable, "-m", "paper_1605_00561_b200._build"], cwd=ROOT,
                       env=env, check=True, capture_output=True)
    rc, out = sanitize("racecheck", lib)
    assert "workload done" in out, out[-2000:]
    assert hazards(out) > 0, out[-2000:]
