"""compute-sanitizer racecheck / synccheck / memcheck on the hot path (SURVEY 4 tier 4): the in-place
RBGS colour passes (which must read only the other colour across CTAs), the row kernels'
warp shuffles, the dense coarse cycle's and the tile-layout sub-cycle's CTA barriers, and the
apply's block reduction, on small adaptive trees with T-junctions and cut cells.

The GPU pool has since closed compute-sanitizer (its wrapper refuses with exit code 86: runs under
it left GPUs needing a reset), so these runs are opt-in (OCTMG_RUN_SANITIZER=1, only where the
tool is allowed); the clean round-2 run is committed as profiles/r02_sanitizer.log."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "memcheck"])
@pytest.mark.parametrize("case", [("tank_small",), ("sphere_small",), ("sphere_small", "OCTMG_COARSE_DENSE=0"),
                                  ("sphere_35", "OCTMG_PASS_GHOST=call")])
@pytest.mark.skipif(os.environ.get("OCTMG_RUN_SANITIZER") != "1",
                    reason="compute-sanitizer is closed on the GPU pool; opt in with OCTMG_RUN_SANITIZER=1")
def test_sanitizer_clean(tool, case):
    assert os.path.exists(SAN), "compute-sanitizer not found"
    env = dict(os.environ, OCTMG_GRAPH_LOOP="0")
    p = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "17", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_case.py"), *case],
                       capture_output=True, text=True, timeout=1200, env=env)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-3000:]
    assert "ok" in p.stdout
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
