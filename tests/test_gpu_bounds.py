"""Memory checking without compute-sanitizer (closed on the GPU pool): the
bounds-checked build of the library (libtfb200_checked.so, -DTF_BOUNDS_CHECK:
every guarded voxel / pixel / table / slot index is checked, a violation is
counted and the access skipped instead of faulting) runs a workload covering
every kernel family — integration (screened, exact, no-cull, colour, split),
raycast (per-lane, cooperative, exact), merges, extraction, the endpoint
histogram, ICP, the peer-memory reduction with emulated ranks — plus one
config-3 frame (8 x 512^3), and must count zero violations."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_1511_07106_b200" / "libtfb200_checked.so"

pytestmark = pytest.mark.gpu


def test_bounds_checked_build_counts_no_violation():
    from paper_1511_07106_b200 import build
    build.build(checked=True)  # (re)built when a source is newer than it
    env = dict(os.environ, TFB200_LIB=str(CHECKED))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_small.py"), "--big"], env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 bounds violations" in r.stdout
