"""The drop-in boundary, proven from the reference's side: the UNMODIFIED
reference package (baseline/_ref) runs its OWN tests with its numba
integrate / raycast / extraction kernels replaced by libtfb200 through the
C ABI (integration/tilefusion_kernels_b200.py):
test_tsdf.py in full, and acceptance gates 1 (tiled pipeline == single
volume, test_acceptance.py:58-79) and 8 (structural invariants end to end:
order-free merge, bitwise determinism, :323-396).  The shim reports how
often each B200 kernel ran, so a silent fallback to numba cannot pass.

Needs baseline/_ref and baseline/_ref_tests (tools/install_reference.sh; both
git-ignored, they travel to the GPU box with the repository)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
REF_TESTS = ROOT / "baseline" / "_ref_tests"

pytestmark = pytest.mark.gpu


def _run(tmp_path, targets, select=None):
    if not (REF / "tilefusion").exists() or not REF_TESTS.exists():
        pytest.skip("reference not installed (tools/install_reference.sh)")
    report = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT / "integration"), str(ROOT)])
    env["NUMBA_CACHE_DIR"] = str(tmp_path / "numba")
    env["TFB200_SHIM_REPORT"] = str(report)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "pytest_b200_shim", "-p", "no:cacheprovider",
           "-o", "addopts=", "--rootdir", str(REF_TESTS), *[str(REF_TESTS / t) for t in targets]]
    if select:
        cmd += ["-k", select]
    r = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    return json.loads(report.read_text()), r.stdout


def test_reference_tsdf_suite_through_the_c_abi(tmp_path):
    calls, out = _run(tmp_path, ["test_tsdf.py"])
    assert "passed" in out and "failed" not in out
    assert calls["integrate_kernel"] >= 5 and calls["raycast_kernel"] >= 4
    assert calls["extract_bound"] >= 2 and calls["extract_kernel"] >= 2


def test_reference_acceptance_gates_1_and_8_through_the_c_abi(tmp_path):
    calls, out = _run(tmp_path, ["test_acceptance.py"],
                      "test_tiled_pipeline_matches_single_volume or "
                      "test_structural_invariants_hold_end_to_end")
    assert "2 passed" in out
    assert calls["integrate_kernel"] > 100 and calls["raycast_kernel"] > 100
