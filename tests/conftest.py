"""Shared fixtures.  `-m gpu` tests need a B200 (they run through libtfb200);
everything else runs on the CPU (oracle vs golden vectors, host logic, ABI
surface, gloo multi-process logic)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtfb200.so")
    config.addinivalue_line("markers", "reference: needs the reference package at /root/reference")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture
def small_intr():
    from paper_1511_07106_b200 import CameraIntrinsics
    return CameraIntrinsics(fx=100.0, fy=100.0, cx=40.0, cy=30.0, width=80, height=60)


@pytest.fixture
def anchored_scene():
    from paper_1511_07106_b200.synth import demo_scene
    return demo_scene()


def reference_module():
    """Import the reference package (build container only) or skip."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference package not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    try:
        import tilefusion  # noqa: F401
    except Exception as exc:  # numba missing etc.
        pytest.skip(f"reference not importable: {exc}")
    import tilefusion
    return tilefusion
