"""The C-ABI library without a GPU: it builds for sm_100a, loads, exports
every entry point include/tfb200.h declares, and rejects bad arguments
through its return codes without touching a device."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_1511_07106_b200 import _native as nat

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tfb200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for required in ("tf_integrate", "tf_raycast", "tf_icp_reduce", "tf_vertex_normal_map",
                     "tf_raymap_merge", "tf_extract_count", "tf_extract_emit",
                     "tf_endpoint_cells", "tf_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = nat.load_library()
    out = subprocess.run(["nm", "-D", "--defined-only", str(nat.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (tf_[a-z0-9_]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    for n in declared_functions():
        assert hasattr(lib, n)
    assert set(nat.EXPORTED) <= exported


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(nat.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_errors_without_gpu():
    lib = nat.load_library()
    assert lib.tf_abi_version() == nat.ABI_VERSION
    cam = nat.TfCamera(100.0, 100.0, 40.0, 30.0, 80, 60)
    rc = lib.tf_integrate(None, 1, None, ctypes.byref(cam), None, None, None, 0.1, 128.0, 1.0,
                          None, 0, None, None)
    assert rc == -1
    assert b"null argument" in lib.tf_last_error()
    rc = lib.tf_raycast(None, 1, ctypes.byref(cam), 0.1, 0, None, None, None, None, None, None,
                        None)
    assert rc == -1


def test_workspace_sizes_are_host_computable():
    lib = nat.load_library()
    vols = (nat.TfVolume * 2)()
    for v in vols:
        v.n = 256
        v.voxel_size = 0.01
    cam = nat.TfCamera(525.0, 525.0, 319.5, 239.5, 640, 480)
    need = lib.tf_integrate_workspace_size(vols, 2, ctypes.byref(cam))
    # pixel table (16 B/px) + two 32^3-brick lists + mip
    assert need >= 640 * 480 * 16 + 2 * 32 ** 3 * 4
    assert lib.tf_icp_workspace_size(640 * 480) == (640 * 480 // 256) * 29 * 8
    assert lib.tf_extract_workspace_size(64) >= (64 ** 3 // 256) * 8


def test_debug_flags_roundtrip():
    lib = nat.load_library()
    lib.tf_set_debug_flags(nat.DEBUG_NO_CULL)
    assert lib.tf_debug_flags() == nat.DEBUG_NO_CULL
    lib.tf_set_debug_flags(0)
    assert lib.tf_debug_flags() == 0


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """Without a CUDA device the operators raise instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1511_07106_b200 import TsdfSubvolume
    with pytest.raises(RuntimeError, match="CUDA"):
        TsdfSubvolume.empty([0, 0, 0], 8, 0.8)


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_1511_07106_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "import oracle" not in text and "from oracle" not in text, py


def test_peer_exchange_abi_rejects_bad_arguments_without_gpu():
    """tf_comm_*: argument checks come before any CUDA call."""
    lib = nat.load_library()
    h = ctypes.c_void_p()
    assert lib.tf_comm_create(2, 2, 640, 480, ctypes.byref(h)) == -1      # rank >= world
    assert lib.tf_comm_create(0, 0, 640, 480, ctypes.byref(h)) == -1      # world < 1
    assert lib.tf_comm_create(0, nat.COMM_MAX_RANKS + 1, 640, 480, ctypes.byref(h)) == -1
    assert lib.tf_comm_create(0, 2, 0, 480, ctypes.byref(h)) == -1        # empty image
    assert b"tf_comm_create" in lib.tf_last_error()
    assert lib.tf_comm_reduce_raymap(None, 0, None) == -1
    assert lib.tf_comm_import(None, None) == -1
    assert lib.tf_comm_export(None, None) == -1
    assert lib.tf_comm_link_local(None, 2) == -1
    e = ctypes.c_int(7)
    assert lib.tf_comm_error(None, ctypes.byref(e)) == -1
    assert lib.tf_comm_destroy(None) == 0
