"""ctypes binding of libtfb200.so (include/tfb200.h) and device plumbing.

There is no fallback: if the library or a CUDA device is missing, every
entry point raises.  PyTorch supplies device memory, the current stream and
the device index only; all arithmetic of the hot path runs in libtfb200.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np
import torch

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["TFB200_LIB"]) if os.environ.get("TFB200_LIB") else _PKG / "libtfb200.so"  # override: A/B runs only
ABI_VERSION = 2
MAX_VOLUMES_PER_LAUNCH = 64  # TFB200_MAX_VOLUMES_PER_LAUNCH

_c_d = ctypes.c_double
_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_p = ctypes.c_void_p
_c_sz = ctypes.c_size_t


class TfVolume(ctypes.Structure):
    _fields_ = [("voxels_dev", _c_p), ("n", _c_i64), ("origin", _c_i64 * 3),
                ("voxel_size", _c_d), ("brick_state_dev", _c_p), ("brick_flags_dev", _c_p),
                ("summary_threshold", ctypes.c_float),
                ("reserved", ctypes.c_int32), ("color_dev", _c_p), ("counters_dev", _c_p)]


class TfCamera(ctypes.Structure):
    _fields_ = [("fx", _c_d), ("fy", _c_d), ("cx", _c_d), ("cy", _c_d), ("width", _c_i64),
                ("height", _c_i64)]


DEBUG_NO_CULL = 1
DEBUG_EXACT_ONLY = 2
DEBUG_NO_FIXEDPOINT = 4
DEBUG_LANE0_ONLY = 8
DEBUG_COOP_ALL = 16
RAYCAST_FRESH = 1  # tf_raycast_ex flag (tfb200.h TF_RAYCAST_FRESH)
PROF_INTEGRATE_UPDATE, PROF_INTEGRATE_ALL, PROF_RAYCAST, PROF_KINDS = 0, 1, 2, 8


def profile_read() -> dict:
    """Summed device ms / launches per profiled kind since the last read."""
    ms = (ctypes.c_double * PROF_KINDS)()
    cnt = (ctypes.c_int64 * PROF_KINDS)()
    check(lib().tf_profile_read(ms, cnt, PROF_KINDS), "tf_profile_read")
    names = ("integrate_update", "integrate_all", "raycast", "integrate_free", "integrate_general",
             "integrate_exact", "raycast_coop", "integrate_screen")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(names)}

# TF_STAT_* slots (tfb200.h)
STAT_VOXEL_UPDATES, STAT_SWEPT_VOXELS, STAT_ACTIVE_BRICKS, STAT_TOTAL_BRICKS = 0, 1, 2, 3
STAT_RAY_SAMPLES, STAT_RAY_HITS, STAT_EXACT_VOXELS, STAT_NOOP_UPDATES = 4, 5, 6, 7
STAT_COL_SKIPPED, STAT_DEPTH_SKIPPED, STAT_FREE_BRICKS, STAT_EXACT_SAMPLES = 8, 9, 10, 11
STAT_CERT_FAILURES = 12
STAT_SUMMARY_SAMPLES = 13
STAT_GENERAL_ALL_FREE = 14
STAT_COOP_RAYS = 15
STAT_FREE_KERNEL_UPDATES = 16
STAT_EXACT_UPDATES = 17
STAT_PART_ALL_FREE = 18
STAT_PART_ALL_SKIP = 19
STAT_COUNT = 24

_VOL = ctypes.POINTER(TfVolume)
_CAM = ctypes.POINTER(TfCamera)

_SIGNATURES = {
    "tf_abi_version": (_c_int, []),
    "tf_last_error": (ctypes.c_char_p, []),
    "tf_set_debug_flags": (None, [ctypes.c_uint32]),
    "tf_debug_flags": (ctypes.c_uint32, []),
    "tf_launch_count": (ctypes.c_uint64, []),
    "tf_debug_bounds_violations": (ctypes.c_uint64, []),
    "tf_debug_ray_clock_buffer": (None, [_c_p]),
    "tf_icp_track_state_size": (ctypes.c_size_t, []),
    "tf_icp_track": (_c_int, [ctypes.c_int, _c_p, _c_p, _c_p, ctypes.POINTER(TfCamera), _c_p, _c_p,
                              _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_d, _c_d,
                              _c_d, _c_p, ctypes.c_size_t, _c_p, _c_p]),
    "tf_debug_weight_division_check": (_c_i64, [_c_i64, ctypes.c_uint64]),
    "tf_debug_ray_interval_check": (_c_i64, [_c_i64, ctypes.c_uint64]),
    "tf_debug_div_check": (_c_i64, [_c_i64, ctypes.c_uint64]),
    "tf_profile_enable": (None, [_c_int]),
    "tf_profile_read": (_c_int, [_c_p, _c_p, _c_int]),
    "tf_integrate_workspace_size": (_c_sz, [_VOL, _c_int, _CAM]),
    "tf_integrate": (_c_int, [_VOL, _c_int, _c_p, _CAM, _c_p, _c_p, _c_p, _c_d, _c_d, _c_d,
                              _c_p, _c_sz, _c_p, _c_p]),
    "tf_integrate_rgb": (_c_int, [_VOL, _c_int, _c_p, _c_p, _CAM, _c_p, _c_p, _c_p, _c_d, _c_d, _c_d,
                                  _c_p, _c_sz, _c_p, _c_p]),
    "tf_integrate_prepare": (_c_int, [_VOL, _c_int, _c_p, _CAM, _c_p, _c_p, _c_p, _c_d, _c_d, _c_d,
                                      _c_p, _c_sz, _c_p]),
    "tf_integrate_finish": (_c_int, [_VOL, _c_int, _c_p, _c_p, _CAM, _c_p, _c_p, _c_p, _c_d, _c_d, _c_d,
                                     _c_p, _c_sz, _c_p, _c_p]),
    "tf_raycast_colors": (_c_int, [_VOL, _c_int, _CAM, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "tf_raycast": (_c_int, [_VOL, _c_int, _CAM, _c_d, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                            _c_p, _c_p]),
    "tf_raycast_workspace_size": (_c_sz, [_c_int, _CAM]),
    "tf_raycast_ws": (_c_int, [_VOL, _c_int, _CAM, _c_d, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                               _c_p, _c_sz, _c_p, _c_p]),
    "tf_raycast_rows": (_c_int, [_VOL, _c_int, _CAM, _c_d, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                                 _c_p, _c_sz, _c_int, _c_int, _c_p, _c_p]),
    "tf_raycast_ex": (_c_int, [_VOL, _c_int, _CAM, _c_d, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                               _c_p, _c_sz, _c_int, _c_int, _c_int, _c_p, _c_p]),
    "tf_trilinear_sample": (_c_int, [_VOL, _c_p, _c_i64, _c_p, _c_p, _c_p]),
    "tf_good_threshold": (ctypes.c_float, [_c_d]),
    "tf_brick_summary": (_c_int, [_VOL, _c_p]),
    "tf_raymap_merge": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "tf_raymap_merge_packed": (_c_int, [_c_p, _c_p, _c_i64, _c_p]),
    "tf_raymap_reset": (_c_int, [_c_p, _c_p, _c_p, _c_i64, _c_p]),
    "tf_raymap_vertices": (_c_int, [_c_p, _c_i64, _c_p, _CAM, _c_p, _c_p, _c_i64,
                                    _c_i64, _c_p]),
    "tf_vertex_normal_map": (_c_int, [_c_p, _c_i64, _c_i64, _c_int, _CAM, _c_p, _c_p, _c_p,
                                      _c_p]),
    "tf_icp_workspace_size": (_c_sz, [_c_i64]),
    "tf_icp_reduce": (_c_int, [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_i64,
                               _c_i64, _c_int, _CAM, _c_p, _c_p, _c_p, _c_p, _c_d, _c_d, _c_p,
                               _c_sz, _c_p, _c_p]),
    "tf_extract_workspace_size": (_c_sz, [_c_i64]),
    "tf_extract_count": (_c_int, [_VOL, _c_p, _c_sz, _c_p, _c_p]),
    "tf_extract_emit": (_c_int, [_VOL, _c_p, _c_sz, _c_p, _c_p, _c_p]),
    "tf_endpoint_cells": (_c_int, [_c_p, _CAM, _c_p, _c_p, _c_d, _c_p, _c_p]),
    "tf_pack_voxels": (_c_int, [_c_p, _c_i64, _c_p, _c_p, _c_p]),
    "tf_unpack_voxels": (_c_int, [_c_p, _c_p, _c_i64, _c_p, _c_p]),
    "tf_bin_endpoints_workspace_size": (_c_sz, [_c_i64]),
    "tf_bin_endpoints": (_c_int, [_c_p, _CAM, _c_p, _c_p, _c_d, _c_i64, _c_p, _c_sz, _c_p, _c_p]),
    "tf_comm_create": (_c_int, [_c_int, _c_int, _c_i64, _c_i64, ctypes.POINTER(_c_p)]),
    "tf_comm_layout": (_c_int, [_c_p, ctypes.POINTER(_c_p), _c_p]),
    "tf_comm_export": (_c_int, [_c_p, _c_p]),
    "tf_comm_import": (_c_int, [_c_p, _c_p]),
    "tf_comm_link_local": (_c_int, [_c_p, _c_int]),
    "tf_comm_reduce_raymap": (_c_int, [_c_p, ctypes.c_uint, _c_p]),
    "tf_comm_error": (_c_int, [_c_p, ctypes.POINTER(_c_int)]),
    "tf_comm_error_poll": (_c_int, [_c_p, ctypes.POINTER(_c_int)]),
    "tf_comm_destroy": (_c_int, [_c_p]),
}

# peer-memory ray-map reduction (tfb200.h "multi-GPU ray-map reduction")
COMM_HANDLE_BYTES = 64
COMM_MAX_RANKS = 64
(COMM_FLAGS, COMM_PART_DIST, COMM_PART_VERT, COMM_PART_NORM, COMM_MODEL_DIST, COMM_MODEL_VERT,
 COMM_MODEL_NORM, COMM_NSECTIONS) = range(8)
COMM_NOWAIT = 1

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def load_library(path: Path | str | None = None) -> ctypes.CDLL:
    """Load libtfb200.so (no CUDA device needed just to load and bind)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build it with `python -m paper_1511_07106_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.tf_abi_version() != ABI_VERSION:
            raise RuntimeError(f"libtfb200 ABI {lib.tf_abi_version()} != {ABI_VERSION}")
        if path is None:
            _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return load_library()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().tf_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------

def device() -> torch.device:
    """The CUDA device the hot path runs on (torch's current device)."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1511_07106_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device buffers must be contiguous CUDA tensors"
    return t.data_ptr()


def mat9(m) -> ctypes.Array:
    a = np.ascontiguousarray(m, dtype=np.float64).reshape(9)
    return (_c_d * 9)(*a.tolist())


def vec3(v) -> ctypes.Array:
    a = np.ascontiguousarray(v, dtype=np.float64).reshape(3)
    return (_c_d * 3)(*a.tolist())


def camera(intr) -> TfCamera:
    return TfCamera(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy),
                    int(intr.width), int(intr.height))


def volume_struct(voxels: torch.Tensor, n: int, origin, voxel_size: float,
                  brick_state: torch.Tensor | None = None, brick_flags: torch.Tensor | None = None,
                  threshold: float = 0.0, color: torch.Tensor | None = None,
                  counters: torch.Tensor | None = None) -> TfVolume:
    o = np.asarray(origin, dtype=np.int64)
    return TfVolume(ptr(voxels), int(n), (_c_i64 * 3)(int(o[0]), int(o[1]), int(o[2])),
                    float(voxel_size), ptr(brick_state) if brick_state is not None else None,
                    ptr(brick_flags) if brick_flags is not None else None, float(threshold), 0,
                    ptr(color) if color is not None else None,
                    ptr(counters) if counters is not None else None)


class _Workspace:
    """Per-device grow-only scratch buffer handed to the C ABI."""

    def __init__(self) -> None:
        self._bufs: dict[int, torch.Tensor] = {}

    def get(self, nbytes: int, slot: str = "main") -> torch.Tensor:
        dev = device()
        key = (dev.index, slot)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
            self._bufs[key] = buf
        return buf


workspace = _Workspace()


class _Stats:
    """Per-device uint64[8] counter block accumulated by the kernels."""

    def __init__(self) -> None:
        self._bufs: dict[int, torch.Tensor] = {}

    def buffer(self) -> torch.Tensor:
        dev = device()
        buf = self._bufs.get(dev.index)
        if buf is None:
            buf = torch.zeros(STAT_COUNT, dtype=torch.int64, device=dev)
            self._bufs[dev.index] = buf
        return buf

    def read(self) -> np.ndarray:
        return self.buffer().cpu().numpy().astype(np.uint64)

    def reset(self) -> None:
        self.buffer().zero_()


stats = _Stats()


def env_flag(name: str) -> bool:
    return os.environ.get(name, "").lower() in ("1", "true", "yes", "on")
