"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle.

The oracle (``tf_oracle.c``) restates the reference tilefusion hot path in
plain C; this module binds it for numpy arrays.  It is imported only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs — as the
checker and as the CPU baseline, never by the product package.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference package itself
(``tests/golden/make_golden.py``) and, when ``/root/reference`` is present,
against the live reference.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libtf_oracle.so"
_lib = None

_d = ctypes.c_double
_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def build(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    src = _HERE / "tf_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.tfo_integrate.restype = _i64
        L.tfo_integrate.argtypes = [_p, _p, _i64, _p, _d, _p, _i64, _i64, _p, _p, _p,
                                    _d, _d, _d, _d, _d, _d, _d, ctypes.c_int]
        L.tfo_sample.restype = ctypes.c_int
        L.tfo_sample.argtypes = [_p, _p, _i64, _d, _d, _d, ctypes.POINTER(_d)]
        L.tfo_raycast.restype = _i64
        L.tfo_raycast.argtypes = [_p, _p, _i64, _p, _d, _d, _i64, _p, _p, _d, _d, _d,
                                  _d, _i64, _i64, _p, _p, _p, ctypes.c_int]
        L.tfo_extract_bound.restype = _i64
        L.tfo_extract_bound.argtypes = [_p, _p, _i64]
        L.tfo_extract.restype = _i64
        L.tfo_extract.argtypes = [_p, _p, _i64, _p, _d, _p, _p]
        L.tfo_vertex_normal_map.restype = None
        L.tfo_vertex_normal_map.argtypes = [_p, _i64, _i64, _d, _d, _d, _d, _p, _p, _p]
        L.tfo_icp_reduce.restype = None
        L.tfo_icp_reduce.argtypes = [_p, _p, _p, _i64, _i64, _p, _p, _p, _i64, _i64,
                                     _p, _p, _p, _p, _d, _d, _d, _d, _i64, _i64, _d,
                                     _d, _p]
        L.tfo_endpoint_cells.restype = _i64
        L.tfo_endpoint_cells.argtypes = [_p, _i64, _i64, _d, _d, _d, _d, _p, _p, _d, _p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags.c_contiguous, "oracle arrays must be C-contiguous"
    return a.ctypes.data


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# integration / sampling / raycast / extraction (reference _kernels.py)
# ---------------------------------------------------------------------------

def integrate(tsdf: np.ndarray, weight: np.ndarray, ht, voxel_size: float,
              depth: np.ndarray, r_cw, t_cw, cam_center, fx, fy, cx, cy, tau,
              max_weight, sample_weight, threads: int = 1) -> int:
    """In-place integrate_kernel (_kernels.py:71-133); returns voxel updates."""
    assert tsdf.dtype == np.float32 and weight.dtype == np.float32
    n = tsdf.shape[0]
    ht = _c(ht, np.int64)
    depth = _c(depth, np.float64)
    r = _c(r_cw, np.float64)
    t = _c(t_cw, np.float64)
    c = _c(cam_center, np.float64)
    h, w = depth.shape
    return int(lib().tfo_integrate(_ptr(tsdf), _ptr(weight), n, _ptr(ht), float(voxel_size),
                                   _ptr(depth), h, w, _ptr(r), _ptr(t), _ptr(c), float(fx),
                                   float(fy), float(cx), float(cy), float(tau),
                                   float(max_weight), float(sample_weight), int(threads)))


def sample(tsdf, weight, qx, qy, qz):
    """_sample (_kernels.py:28-68) -> (valid, value)."""
    v = _d(0.0)
    ok = lib().tfo_sample(_ptr(tsdf), _ptr(weight), tsdf.shape[0], float(qx), float(qy),
                          float(qz), ctypes.byref(v))
    return bool(ok), (v.value if ok else 0.0)


def raycast(tsdf, weight, ht, voxel_size, tau, coarse_step, r_wc, cam_center, fx, fy,
            cx, cy, out_dist, out_vert, out_norm, threads: int = 1) -> int:
    """In-place raycast_kernel merge (_kernels.py:266-451); returns samples."""
    ht = _c(ht, np.int64)
    r = _c(r_wc, np.float64)
    c = _c(cam_center, np.float64)
    h, w = out_dist.shape
    return int(lib().tfo_raycast(_ptr(tsdf), _ptr(weight), tsdf.shape[0], _ptr(ht),
                                 float(voxel_size), float(tau), int(coarse_step), _ptr(r),
                                 _ptr(c), float(fx), float(fy), float(cx), float(cy), h, w,
                                 _ptr(out_dist), _ptr(out_vert), _ptr(out_norm),
                                 int(threads)))


def extract(tsdf, weight, ht, voxel_size):
    """extract_bound + extract_kernel (_kernels.py:454-578) -> (verts, norms)."""
    n = tsdf.shape[0]
    bound = int(lib().tfo_extract_bound(_ptr(tsdf), _ptr(weight), n))
    verts = np.empty((bound, 3))
    norms = np.empty((bound, 3))
    ht = _c(ht, np.int64)
    count = int(lib().tfo_extract(_ptr(tsdf), _ptr(weight), n, _ptr(ht), float(voxel_size),
                                  _ptr(verts), _ptr(norms)))
    return verts[:count].copy(), norms[:count].copy()


# ---------------------------------------------------------------------------
# ICP pieces (geometry.py / tracking.py)
# ---------------------------------------------------------------------------

def vertex_normal_map(depth, fx, fy, cx, cy):
    """VertexNormalMap.from_depth (geometry.py:313-317) -> (verts, norms, valid)."""
    depth = _c(depth, np.float64)
    h, w = depth.shape
    verts = np.empty((h, w, 3))
    norms = np.empty((h, w, 3))
    valid = np.empty((h, w), np.uint8)
    lib().tfo_vertex_normal_map(_ptr(depth), h, w, float(fx), float(fy), float(cx),
                                float(cy), _ptr(verts), _ptr(norms), _ptr(valid))
    return verts, norms, valid.astype(bool)


def icp_reduce(src_v, src_n, src_valid, mdl_v, mdl_n, mdl_valid, r_est, t_est, r_ref,
               t_ref, fx, fy, cx, cy, width, height, max_d2, cos_min) -> np.ndarray:
    """Per-pixel _solve_step terms (tracking.py:76-108) -> 29 sums."""
    src_v = _c(src_v, np.float64)
    src_n = _c(src_n, np.float64)
    sv = _c(src_valid, np.uint8)
    mdl_v = _c(mdl_v, np.float64)
    mdl_n = _c(mdl_n, np.float64)
    mv = _c(mdl_valid, np.uint8)
    out = np.zeros(29)
    args = [_c(r_est, np.float64), _c(t_est, np.float64), _c(r_ref, np.float64),
            _c(t_ref, np.float64)]
    lib().tfo_icp_reduce(_ptr(src_v), _ptr(src_n), _ptr(sv), sv.shape[0], sv.shape[1],
                         _ptr(mdl_v), _ptr(mdl_n), _ptr(mv), mv.shape[0], mv.shape[1],
                         *[_ptr(a) for a in args], float(fx), float(fy), float(cx),
                         float(cy), int(width), int(height), float(max_d2), float(cos_min),
                         _ptr(out))
    return out


def endpoint_cells(depth, fx, fy, cx, cy, r_wc, t_wc, block_side) -> np.ndarray:
    """Per-valid-pixel endpoint cells of bin_endpoints (volumes.py:318-326)."""
    depth = _c(depth, np.float64)
    h, w = depth.shape
    cells = np.empty((h * w, 3), np.int64)
    k = int(lib().tfo_endpoint_cells(_ptr(depth), h, w, float(fx), float(fy), float(cx),
                                     float(cy), _ptr(_c(r_wc, np.float64)),
                                     _ptr(_c(t_wc, np.float64)), float(block_side),
                                     _ptr(cells)))
    return cells[:k].copy()


def bin_endpoints(depth, fx, fy, cx, cy, r_wc, t_wc, spacing, voxel_size) -> dict:
    """bin_endpoints (volumes.py:305-331): tile key -> endpoint count."""
    cells = endpoint_cells(depth, fx, fy, cx, cy, r_wc, t_wc, spacing * voxel_size)
    if len(cells) == 0:
        return {}
    uniq, counts = np.unique(cells, axis=0, return_counts=True)
    return {(int(c[0] * spacing), int(c[1] * spacing), int(c[2] * spacing)): int(k)
            for c, k in zip(uniq, counts)}


def solve_from_sums(sums: np.ndarray, min_pairs: int):
    """Host 6x6 step of _solve_step (tracking.py:100-120) from the 29 sums."""
    count = int(round(sums[28]))
    if count < min_pairs:
        return None
    ata = np.empty((6, 6))
    k = 0
    for i in range(6):
        for j in range(i, 6):
            ata[i, j] = ata[j, i] = sums[k]
            k += 1
    atb = sums[21:27].copy()
    if np.linalg.cond(ata) > 1.0e12:
        return None
    try:
        delta = np.linalg.solve(ata, atb)
    except np.linalg.LinAlgError:
        return None
    if not np.all(np.isfinite(delta)):
        return None
    return delta, count, float(np.sqrt(sums[27] / count))


# ---------------------------------------------------------------------------
# tracking.track (tracking.py:123-196) over the oracle's per-pixel pieces
# ---------------------------------------------------------------------------

def _rodrigues(axis, angle: float) -> np.ndarray:
    """rotation_from_axis_angle (geometry.py:211-219)."""
    import math
    axis = np.asarray(axis, dtype=np.float64)
    norm = np.linalg.norm(axis)
    if norm == 0.0 or angle == 0.0:
        return np.eye(3)
    x, y, z = axis / norm
    k = np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])
    return np.eye(3) + math.sin(angle) * k + (1.0 - math.cos(angle)) * (k @ k)


def _orthonormalized(rot: np.ndarray) -> np.ndarray:
    """Pose.orthonormalized (geometry.py:169-176)."""
    u, _, vt = np.linalg.svd(rot)
    r = u @ vt
    if np.linalg.det(r) < 0:
        u[:, -1] = -u[:, -1]
        r = u @ vt
    return r


def track(depth, fx, fy, cx, cy, model_dist, model_vert, model_norm, ref_rot, ref_t,
          seed_rot, seed_t, max_distance=0.10, max_angle_deg=20.0, iterations=(10, 5, 4),
          min_correspondences=1000, step_eps=1.0e-10):
    """tracking.track (tracking.py:123-196): stride-2 pyramids of the frame and
    the model (geometry.py:256-258, :326-332; CameraIntrinsics.scaled :44-57),
    coarsest level first, per step icp_reduce + solve_from_sums + the Rodrigues
    update re-orthonormalised (:178-183).  Returns (rot, t, lost, count, rms)."""
    depth = np.asarray(depth, np.float64)
    ref_rot = np.asarray(ref_rot, np.float64)
    ref_t = np.asarray(ref_t, np.float64)
    inv_r = ref_rot.T.copy()
    inv_t = -(inv_r @ ref_t)
    est_r, est_t = np.asarray(seed_rot, np.float64), np.asarray(seed_t, np.float64)
    cos_min = float(np.cos(np.deg2rad(max_angle_deg)))
    levels = len(iterations)
    h, w = depth.shape
    count, rms, lost = 0, float("inf"), False
    for level in range(levels - 1, -1, -1):
        s = 1 << level
        d = depth[::s, ::s]
        lw = max(1, int(round(w * 0.5 ** level)))
        lh = max(1, int(round(h * 0.5 ** level)))
        lfx, lfy, lcx, lcy = fx, fy, cx, cy
        for _ in range(level):  # scaled(0.5) applied level times
            lfx, lfy, lcx, lcy = lfx * 0.5, lfy * 0.5, lcx * 0.5, lcy * 0.5
        sv, sn, sok = vertex_normal_map(d, lfx, lfy, lcx, lcy)
        sok = sok & np.all(np.isfinite(sn), axis=-1)
        md = model_dist[::s, ::s]
        mv, mn = model_vert[::s, ::s], model_norm[::s, ::s]
        mok = np.isfinite(md)
        min_pairs = max(6, min_correspondences // 4 ** level)
        for _ in range(iterations[level]):
            sums = icp_reduce(sv, sn, sok, mv, mn, mok, est_r, est_t, inv_r, inv_t, lfx, lfy,
                              lcx, lcy, lw, lh, max_distance ** 2, cos_min)
            step = solve_from_sums(sums, min_pairs)
            if step is None:
                lost = True
                break
            delta, count, rms = step
            rot = _rodrigues(delta[:3], float(np.linalg.norm(delta[:3])))
            est_r, est_t = _orthonormalized(rot @ est_r), rot @ est_t + delta[3:]
            if float(np.linalg.norm(delta)) < step_eps:
                break
        if lost:
            break
    if lost:
        return np.asarray(seed_rot, np.float64), np.asarray(seed_t, np.float64), True, count, rms
    return est_r, est_t, False, count, rms
