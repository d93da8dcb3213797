"""Frame-to-model tracking: projective point-to-plane ICP on the GPU.

Drop-in for tilefusion/tracking.py.  ``track`` keeps the reference's
control flow exactly (pyramid of stride-2 levels, coarsest first, per-level
iteration counts and pair minimums, Rodrigues update + SVD
re-orthonormalisation, loss semantics; tracking.py:123-196) and runs all of
it on the device in one call (tf_icp_track):

* the source vertex / normal maps of every level (tf_vertex_normal_map,
  read straight from the full-resolution depth at stride 2^level);
* every ``_solve_step``'s per-pixel work — transform, projective
  association, distance / angle gates, and a deterministic warp-shuffle
  reduction of A^T A, A^T r, sum r^2 and the inlier count (29 doubles);
* the host part of ``_solve_step`` (tracking.py:100-120: pair minimum, the
  cond > 1e12 gate, LU solve with partial pivoting, finiteness) and the
  pose update (:178-183), in a single-warp kernel per step; steps after a
  loss or convergence return at once.

One read-back per frame (the final pose, loss flag, count and rms).
``track_host`` is the same loop with one host round trip per step (the 6x6
part in numpy, operation for operation as the reference); ``icp_sums`` /
``solve_step`` expose a single step (parity tests replay the reference's
steps through them).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .geometry import CameraIntrinsics, Pose, rotation_from_axis_angle
from .tsdf import RayMap, device_depth


@dataclass(frozen=True)
class TrackingParams:
    """Projective point-to-plane ICP knobs (tracking.py:28-51).

    ``iterations`` is indexed by pyramid level (0 = full resolution); levels
    run coarsest first.  ``min_correspondences`` applies at full resolution
    and is divided by 4 per level above it.
    """

    max_distance: float = 0.10
    max_angle_deg: float = 20.0
    iterations: tuple[int, ...] = (10, 5, 4)
    min_correspondences: int = 1000
    step_eps: float = 1.0e-10

    def __post_init__(self) -> None:
        if self.max_distance <= 0.0:
            raise ValueError("max_distance must be positive")
        if not 0.0 < self.max_angle_deg < 90.0:
            raise ValueError("max_angle_deg must be in (0, 90)")
        if len(self.iterations) == 0 or any(i < 1 for i in self.iterations):
            raise ValueError("iterations must be a non-empty tuple of >= 1")
        if self.min_correspondences < 6:
            raise ValueError("min_correspondences must be at least 6")


@dataclass(frozen=True)
class TrackResult:
    pose: Pose
    lost: bool
    correspondences: int
    residual_rms: float


def _level_shape(full_h: int, full_w: int, level: int) -> tuple[int, int]:
    s = 1 << level
    return (full_h + s - 1) // s, (full_w + s - 1) // s


@dataclass
class SourceLevel:
    """Device vertex / normal map of one pyramid level."""

    intr: CameraIntrinsics
    level: int
    verts: torch.Tensor
    norms: torch.Tensor
    valid: torch.Tensor


def source_level(depth: torch.Tensor, intr: CameraIntrinsics, level: int) -> SourceLevel:
    """tf_vertex_normal_map of ``depth`` (full resolution) at stride 2^level."""
    full_h, full_w = depth.shape
    h, w = _level_shape(full_h, full_w, level)
    if (h, w) != (intr.height, intr.width):
        raise ValueError(f"depth shape {(h, w)} does not match intrinsics "
                         f"{intr.height}x{intr.width}")
    dev = depth.device
    verts = torch.empty((h, w, 3), dtype=torch.float64, device=dev)
    norms = torch.empty((h, w, 3), dtype=torch.float64, device=dev)
    valid = torch.empty((h, w), dtype=torch.uint8, device=dev)
    nat.check(nat.lib().tf_vertex_normal_map(nat.ptr(depth), full_w, full_h, level,
                                             nat.camera(intr), nat.ptr(verts), nat.ptr(norms),
                                             nat.ptr(valid), nat.stream_handle()),
              "tf_vertex_normal_map")
    return SourceLevel(intr, level, verts, norms, valid)


def vertex_normal_map_device(intr: CameraIntrinsics, frame) -> tuple:
    """VertexNormalMap.from_depth on the device -> (verts, norms, valid) tensors."""
    depth = device_depth(frame)
    if tuple(depth.shape) != (intr.height, intr.width):
        raise ValueError(f"depth shape {tuple(depth.shape)} does not match intrinsics "
                         f"{intr.height}x{intr.width}")
    lvl = source_level(depth, intr, 0)
    return lvl.verts, lvl.norms, lvl.valid


class _SumsReader:
    """Pinned host landing buffer for the 29 ICP sums."""

    def __init__(self) -> None:
        self._dev: dict = {}
        self._host: dict = {}

    def buffers(self):
        d = nat.device()
        if d.index not in self._dev:
            self._dev[d.index] = torch.zeros(29, dtype=torch.float64, device=d)
            self._host[d.index] = torch.zeros(29, dtype=torch.float64).pin_memory()
        return self._dev[d.index], self._host[d.index]


_sums = _SumsReader()


def icp_sums(src: SourceLevel, model: RayMap, estimate: Pose, ref_inv: Pose,
             params: TrackingParams) -> np.ndarray:
    """The 29 normal-equation sums of one _solve_step (tracking.py:76-108)."""
    model._device_read()
    h, w = src.valid.shape
    L = nat.lib()
    need = L.tf_icp_workspace_size(h * w)
    ws = nat.workspace.get(need, slot="icp")
    out_dev, out_host = _sums.buffers()
    mh, mw = model.distance_dev.shape
    cos_min = float(np.cos(np.deg2rad(params.max_angle_deg)))
    nat.check(L.tf_icp_reduce(
        nat.ptr(src.verts), nat.ptr(src.norms), nat.ptr(src.valid), w, h,
        nat.ptr(model.distance_dev), nat.ptr(model.vertices_dev), nat.ptr(model.normals_dev),
        mw, mh, src.level, nat.camera(src.intr), nat.mat9(estimate.rotation),
        nat.vec3(estimate.translation), nat.mat9(ref_inv.rotation), nat.vec3(ref_inv.translation),
        float(params.max_distance ** 2), cos_min, nat.ptr(ws), ws.numel(), nat.ptr(out_dev),
        nat.stream_handle()), "tf_icp_reduce")
    out_host.copy_(out_dev, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out_host.numpy().copy()


def solve_from_sums(sums: np.ndarray, min_pairs: int):
    """The host 6x6 part of _solve_step (tracking.py:100-120)."""
    count = int(round(float(sums[28])))
    if count < min_pairs:
        return None
    ata = np.empty((6, 6))
    k = 0
    for i in range(6):
        for j in range(i, 6):
            ata[i, j] = ata[j, i] = sums[k]
            k += 1
    atb = np.array(sums[21:27], dtype=np.float64)
    # degenerate geometry leaves unobservable motion: report lost, not a guess
    if np.linalg.cond(ata) > 1.0e12:
        return None
    try:
        delta = np.linalg.solve(ata, atb)
    except np.linalg.LinAlgError:
        return None
    if not np.all(np.isfinite(delta)):
        return None
    return delta, count, float(np.sqrt(float(sums[27]) / count))


def solve_step(src: SourceLevel, model: RayMap, estimate: Pose, ref_inv: Pose,
               params: TrackingParams, min_pairs: int):
    """One linearised update -> (delta, count, rms) or None when lost."""
    return solve_from_sums(icp_sums(src, model, estimate, ref_inv, params), min_pairs)


def apply_delta(estimate: Pose, delta: np.ndarray) -> Pose:
    """Left-multiply the Rodrigues increment and re-orthonormalise (tracking.py:178-181)."""
    rot = rotation_from_axis_angle(delta[:3], float(np.linalg.norm(delta[:3])))
    return Pose(rot @ estimate.rotation, rot @ estimate.translation + delta[3:]).orthonormalized()


def _pyramid(frame, intr: CameraIntrinsics, params: TrackingParams) -> list[SourceLevel]:
    depth = device_depth(frame)
    if tuple(depth.shape) != (intr.height, intr.width):
        raise ValueError(f"depth shape {tuple(depth.shape)} does not match intrinsics "
                         f"{intr.height}x{intr.width}")
    levels = len(params.iterations)
    intrs = [intr]
    for _ in range(levels - 1):
        intrs.append(intrs[-1].scaled(0.5))
    return [source_level(depth, intrs[l], l) for l in range(levels)]


class _TrackState:
    """Device state of tf_icp_track and its pinned landing buffer."""

    def __init__(self) -> None:
        self._bufs: dict = {}

    def buffers(self):
        d = nat.device()
        if d.index not in self._bufs:
            n = int(nat.lib().tf_icp_track_state_size()) // 8
            self._bufs[d.index] = (torch.zeros(n, dtype=torch.float64, device=d),
                                   torch.zeros(n, dtype=torch.float64).pin_memory())
        return self._bufs[d.index]


_track_state = _TrackState()


def track(frame, intr: CameraIntrinsics, model: RayMap, ref_pose: Pose,
          params: TrackingParams = TrackingParams(), init: Pose | None = None) -> TrackResult:
    """Align a depth frame against a rendered model view (tracking.py:123-196).

    ``frame`` is a DepthFrame (uploaded once) or a resident float64 depth
    tensor.  Returns the refined camera-to-world pose, or the seed flagged
    lost when too few pairs survive or the normal system is degenerate.  The
    whole pyramid runs on the device (tf_icp_track) with one read-back at the
    end; ``track_host`` is the same loop with the 6x6 part in numpy.
    """
    pyramid = _pyramid(frame, intr, params)
    model._device_read()
    levels = len(pyramid)
    L = nat.lib()
    h0, w0 = pyramid[0].valid.shape
    ws = nat.workspace.get(L.tf_icp_workspace_size(h0 * w0), slot="icp")
    state, host = _track_state.buffers()
    ptrs = lambda ts: (ctypes.c_void_p * levels)(*[t.data_ptr() for t in ts])
    cams = (nat.TfCamera * levels)(*[nat.camera(p.intr) for p in pyramid])
    its = (ctypes.c_int * levels)(*[int(i) for i in params.iterations])
    mins = (ctypes.c_int * levels)(*[max(6, params.min_correspondences // 4 ** l) for l in range(levels)])
    ref_inv = ref_pose.invert()
    seed = init if init is not None else ref_pose
    mh, mw = model.distance_dev.shape
    nat.check(L.tf_icp_track(
        levels, ptrs([p.verts for p in pyramid]), ptrs([p.norms for p in pyramid]),
        ptrs([p.valid for p in pyramid]), cams, its, mins, nat.ptr(model.distance_dev),
        nat.ptr(model.vertices_dev), nat.ptr(model.normals_dev), mw, mh,
        nat.mat9(ref_inv.rotation), nat.vec3(ref_inv.translation), nat.mat9(seed.rotation),
        nat.vec3(seed.translation), float(params.max_distance ** 2),
        float(np.cos(np.deg2rad(params.max_angle_deg))), float(params.step_eps), nat.ptr(ws), ws.numel(),
        nat.ptr(state), nat.stream_handle()), "tf_icp_track")
    host.copy_(state, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    st = host.numpy()
    count = int(st[13])
    rms = float(st[14]) if count > 0 else float("inf")
    if st[12] != 0.0:
        return TrackResult(pose=seed, lost=True, correspondences=count, residual_rms=rms)
    pose = Pose(st[0:9].reshape(3, 3).copy(), st[9:12].copy())
    return TrackResult(pose=pose, lost=False, correspondences=count, residual_rms=rms)


def track_host(frame, intr: CameraIntrinsics, model: RayMap, ref_pose: Pose,
               params: TrackingParams = TrackingParams(), init: Pose | None = None) -> TrackResult:
    """track() with one host round trip per step: the 6x6 gate / solve and
    the pose update in numpy, operation for operation as tracking.py:100-183."""
    pyramid = _pyramid(frame, intr, params)
    levels = len(pyramid)

    ref_inv = ref_pose.invert()
    estimate = init if init is not None else ref_pose
    lost = False
    count = 0
    rms = float("inf")
    for level in range(levels - 1, -1, -1):
        min_pairs = max(6, params.min_correspondences // 4 ** level)
        for _ in range(params.iterations[level]):
            step = solve_step(pyramid[level], model, estimate, ref_inv, params, min_pairs)
            if step is None:
                lost = True
                break
            delta, count, rms = step
            estimate = apply_delta(estimate, delta)
            if float(np.linalg.norm(delta)) < params.step_eps:
                break
        if lost:
            break
    if lost:
        return TrackResult(pose=init if init is not None else ref_pose, lost=True,
                           correspondences=count, residual_rms=rms)
    return TrackResult(pose=estimate, lost=False, correspondences=count, residual_rms=rms)
