"""Device-resident TSDF subvolumes: integration, raycast, sampling, extraction.

Drop-in for the reference module tilefusion/tsdf.py: the same names,
signatures, in-place semantics and errors, with the storage moved to the GPU
and the operators running in libtfb200 (include/tfb200.h):

* ``TsdfSubvolume`` keeps its voxels as one device tensor ``voxels``
  float32 [n, n, n, 2] = (tsdf, weight) interleaved, x fastest — the layout
  of the reference spill body (volumes.py:43-66).  ``tsdf`` / ``weight`` are
  host mirrors: fetched on first access and, while a caller holds them, kept
  coherent both ways (uploaded before the next kernel reads the volume,
  refreshed in place after a kernel writes it), which reproduces the
  reference's shared-numpy-array behaviour.  The hot path never touches them.
* ``RayMap`` keeps distance / vertices / normals as device float64 tensors
  with the same mirror protocol.
* ``integrate`` / ``raycast`` accept one volume like the reference and
  ``integrate_volumes`` / ``raycast_volumes`` fuse many volumes into one
  launch; both give bit-identical results.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _native as nat
from .geometry import Array, CameraIntrinsics, DepthFrame, Pose


@dataclass(frozen=True)
class FusionParams:
    """Integration / raycast knobs shared by all subvolumes (tsdf.py:20-38)."""

    truncation: float
    max_weight: float = 128.0
    sample_weight: float = 1.0

    def __post_init__(self) -> None:
        if self.truncation <= 0:
            raise ValueError(f"truncation must be positive, got {self.truncation}")
        if self.max_weight < self.sample_weight or self.sample_weight <= 0:
            raise ValueError("weights must satisfy 0 < sample_weight <= max_weight")

    @classmethod
    def for_voxel_size(cls, voxel_size: float, truncation_scale: float = 4.0,
                       max_weight: float = 128.0, sample_weight: float = 1.0) -> "FusionParams":
        return cls(truncation=truncation_scale * voxel_size, max_weight=max_weight,
                   sample_weight=sample_weight)


class _Mirror:
    """Host copies of device tensors, coherent while handed out.

    ``fetch`` downloads once and marks the copies exposed; ``before_read``
    uploads exposed copies (a caller may have edited them) before a kernel
    reads the device data; ``after_write`` refreshes exposed copies in place
    after a kernel wrote the device data, or drops unexposed ones.
    """

    def __init__(self, download, upload) -> None:
        # the owner's bound methods, held weakly: a strong reference would make
        # owner -> mirror -> method -> owner a cycle, and a dropped volume's
        # device memory would then wait for the cyclic garbage collector
        self._download = weakref.WeakMethod(download)  # () -> dict[str, np.ndarray]
        self._upload = weakref.WeakMethod(upload)      # (dict) -> None
        self.host: dict | None = None
        self.exposed = False

    def fetch(self) -> dict:
        if self.host is None:
            self.host = self._download()()
        self.exposed = True
        return self.host

    def before_read(self) -> None:
        if self.exposed and self.host is not None:
            self._upload()(self.host)

    def after_write(self) -> None:
        if self.exposed and self.host is not None:
            fresh = self._download()()
            for k, v in fresh.items():
                np.copyto(self.host[k], v)
        else:
            self.host = None
            self.exposed = False

    def detach(self) -> None:
        """Forget host copies (after an upload that replaced the device data)."""
        self.host = None
        self.exposed = False


class TsdfSubvolume:
    """One dense TSDF grid on the global voxel lattice (tsdf.py:41-107).

    World position of local voxel (x, y, z) is
    ``voxel_size * (origin_voxel + (x, y, z))``; host arrays are [z, y, x].
    """

    def __init__(self, origin_voxel, voxels_per_side: int, side_length: float,
                 tsdf: Array | None = None, weight: Array | None = None, *,
                 voxels: torch.Tensor | None = None) -> None:
        origin = np.asarray(origin_voxel, dtype=np.int64)
        if origin.shape != (3,):
            raise ValueError("origin_voxel must be an integer 3-vector")
        if voxels_per_side < 2:
            raise ValueError("a subvolume needs at least 2 voxels per side")
        if side_length <= 0:
            raise ValueError("side_length must be positive")
        n = int(voxels_per_side)
        shape = (n, n, n)
        self.origin_voxel = origin
        self.voxels_per_side = n
        self.side_length = float(side_length)
        if voxels is not None:
            if tuple(voxels.shape) != shape + (2,) or voxels.dtype != torch.float32:
                raise ValueError(f"voxels must be float32 {shape + (2,)}")
            self.voxels = voxels.contiguous()
        else:
            if tsdf is None or weight is None:
                raise ValueError("give tsdf and weight arrays, or a voxels tensor")
            t = np.asarray(tsdf)
            w = np.asarray(weight)
            if t.shape != shape or w.shape != shape:
                raise ValueError(f"voxel arrays must have shape {shape}")
            pair = np.stack([t.astype(np.float32, copy=False), w.astype(np.float32, copy=False)], -1)
            self.voxels = torch.from_numpy(np.ascontiguousarray(pair)).to(nat.device())
        self._mirror = _Mirror(self._download, self._upload)
        # free-space brick summary (TfVolume.brick_state_dev): built lazily for a
        # truncation, kept exact by tf_integrate, dropped when the voxels are
        # replaced from the host
        self.brick_bad: torch.Tensor | None = None    # packed per-brick state
        self.brick_flags: torch.Tensor | None = None  # derived per-brick flags
        self._summary_t: float | None = None
        # optional colour (not in the reference): uint8 [n, n, n, 4] = (r, g, b, count)
        self.color: torch.Tensor | None = None
        # optional per-volume work counters (TfVolume.counters_dev, int64[2]:
        # general / free-space bricks swept), set by the multi-GPU ownership
        self.counters: torch.Tensor | None = None

    def enable_color(self) -> "TsdfSubvolume":
        """Give the volume a colour channel (all unobserved); returns it."""
        if self.color is None:
            n = self.voxels_per_side
            self.color = torch.zeros((n, n, n, 4), dtype=torch.uint8, device=self.voxels.device)
        return self

    def invalidate_summary(self) -> None:
        """Call after writing ``voxels`` directly (outside the package's kernels)."""
        self._summary_t = None

    # ---- host mirrors --------------------------------------------------------
    def _download(self) -> dict:
        pair = self.voxels.cpu().numpy()
        return {"tsdf": np.ascontiguousarray(pair[..., 0]),
                "weight": np.ascontiguousarray(pair[..., 1])}

    def _upload(self, host: dict) -> None:
        pair = np.stack([host["tsdf"], host["weight"]], -1).astype(np.float32, copy=False)
        self.voxels.copy_(torch.from_numpy(np.ascontiguousarray(pair)))

    @property
    def tsdf(self) -> Array:
        return self._mirror.fetch()["tsdf"]

    @property
    def weight(self) -> Array:
        return self._mirror.fetch()["weight"]

    def _device_read(self) -> None:
        if self._mirror.exposed and self._mirror.host is not None:
            self._summary_t = None  # host copies are about to be uploaded
        self._mirror.before_read()

    def _device_written(self) -> None:
        self._mirror.after_write()

    def _summary_for(self, tau: float) -> tuple[torch.Tensor, float]:
        L = nat.lib()
        thr = float(L.tf_good_threshold(float(tau)))
        if self._summary_t != thr:
            nb = (self.voxels_per_side + 7) // 8
            if self.brick_bad is None:
                self.brick_bad = torch.empty(nb ** 3, dtype=torch.int32, device=self.voxels.device)
                ns = (nb + 7) // 8  # superbrick flags follow the brick flags
                self.brick_flags = torch.empty(nb ** 3 + ns ** 3, dtype=torch.uint8,
                                               device=self.voxels.device)
            vol = nat.volume_struct(self.voxels, self.voxels_per_side, self.origin_voxel,
                                    self.voxel_size, self.brick_bad, self.brick_flags, thr)
            nat.check(L.tf_brick_summary(vol, nat.stream_handle()), "tf_brick_summary")
            self._summary_t = thr
        return self.brick_bad, thr

    # ---- reference API ---------------------------------------------------------
    @classmethod
    def empty(cls, origin_voxel, voxels_per_side: int, side_length: float) -> "TsdfSubvolume":
        n = int(voxels_per_side)
        if n < 2:
            raise ValueError("a subvolume needs at least 2 voxels per side")
        vox = torch.zeros((n, n, n, 2), dtype=torch.float32, device=nat.device())
        return cls(origin_voxel, n, side_length, voxels=vox)

    @property
    def voxel_size(self) -> float:
        return self.side_length / self.voxels_per_side

    @property
    def world_min(self) -> Array:
        return self.origin_voxel * self.voxel_size

    @property
    def world_max(self) -> Array:
        return (self.origin_voxel + self.voxels_per_side - 1) * self.voxel_size

    def payload_bytes(self) -> int:
        return self.voxels_per_side ** 3 * 8

    def observed_count(self) -> int:
        self._device_read()
        return int((self.voxels[..., 1] > 0).sum().item())

    def copy(self) -> "TsdfSubvolume":
        self._device_read()
        return TsdfSubvolume(self.origin_voxel.copy(), self.voxels_per_side, self.side_length,
                             voxels=self.voxels.clone())

    def native(self, tau: float | None = None) -> nat.TfVolume:
        """ABI descriptor; with ``tau`` it carries the brick summary for that truncation."""
        if tau is None:
            return nat.volume_struct(self.voxels, self.voxels_per_side, self.origin_voxel,
                                     self.voxel_size, color=self.color, counters=self.counters)
        bad, thr = self._summary_for(tau)
        return nat.volume_struct(self.voxels, self.voxels_per_side, self.origin_voxel,
                                 self.voxel_size, bad, self.brick_flags, thr, color=self.color,
                                 counters=self.counters)

    def __repr__(self) -> str:
        return (f"TsdfSubvolume(origin_voxel={self.origin_voxel!r}, "
                f"voxels_per_side={self.voxels_per_side}, side_length={self.side_length})")


# ---------------------------------------------------------------------------
# frames on the device
# ---------------------------------------------------------------------------

def device_depth(frame) -> torch.Tensor:
    """The frame's depth as a contiguous float64 device tensor (one H2D copy).

    Accepts a DepthFrame, a numpy array or an already-resident tensor (which
    is used as is).  Callers that process one frame many times (the pipeline)
    upload once and pass the tensor.
    """
    if isinstance(frame, torch.Tensor):
        # pinned host frames upload without blocking the host (stream-ordered;
        # torch's pinned allocator keeps the buffer alive until the copy ran)
        t = frame.to(device=nat.device(), dtype=torch.float64,
                     non_blocking=frame.device.type == "cpu" and frame.is_pinned())
        return t.contiguous()
    data = frame.data if isinstance(frame, DepthFrame) else np.asarray(frame, dtype=np.float64)
    host = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64))
    return host.to(nat.device())


def _vol_array(vols: Sequence[TsdfSubvolume], tau: float | None = None):
    arr = (nat.TfVolume * max(1, len(vols)))()
    for i, v in enumerate(vols):
        arr[i] = v.native(tau)
    return arr


# ---------------------------------------------------------------------------
# integration (tsdf.py:110-144)
# ---------------------------------------------------------------------------

def device_rgb(color, intr: CameraIntrinsics) -> torch.Tensor:
    """A colour frame (uint8 [H, W, 3], numpy or tensor) as a contiguous device tensor."""
    t = color if isinstance(color, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(color))
    if t.dtype != torch.uint8 or tuple(t.shape) != (intr.height, intr.width, 3):
        raise ValueError(f"colour frame must be uint8 {(intr.height, intr.width, 3)}")
    return t.to(nat.device()).contiguous()


def integrate_volumes(volumes: Sequence[TsdfSubvolume], frame, pose: Pose,
                      intr: CameraIntrinsics, params: FusionParams,
                      stats: torch.Tensor | None = None, color=None, *, phase: str = "all",
                      workspace_slot: str = "main") -> None:
    """Fuse one depth frame into every volume with one fused launch sequence.

    ``color`` (uint8 [H, W, 3]) is fused into the volumes that have a colour
    channel (``enable_color``): a running mean of the observations while the
    voxel lies in the truncation band (include/tfb200.h, tf_integrate_rgb).

    ``phase`` "prepare" then "finish" (same arguments, same
    ``workspace_slot``) split the call in two (tf_integrate_prepare /
    tf_integrate_finish), so the first half can run on another stream.
    """
    if phase not in ("all", "prepare", "finish"):
        raise ValueError(f"phase must be 'all', 'prepare' or 'finish', not {phase!r}")
    volumes = list(volumes)
    if not volumes:
        return
    depth = device_depth(frame)
    if tuple(depth.shape) != (intr.height, intr.width):
        raise ValueError("frame size does not match intrinsics")
    rgb = device_rgb(color, intr) if color is not None else None
    for v in volumes:
        v._device_read()
    inverse = pose.invert()
    arr = _vol_array(volumes, params.truncation)
    cam = nat.camera(intr)
    L = nat.lib()
    need = L.tf_integrate_workspace_size(arr, len(volumes), cam)
    ws = nat.workspace.get(need, workspace_slot)
    geom = (cam, nat.mat9(inverse.rotation), nat.vec3(inverse.translation), nat.vec3(pose.translation),
            float(params.truncation), float(params.max_weight), float(params.sample_weight),
            nat.ptr(ws), ws.numel())
    if phase == "prepare":
        nat.check(L.tf_integrate_prepare(arr, len(volumes), nat.ptr(depth), *geom, nat.stream_handle()),
                  "tf_integrate_prepare")
        return
    fn = L.tf_integrate_rgb if phase == "all" else L.tf_integrate_finish
    nat.check(fn(arr, len(volumes), nat.ptr(depth), nat.ptr(rgb) if rgb is not None else None, *geom,
                 nat.ptr(stats if stats is not None else nat.stats.buffer()), nat.stream_handle()),
              "tf_integrate")
    for v in volumes:
        v._device_written()


class SplitIntegrator:
    """integrate_volumes with its first half (pixel tables, depth mips,
    culling: tf_integrate_prepare) on a side stream, so it overlaps the tail
    of the previous frame's raycast; the second half (the voxel updates) runs
    on the current stream after it.  The side stream waits for the previous
    call's updates to release this integrator's own workspace and for the
    depth: ``depth_ready`` is an event after which the depth is valid, True
    when it has no pending producer (a resident frame), or None — then the
    whole call runs on the current stream (no overlap, no cross-stream
    synchronisation).  Results are those of integrate_volumes."""

    def __init__(self) -> None:
        self._prep = self._ws_free = self._prepared = None
        self._slot = f"split{id(self)}"

    def __call__(self, volumes: Sequence[TsdfSubvolume], depth, pose: Pose, intr: CameraIntrinsics,
                 params: FusionParams, stats: torch.Tensor | None = None, color=None,
                 depth_ready=None) -> None:
        volumes = list(volumes)
        if (depth_ready is None or not volumes or len(volumes) > nat.MAX_VOLUMES_PER_LAUNCH
                or not isinstance(depth, torch.Tensor) or not depth.is_cuda
                or any(v._mirror.exposed for v in volumes)):
            # nothing to overlap with, or a volume's host mirror is handed out
            # (its upload and summary rebuild must stay ordered after the
            # previous frame's raycast, which reads the same voxels): one call
            # on the current stream
            integrate_volumes(volumes, depth, pose, intr, params, stats, color=color)
            return
        main = torch.cuda.current_stream(depth.device)
        if self._prep is None:
            self._prep = torch.cuda.Stream(device=depth.device)
            self._ws_free, self._prepared = torch.cuda.Event(), torch.cuda.Event()
            self._ws_free.record(main)
        prep = self._prep
        # the workspace is (re)allocated here, on the current stream, and marked
        # as used by the side stream, so the caching allocator never hands a
        # block one of the two streams still uses to the other
        # brick summaries are (re)built here, on the current stream, so the
        # side stream only reads the depth, the volumes' geometry and its
        # own workspace
        arr = _vol_array(volumes, params.truncation)
        ws = nat.workspace.get(nat.lib().tf_integrate_workspace_size(arr, len(volumes), nat.camera(intr)),
                               self._slot)
        if depth_ready is not True:
            prep.wait_event(depth_ready)
        prep.wait_event(self._ws_free)
        with torch.cuda.stream(prep):
            integrate_volumes(volumes, depth, pose, intr, params, phase="prepare", workspace_slot=self._slot)
        ws.record_stream(prep)
        self._prepared.record(prep)
        main.wait_event(self._prepared)
        integrate_volumes(volumes, depth, pose, intr, params, stats, color=color, phase="finish",
                          workspace_slot=self._slot)
        self._ws_free.record(main)
        depth.record_stream(prep)


def integrate(subvolume: TsdfSubvolume, frame: DepthFrame, pose: Pose, intr: CameraIntrinsics,
              params: FusionParams, color=None) -> TsdfSubvolume:
    """Fuse one depth frame (and optionally its colour) into the subvolume in place; returns it."""
    data = frame.data if isinstance(frame, DepthFrame) else frame
    if tuple(data.shape) != (intr.height, intr.width):  # tsdf.py:124-125
        raise ValueError("frame size does not match intrinsics")
    integrate_volumes([subvolume], frame, pose, intr, params, color=color)
    return subvolume


def raycast_colors(volumes: Sequence[TsdfSubvolume], raymap: "RayMap", pose: Pose,
                   intr: CameraIntrinsics) -> torch.Tensor:
    """Colours (float32 [H, W, 3], device) of a ray map rendered from ``pose``:
    trilinear colour at each hit from the first listed volume with the hit
    cell's 8 corners coloured; 0 without a hit or colour (tf_raycast_colors)."""
    volumes = [v for v in volumes if v.color is not None]
    out = torch.zeros((intr.height, intr.width, 3), dtype=torch.float32, device=nat.device())
    if not volumes:
        return out
    raymap._device_read()
    arr = _vol_array(volumes)
    nat.check(nat.lib().tf_raycast_colors(arr, len(volumes), nat.camera(intr), nat.mat9(pose.rotation),
                                          nat.vec3(pose.translation), nat.ptr(raymap.distance_dev),
                                          nat.ptr(out), nat.stream_handle()), "tf_raycast_colors")
    return out


def trilinear_sample(subvolume: TsdfSubvolume, point: Array) -> float | None:
    """TSDF at a world point, or None where not fully observed (tsdf.py:147-153)."""
    subvolume._device_read()
    pts = torch.as_tensor(np.asarray(point, dtype=np.float64).reshape(1, 3), device=nat.device())
    vals = torch.empty(1, dtype=torch.float64, device=pts.device)
    ok = torch.empty(1, dtype=torch.uint8, device=pts.device)
    nat.check(nat.lib().tf_trilinear_sample(subvolume.native(), nat.ptr(pts), 1, nat.ptr(vals),
                                            nat.ptr(ok), nat.stream_handle()),
              "tf_trilinear_sample")
    return float(vals.item()) if bool(ok.item()) else None


# ---------------------------------------------------------------------------
# ray maps and raycast (tsdf.py:156-225)
# ---------------------------------------------------------------------------

class RayMap:
    """Per-pixel surface prediction merged across subvolumes (tsdf.py:156-190).

    ``distance`` is the Euclidean hit distance from the camera centre (+inf =
    no surface); vertices / normals are world-space.  Device tensors
    ``distance_dev`` [H, W] and ``vertices_dev`` / ``normals_dev`` [H, W, 3]
    are authoritative; the numpy attributes are coherent host mirrors.
    """

    def __init__(self, vertices=None, normals=None, distance=None, *,
                 device_tensors: tuple | None = None) -> None:
        if device_tensors is not None:
            self.vertices_dev, self.normals_dev, self.distance_dev = device_tensors
        else:
            dev = nat.device()
            self.vertices_dev = torch.as_tensor(np.ascontiguousarray(vertices, np.float64)).to(dev)
            self.normals_dev = torch.as_tensor(np.ascontiguousarray(normals, np.float64)).to(dev)
            self.distance_dev = torch.as_tensor(np.ascontiguousarray(distance, np.float64)).to(dev)
        self._mirror = _Mirror(self._download, self._upload)

    def _download(self) -> dict:
        return {"vertices": self.vertices_dev.cpu().numpy(),
                "normals": self.normals_dev.cpu().numpy(),
                "distance": self.distance_dev.cpu().numpy()}

    def _upload(self, host: dict) -> None:
        self.vertices_dev.copy_(torch.from_numpy(np.ascontiguousarray(host["vertices"])))
        self.normals_dev.copy_(torch.from_numpy(np.ascontiguousarray(host["normals"])))
        self.distance_dev.copy_(torch.from_numpy(np.ascontiguousarray(host["distance"])))

    @property
    def vertices(self) -> Array:
        return self._mirror.fetch()["vertices"]

    @property
    def normals(self) -> Array:
        return self._mirror.fetch()["normals"]

    @property
    def distance(self) -> Array:
        return self._mirror.fetch()["distance"]

    def _device_read(self) -> None:
        self._mirror.before_read()

    def _device_written(self) -> None:
        self._mirror.after_write()

    @classmethod
    def empty(cls, intr: CameraIntrinsics) -> "RayMap":
        dev = nat.device()
        h, w = intr.height, intr.width
        return cls(device_tensors=(
            torch.zeros((h, w, 3), dtype=torch.float64, device=dev),
            torch.zeros((h, w, 3), dtype=torch.float64, device=dev),
            torch.full((h, w), float("inf"), dtype=torch.float64, device=dev)))

    def reset(self) -> "RayMap":
        """Back to the empty state in place (no host round trip, one launch)."""
        d, v, n = self.distance_dev, self.vertices_dev, self.normals_dev
        if d.is_contiguous() and v.is_contiguous() and n.is_contiguous():
            nat.check(nat.lib().tf_raymap_reset(d.data_ptr(), v.data_ptr(), n.data_ptr(), d.numel(),
                                                nat.stream_handle()), "tf_raymap_reset")
        else:
            v.zero_()
            n.zero_()
            d.fill_(float("inf"))
        self._device_written()
        return self

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self.distance_dev.shape)

    @property
    def valid(self) -> Array:
        return np.isfinite(self.distance)

    def copy(self) -> "RayMap":
        self._device_read()
        return RayMap(device_tensors=(self.vertices_dev.clone(), self.normals_dev.clone(),
                                      self.distance_dev.clone()))

    def downsampled(self) -> "RayMap":
        self._device_read()
        return RayMap(device_tensors=(self.vertices_dev[::2, ::2].contiguous(),
                                      self.normals_dev[::2, ::2].contiguous(),
                                      self.distance_dev[::2, ::2].contiguous()))

    def merge_from(self, other: "RayMap") -> "RayMap":
        """_hit_wins merge of another map into this one (tsdf_raymap_merge)."""
        self._device_read()
        other._device_read()
        nat.check(nat.lib().tf_raymap_merge(
            nat.ptr(self.distance_dev), nat.ptr(self.vertices_dev), nat.ptr(self.normals_dev),
            nat.ptr(other.distance_dev), nat.ptr(other.vertices_dev), nat.ptr(other.normals_dev),
            self.distance_dev.numel(), nat.stream_handle()), "tf_raymap_merge")
        self._device_written()
        return self


def coarse_step(params: FusionParams, voxel_size: float) -> int:
    """Coarse march stride in fine lattice steps (tsdf.py:207)."""
    return max(2, int(round(0.5 * params.truncation / voxel_size)))


def raycast_volumes(volumes: Sequence[TsdfSubvolume], pose: Pose, intr: CameraIntrinsics,
                    raymap: RayMap, params: FusionParams,
                    stats: torch.Tensor | None = None, rows: tuple[int, int] | None = None,
                    fresh: bool = False) -> RayMap:
    """Render every volume into ``raymap`` with one fused launch.

    ``rows`` = (rank, world): trace only the 8-pixel block rows b with
    b % world == rank (tf_raycast_rows; the rest of the map is untouched).
    ``fresh``: render into an emptied map (``raymap.reset()`` + render) — the
    first launch writes every pixel instead of merging (TF_RAYCAST_FRESH),
    so the reset costs no launch.

    Volumes are grouped by coarse stride (the reference computes it per
    volume, tsdf.py:207); the merge is order-free so grouping is exact.
    """
    volumes = list(volumes)
    if tuple(raymap.shape) != (intr.height, intr.width):
        raise ValueError("raymap size does not match intrinsics")
    if not volumes:
        return raymap.reset() if fresh else raymap
    if fresh and rows is not None:
        raymap.reset()
        fresh = False
    if not fresh:
        raymap._device_read()
    for v in volumes:
        v._device_read()
    groups: dict[int, list[TsdfSubvolume]] = {}
    for v in volumes:
        groups.setdefault(coarse_step(params, v.voxel_size), []).append(v)
    cam = nat.camera(intr)
    r = nat.mat9(pose.rotation)
    c = nat.vec3(pose.translation)
    st = stats if stats is not None else nat.stats.buffer()
    L = nat.lib()
    stream = nat.stream_handle()
    for coarse, vols in groups.items():
        arr = _vol_array(vols, params.truncation)
        # the cooperative pass's scratch: one workspace per stream (launches on
        # a stream are ordered; two streams never share one)
        ws = nat.workspace.get(L.tf_raycast_workspace_size(len(vols), cam), f"raycast{stream}")
        if fresh:  # the first group writes every pixel; later groups merge into it
            nat.check(L.tf_raycast_ex(arr, len(vols), cam, float(params.truncation), int(coarse),
                                      r, c, nat.ptr(raymap.distance_dev),
                                      nat.ptr(raymap.vertices_dev), nat.ptr(raymap.normals_dev),
                                      nat.ptr(ws), ws.numel(), 1, 0, nat.RAYCAST_FRESH, nat.ptr(st), stream),
                      "tf_raycast_ex")
            fresh = False
        elif rows is None:
            nat.check(L.tf_raycast_ws(arr, len(vols), cam, float(params.truncation), int(coarse),
                                      r, c, nat.ptr(raymap.distance_dev),
                                      nat.ptr(raymap.vertices_dev), nat.ptr(raymap.normals_dev),
                                      nat.ptr(ws), ws.numel(), nat.ptr(st), stream), "tf_raycast_ws")
        else:
            nat.check(L.tf_raycast_rows(arr, len(vols), cam, float(params.truncation), int(coarse),
                                        r, c, nat.ptr(raymap.distance_dev),
                                        nat.ptr(raymap.vertices_dev), nat.ptr(raymap.normals_dev),
                                        nat.ptr(ws), ws.numel(), int(rows[1]), int(rows[0]), nat.ptr(st),
                                        stream), "tf_raycast_rows")
    raymap._device_written()
    return raymap


def raycast(subvolume: TsdfSubvolume, pose: Pose, intr: CameraIntrinsics, raymap: RayMap,
            params: FusionParams) -> RayMap:
    """Render the subvolume's zero surface into ``raymap`` (min-distance merge)."""
    return raycast_volumes([subvolume], pose, intr, raymap, params)


# ---------------------------------------------------------------------------
# point clouds (tsdf.py:228-280)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class PointCloud:
    """Vertices with unit normals, both (N, 3) float64 host arrays."""

    vertices: Array
    normals: Array

    def __post_init__(self) -> None:
        v = np.asarray(self.vertices, dtype=np.float64).reshape(-1, 3)
        n = np.asarray(self.normals, dtype=np.float64).reshape(-1, 3)
        if len(v) != len(n):
            raise ValueError("vertex and normal counts differ")
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "normals", n)

    def __len__(self) -> int:
        return len(self.vertices)

    @classmethod
    def empty(cls) -> "PointCloud":
        return cls(np.zeros((0, 3)), np.zeros((0, 3)))

    @classmethod
    def concatenate(cls, clouds: Iterable["PointCloud"]) -> "PointCloud":
        clouds = list(clouds)
        if not clouds:
            return cls.empty()
        return cls(np.concatenate([c.vertices for c in clouds]),
                   np.concatenate([c.normals for c in clouds]))


def extract_points_device(subvolume: TsdfSubvolume) -> tuple[torch.Tensor, torch.Tensor]:
    """Order-preserving extraction on the device -> (verts, norms) [N, 3]."""
    subvolume._device_read()
    L = nat.lib()
    vol = subvolume.native()
    need = L.tf_extract_workspace_size(subvolume.voxels_per_side)
    ws = nat.workspace.get(need, slot="extract")
    count = torch.zeros(1, dtype=torch.int64, device=nat.device())
    nat.check(L.tf_extract_count(vol, nat.ptr(ws), ws.numel(), nat.ptr(count),
                                 nat.stream_handle()), "tf_extract_count")
    n = int(count.item())
    verts = torch.empty((n, 3), dtype=torch.float64, device=count.device)
    norms = torch.empty((n, 3), dtype=torch.float64, device=count.device)
    if n:
        nat.check(L.tf_extract_emit(vol, nat.ptr(ws), ws.numel(), nat.ptr(verts), nat.ptr(norms),
                                    nat.stream_handle()), "tf_extract_emit")
    return verts, norms


def extract_points(subvolume: TsdfSubvolume) -> PointCloud:
    """One vertex per voxel straddling the zero surface (tsdf.py:261-280)."""
    verts, norms = extract_points_device(subvolume)
    return PointCloud(verts.cpu().numpy(), norms.cpu().numpy())
