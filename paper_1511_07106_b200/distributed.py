"""Multi-GPU volume ownership: one process per GPU, torch.distributed (NCCL).

The paper's CPU<->GPU volume swapping becomes ownership:

* every active volume is owned by exactly one rank (``owner_of``: the i-th
  allocated key goes to rank i mod world, deterministic and balanced by
  count);
* each frame's depth is broadcast from rank 0 (``broadcast_frame``) and each
  rank integrates only its own volumes — integration has no data-path
  collective;
* each rank raycasts its volumes into a partial ray map; the partial maps are
  all-gathered and merged with the _hit_wins total order (tf_raymap_merge),
  in rank order, so every rank holds the identical full model.  _hit_wins is
  a strict total order, so the result equals the single-GPU raycast over all
  volumes bit for bit (the reference's order-free invariant,
  test_acceptance.py:349-361).

ICP runs replicated on every rank over the merged model (no per-iteration
collective).  The host-side schedule is backend-agnostic and is tested with
gloo on CPU (tests/test_distributed_cpu.py); the CUDA merge is tested on one
GPU.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist

from . import _native as nat
from .geometry import CameraIntrinsics, Pose
from .tsdf import FusionParams, RayMap, TsdfSubvolume, integrate_volumes, raycast_volumes


def owner_of(index: int, world: int) -> int:
    """Rank owning the index-th allocated volume."""
    return index % world


def owned_keys(keys: Sequence, rank: int, world: int) -> list:
    return [k for i, k in enumerate(keys) if owner_of(i, world) == rank]


def broadcast_frame(depth: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Frame broadcast from ``src`` (NCCL over NVLink on GPUs)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(depth, src=src, group=group)
    return depth


def gather_partials(parts: Sequence[torch.Tensor], group=None) -> list[list[torch.Tensor]]:
    """All-gather each tensor of this rank's partial map -> [rank][part]."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return [list(parts)]
    out = [[torch.empty_like(p) for p in parts] for _ in range(world)]
    for i, p in enumerate(parts):
        dist.all_gather([out[r][i] for r in range(world)], p.contiguous(), group=group)
    return out


def merge_in_rank_order(gathered: list, merge: Callable) -> list:
    """Fold rank r's partial into the running result for r = 1..world-1."""
    acc = [t.clone() for t in gathered[0]]
    for r in range(1, len(gathered)):
        merge(acc, gathered[r])
    return acc


class ShardedFusion:
    """The per-rank slice of a static multi-volume map.

    ``step(depth, pose)`` integrates this rank's volumes, raycasts them into a
    partial map and merges all ranks' partials into ``model`` on every rank.
    """

    def __init__(self, keys: Sequence, voxels_per_side: int, side_length: float,
                 params: FusionParams, intr: CameraIntrinsics, rank: int = 0, world: int = 1,
                 group=None) -> None:
        self.rank, self.world, self.group = rank, world, group
        self.params, self.intr = params, intr
        self.keys = owned_keys(keys, rank, world)
        self.tiles = [TsdfSubvolume.empty(k, voxels_per_side, side_length) for k in self.keys]
        self.partial = RayMap.empty(intr)
        self.model = RayMap.empty(intr)
        self.stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device=self.partial.distance_dev.device)

    def step(self, depth: torch.Tensor, pose: Pose) -> RayMap:
        integrate_volumes(self.tiles, depth, pose, self.intr, self.params, self.stats)
        self.partial.reset()
        raycast_volumes(self.tiles, pose, self.intr, self.partial, self.params, self.stats)
        if self.world == 1:
            self.model, self.partial = self.partial, self.model
            return self.model
        parts = [self.partial.distance_dev, self.partial.vertices_dev, self.partial.normals_dev]
        gathered = gather_partials(parts, self.group)

        def merge(acc, other):
            dst = RayMap(device_tensors=(acc[1], acc[2], acc[0]))
            dst.merge_from(RayMap(device_tensors=(other[1], other[2], other[0])))

        d, v, n = merge_in_rank_order(gathered, merge)
        self.model = RayMap(device_tensors=(v, n, d))
        return self.model
