"""Multi-GPU volume ownership: one process per GPU, torch.distributed (NCCL).

The paper's CPU<->GPU volume swapping becomes ownership:

* every active volume is owned by exactly one rank (``owned_keys``: contiguous
  chunks of a checkerboard "spread" order of the keys, deterministic and
  balanced by count, mixing busy and quiet regions of the map);
* each frame's depth is broadcast from rank 0 (``broadcast_frame``) and each
  rank integrates only its own volumes — integration has no data-path
  collective;
* each rank raycasts its volumes into a partial ray map; the partial maps are
  reduced by a row-block exchange: every rank packs its
  partial as (t, nx, ny, nz) records, an all-to-all gives rank r every
  rank's records of row block r, rank r folds them with the _hit_wins total
  order in rank order (tf_raymap_merge_packed), and an all-gather of the
  merged blocks gives every rank the full model; vertices are rebuilt from t
  with the raycast's own arithmetic (tf_raymap_vertices), so they are the
  bits the raycast wrote.  _hit_wins is a strict total order, so the result
  equals the single-GPU raycast over all volumes bit for bit (the
  reference's order-free invariant, test_acceptance.py:349-361).  Traffic
  per rank and frame: 2 x 32 B x pixels x (world - 1) / world.

On GPUs that can map each other's memory (NVLink / NVSwitch) the exchange,
the fold and the all-gather are one kernel per rank over peer memory
(``PeerExchange``, csrc/comm.cu): each rank's raycast writes its partial into
a region its peers have mapped, and the reduce kernel reads its row block of
every partial and stores the merged rows into every rank's model; the NCCL
row-block exchange above remains for ranks without peer access (and runs the
same host schedule on gloo in the CPU tests).

ICP runs replicated on every rank over the merged model (no per-iteration
collective).  The host-side schedule is backend-agnostic and is tested with
gloo on CPU (tests/test_distributed_cpu.py); the CUDA merge is tested on one
GPU.
"""

from __future__ import annotations

import ctypes
import weakref
from typing import Callable, Sequence

import torch
import torch.distributed as dist

from . import _native as nat
from .geometry import CameraIntrinsics, Pose
from .tsdf import (FusionParams, RayMap, SplitIntegrator, TsdfSubvolume, integrate_volumes,
                   raycast_volumes)


def owner_of(index: int, world: int) -> int:
    """Rank owning the index-th allocated volume (round-robin)."""
    return index % world


def spread_order(keys: Sequence) -> list:
    """Keys reordered so that contiguous chunks mix the regions of the map.

    Tiles of a scene are not equally busy (a floor, an object fill some of
    them), and neighbours tend to be alike; chunking keys in checkerboard order
    (parity of the tile's grid coordinates, then x, y, z) gives every rank a
    spread of the map: with the 2x2x2 grid of config 3, 2 ranks each get one
    tile of every (y, z) row and 4 ranks each get one tile per y and per z
    layer, instead of whole layers.
    """
    keys = list(keys)
    if not all(isinstance(k, tuple) and len(k) == 3 for k in keys):
        return keys  # not grid keys: allocation order
    axes = [sorted({k[a] for k in keys}) for a in range(3)]
    grid = [tuple(axes[a].index(k[a]) for a in range(3)) for k in keys]
    order = sorted(range(len(keys)), key=lambda i: (sum(grid[i]) % 2, grid[i]))
    return [keys[i] for i in order]


def owned_keys(keys: Sequence, rank: int, world: int) -> list:
    """This rank's keys: a contiguous chunk of the spread order, in allocation order."""
    spread = spread_order(keys)
    n = len(spread)
    mine = {spread[i] for i in range(n) if i * world // n == rank} if n else set()
    return [k for k in keys if k in mine]


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


def row_block(height: int, world: int) -> int:
    """Rows per block of the row-block exchange (the last block is padded)."""
    return -(-height // world)


def rowblock_exchange(packed: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-to-all of packed partial records [world * B, W, 4] (rows padded to
    world * B); returns [world, B, W, 4]: every rank's records of this rank's
    row block, in rank order."""
    if world == 1:
        return packed.view(1, *packed.shape)
    recv = torch.empty_like(packed)
    dist.all_to_all_single(recv, packed.contiguous(), group=group)
    return recv.view(world, packed.shape[0] // world, *packed.shape[1:])


def merge_blocks(blocks: torch.Tensor, merge: Callable) -> torch.Tensor:
    """Fold the ranks' records of one row block in rank order (merge(acc, other))."""
    acc = blocks[0].clone()
    for r in range(1, blocks.shape[0]):
        merge(acc, blocks[r])
    return acc


def gather_blocks(block: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather of every rank's merged block -> [world * B, W, 4]."""
    if world == 1:
        return block
    out = torch.empty((world,) + tuple(block.shape), dtype=block.dtype, device=block.device)
    dist.all_gather(list(out.unbind(0)), block.contiguous(), group=group)
    return out.view(world * block.shape[0], *block.shape[1:])


def merge_packed_cuda(acc: torch.Tensor, other: torch.Tensor) -> None:
    nat.check(nat.lib().tf_raymap_merge_packed(nat.ptr(acc), nat.ptr(other), acc.numel() // 4,
                                               nat.stream_handle()), "tf_raymap_merge_packed")


def exchange_handles(handle: bytes, world: int, group=None) -> list[bytes]:
    """All-gather of every rank's IPC handle bytes, in rank order (host plumbing)."""
    if world == 1:
        return [handle]
    out: list = [None] * world
    dist.all_gather_object(out, handle, group=group)
    return out


def peer_exchange_supported(world: int, group=None) -> bool:
    """True when every rank sits on its own CUDA device and every pair of
    those devices can map each other's memory (one node, NVLink / NVSwitch)."""
    if world == 1 or not torch.cuda.is_available():
        return False
    mine = torch.cuda.current_device()
    devs: list = [None] * world
    dist.all_gather_object(devs, mine, group=group)
    ok = len(set(devs)) == world and all(
        torch.cuda.can_device_access_peer(mine, d) for d in devs if d != mine)
    oks: list = [None] * world
    dist.all_gather_object(oks, bool(ok), group=group)
    return all(oks)


class _RegionView:
    """CUDA array interface over a section of a comm region (float64); keeps
    the owning PeerExchange alive while any tensor views it."""

    def __init__(self, address: int, shape: tuple, owner) -> None:
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                         "data": (address, False), "version": 2,
                                         "strides": None}
        self._owner = owner


class PeerExchange:
    """Peer-memory ray-map reduction across the ranks' GPUs (csrc/comm.cu).

    ``partial`` is the RayMap this rank's raycast writes (in the region its
    peers map); after ``reduce()`` every rank's ``model`` holds the merged map,
    equal bit for bit to the single-GPU raycast over all volumes.
    ``connect()`` maps the peers' regions (IPC handles all-gathered over the
    process group).  ``link_local`` wires emulated ranks of one process on one
    device instead (tests; their reductions run with ``nowait=True``).
    """

    def __init__(self, intr: CameraIntrinsics, rank: int, world: int) -> None:
        lib = nat.lib()
        h = ctypes.c_void_p()
        nat.check(lib.tf_comm_create(rank, world, intr.width, intr.height, ctypes.byref(h)),
                  "tf_comm_create")
        self._h = h
        weakref.finalize(self, lib.tf_comm_destroy, ctypes.c_void_p(h.value))
        self.rank, self.world = rank, world
        base = ctypes.c_void_p()
        offs = (ctypes.c_int64 * nat.COMM_NSECTIONS)()
        nat.check(lib.tf_comm_layout(h, ctypes.byref(base), offs), "tf_comm_layout")
        dev = nat.device()
        hh, ww = intr.height, intr.width

        def view(sec: int, shape: tuple) -> torch.Tensor:
            return torch.as_tensor(_RegionView(base.value + offs[sec], shape, self), device=dev)

        self.partial = RayMap(device_tensors=(view(nat.COMM_PART_VERT, (hh, ww, 3)),
                                              view(nat.COMM_PART_NORM, (hh, ww, 3)),
                                              view(nat.COMM_PART_DIST, (hh, ww))))
        self.model = RayMap(device_tensors=(view(nat.COMM_MODEL_VERT, (hh, ww, 3)),
                                            view(nat.COMM_MODEL_NORM, (hh, ww, 3)),
                                            view(nat.COMM_MODEL_DIST, (hh, ww))))

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(nat.COMM_HANDLE_BYTES)
        nat.check(nat.lib().tf_comm_export(self._h, buf), "tf_comm_export")
        return buf.raw

    def connect(self, group=None) -> None:
        handles = exchange_handles(self.export(), self.world, group)
        nat.check(nat.lib().tf_comm_import(self._h, b"".join(handles)), "tf_comm_import")

    @staticmethod
    def link_local(exchanges: Sequence["PeerExchange"]) -> None:
        arr = (ctypes.c_void_p * len(exchanges))(*[e._h.value for e in exchanges])
        nat.check(nat.lib().tf_comm_link_local(arr, len(exchanges)), "tf_comm_link_local")

    def reduce(self, nowait: bool = False) -> RayMap:
        # a wait that timed out leaves the flag raised for good and every later
        # wait returns at once, so the merged maps would be folded unsynchronised:
        # surface it on the next frame (the flag copy of the last completed
        # reduction, no host synchronisation)
        if self.poll_error():
            raise RuntimeError("peer-memory ray-map reduction: a flag wait timed out "
                               "(a peer stopped or its GPU is unreachable)")
        nat.check(nat.lib().tf_comm_reduce_raymap(self._h, nat.COMM_NOWAIT if nowait else 0,
                                                  nat.stream_handle()), "tf_comm_reduce_raymap")
        self.model._device_written()
        return self.model

    def poll_error(self) -> int:
        """The error flag as of the last completed reduction (non-blocking)."""
        e = ctypes.c_int()
        nat.check(nat.lib().tf_comm_error_poll(self._h, ctypes.byref(e)), "tf_comm_error_poll")
        return e.value

    def error(self) -> int:
        """1 when a flag wait timed out (synchronous read)."""
        e = ctypes.c_int()
        nat.check(nat.lib().tf_comm_error(self._h, ctypes.byref(e)), "tf_comm_error")
        return e.value


def _connect_peers(intr: CameraIntrinsics, rank: int, world: int, group, required: bool):
    """Every rank's PeerExchange, mapped to every peer — or None on every rank
    when any rank could not create, export or map a region (the ranks agree
    through two all-gathers, so none is left waiting in a collective)."""
    pe, handle = None, None
    try:
        pe = PeerExchange(intr, rank, world)
        handle = pe.export()
    except RuntimeError:
        pe = None
    handles = exchange_handles(handle, world, group)
    ok = pe is not None and all(h is not None for h in handles)
    if ok:
        try:
            nat.check(nat.lib().tf_comm_import(pe._h, b"".join(handles)), "tf_comm_import")
        except RuntimeError:
            ok = False
    oks: list = [None] * world
    dist.all_gather_object(oks, ok, group=group)
    if all(oks):
        return pe
    if required:
        raise RuntimeError("peer-memory exchange requested but a rank could not map its peers")
    return None


# ---------------------------------------------------------------------------
# re-tiling and load-balanced ownership (hard part 4)
# ---------------------------------------------------------------------------

def valid_retile(voxels_per_side: int, k: int) -> bool:
    """A tile of n voxels splits into k^3 cubic sub-tiles with the reference's
    2-voxel overlap iff k divides n - 2 (spacing (n - 2) / k, size spacing + 2)."""
    return k >= 1 and (voxels_per_side - 2) % k == 0 and (voxels_per_side - 2) // k >= 2


def default_retile(world: int, voxels_per_side: int = 512) -> int:
    """Sub-tiles per axis at ``world`` ranks: none on one GPU; enough that the
    sub-tiles outnumber the ranks several times over (k^3 >= 4 world per tile
    group of 8) — the largest valid k <= the target."""
    if world <= 1:
        return 1
    target = 2 if world <= 4 else 3
    for k in range(target, 0, -1):
        if valid_retile(voxels_per_side, k):
            return k
    return 1


def retile(keys: Sequence, voxels_per_side: int, voxel_size: float, k: int) -> tuple[list, int]:
    """Split every tile into k^3 sub-tiles with a 2-voxel overlap.

    Tile ``key`` (origin voxel o, n voxels per side, volumes.py:117-153)
    covers global voxels o .. o + n - 1; sub-tile (i, j, l) covers
    o + (i, j, l) * s .. + s + 1 with s = (n - 2) / k, so neighbours share two
    voxel layers exactly like the reference's tiles (_kernels.py:8-14) and
    the union is the tile.  Every voxel's update depends only on its global
    lattice coordinate (_kernels.py:99-133), so each sub-tile's voxels equal
    the tile's bit for bit; the merged raycast of the sub-tiles moves by the
    rounding of the local coordinates only.  Returns
    (sub-tile keys in tile order, sub-tile voxels per side)."""
    n = int(voxels_per_side)
    if k == 1:
        return [tuple(int(x) for x in key) for key in keys], n
    if not valid_retile(n, k):
        raise ValueError(f"cannot split {n}-voxel tiles into {k}^3 sub-tiles with a 2-voxel overlap")
    s = (n - 2) // k
    m = s + 2
    if (m * voxel_size) / m != voxel_size:
        raise ValueError("sub-tile side length does not round-trip the voxel size")
    out = []
    for key in keys:
        o = [int(x) for x in key]
        for i in range(k):
            for j in range(k):
                for l in range(k):
                    out.append((o[0] + i * s, o[1] + j * s, o[2] + l * s))
    return out, m


_retile = retile  # ShardedFusion's keyword argument shadows the name


def balanced_owners(costs: Sequence[float], world: int, current: Sequence[int] | None = None,
                    slack: float = 0.05) -> list[int]:
    """Sticky longest-processing-time assignment of units to ranks.

    Units in decreasing cost (ties: lower index first) go to the least-loaded
    rank (ties: lower rank), except that a unit stays with its current owner
    while that owner's load after taking it stays within ``slack`` x the mean
    load of the least-loaded choice — so a balanced assignment is kept and a
    rebalance moves few units.  Deterministic: every rank computes the same
    result from the same (all-reduced) costs."""
    nunits = len(costs)
    if world <= 1:
        return [0] * nunits
    load = [0.0] * world
    owner = [0] * nunits
    mean = sum(costs) / world if nunits else 0.0
    for u in sorted(range(nunits), key=lambda i: (-costs[i], i)):
        best = min(range(world), key=lambda r: (load[r], r))
        r = best
        if current is not None:
            c = current[u]
            if load[c] + costs[u] <= load[best] + costs[u] + slack * mean:
                r = c
        owner[u] = r
        load[r] += costs[u]
    return owner


def initial_owners(keys: Sequence, world: int) -> list[int]:
    """Owners before any work was measured: contiguous chunks of the
    checkerboard spread order (spread_order)."""
    spread = spread_order(keys)
    pos = {k: i for i, k in enumerate(spread)}
    n = len(keys)
    return [pos[k] * world // n for k in keys] if n else []


def move_units(moves: Sequence[tuple], rank: int, payloads: dict, alloc: Callable,
               group=None) -> dict:
    """Point-to-point moves of whole units between ranks (collective over the
    ranks that take part).  ``moves`` = [(unit, src, dst)] in the same order
    on every rank; ``payloads[unit]`` = the tensors this rank sends (src ==
    rank); ``alloc(unit)`` = empty tensors of the same shapes for a unit it
    receives (dst == rank).  Returns {unit: received tensors}.  NCCL moves
    device tensors directly (NVLink); gloo has no device send / recv, so the
    tensors go through host memory there."""
    staged = dist.get_backend(group) == "gloo"
    ops, out, host_in = [], {}, {}
    for u, a, b in moves:
        if a == b:
            continue
        if rank == a:
            for t in payloads[u]:
                t = t.contiguous()
                ops.append(dist.P2POp(dist.isend, t.cpu() if staged else t, b, group=group))
        elif rank == b:
            bufs = alloc(u)
            out[u] = bufs
            host_in[u] = [t.new_empty(t.shape, device="cpu") if staged else t for t in bufs]
            for t in host_in[u]:
                ops.append(dist.P2POp(dist.irecv, t, a, group=group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if staged:
        for u, bufs in out.items():
            for dev_t, host_t in zip(bufs, host_in[u]):
                dev_t.copy_(host_t)
    return out


def fits_replicated(ntiles: int, voxels_per_side: int, color: bool = False, share: float = 0.4) -> bool:
    """Whether every rank can hold the whole map: its voxels (8 B, + 4 B of
    colour) within ``share`` of this GPU's memory."""
    per = 8 + (4 if color else 0)
    need = ntiles * voxels_per_side ** 3 * per
    total = torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory
    return need <= share * total


WORK_GENERAL_BRICK = 4.0  # relative cost of a general brick vs a certified free-space one


class ShardedFusion:
    """The per-rank slice of a static multi-volume map.

    The map's tiles are split into ``retile``^3 sub-tiles each (``retile``;
    1 keeps the tiles), and every sub-tile is owned by one rank.
    ``step(depth, pose)`` integrates this rank's sub-tiles, raycasts them
    into a partial map and merges all ranks' partials into ``model`` on
    every rank: over peer memory (``exchange="p2p"``, one kernel, the
    default when every pair of the ranks' GPUs can map each other) or with
    the NCCL row-block exchange (``exchange="collective"``).

    Ownership follows the work: the culling stage counts, per sub-tile, the
    bricks it sweeps (TfVolume.counters_dev); every ``rebalance_every``
    frames the counts are all-reduced, ``balanced_owners`` recomputes the
    assignment (sticky LPT) and the sub-tiles that change owner move between
    GPUs (NCCL send / recv of their voxels).  Integration has no data-path
    collective; a migration moves 8 B per voxel of the moved sub-tiles.
    """

    MODES = ("auto", "volumes", "replicated")

    def __init__(self, keys: Sequence, voxels_per_side: int, side_length: float,
                 params: FusionParams, intr: CameraIntrinsics, rank: int = 0, world: int = 1,
                 group=None, color: bool = False, exchange: str = "auto", retile: int = 1,
                 rebalance_every: int = 8, mode: str = "volumes") -> None:
        if exchange not in ("auto", "p2p", "collective"):
            raise ValueError(f"exchange must be 'auto', 'p2p' or 'collective', not {exchange!r}")
        if mode not in self.MODES:
            raise ValueError(f"mode must be one of {self.MODES}, not {mode!r}")
        self.rank, self.world, self.group = rank, world, group
        self.params, self.intr = params, intr
        self.parent_keys = [tuple(int(x) for x in k) for k in keys]
        vs = side_length / voxels_per_side
        self.voxel_size = vs
        if mode == "auto":
            mode = "replicated" if world > 1 and fits_replicated(len(keys), voxels_per_side, color) else "volumes"
        # replicated: every rank holds and integrates every tile and traces
        # 1/world of the image rows over all of them — each pixel is traced
        # over every volume by exactly one rank, so the merged model is the
        # single-GPU one bit for bit (and occluded volumes are skipped as on
        # one GPU); volumes: the tiles, re-tiled, are owned by the ranks
        self.mode = mode if world > 1 else "volumes"
        self.replicated = self.mode == "replicated"
        if self.replicated:
            retile = 1
        self.units, self.unit_n = _retile(self.parent_keys, voxels_per_side, vs, retile)
        self.retile_k = retile
        self.color = color
        self.owner = [rank] * len(self.units) if self.replicated else initial_owners(self.units, world)
        self.rebalance_every = rebalance_every if world > 1 and not self.replicated else 0
        self._dev = torch.device("cuda", torch.cuda.current_device())
        self._tiles: dict[int, TsdfSubvolume] = {}
        # per-unit work counters (general, free bricks), one row per unit
        self._counters = torch.zeros((len(self.units), 2), dtype=torch.int64, device=self._dev)
        for u in range(len(self.units)):
            if self.owner[u] == rank:
                self._tiles[u] = self._new_tile(u)
        self._refresh()
        self.partial = RayMap.empty(intr)
        self.model = RayMap.empty(intr)
        self.stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device=self._dev)
        # row-block exchange buffer: (t, n) records, rows padded to world * B; the
        # padding rows stay "no hit"
        b = row_block(intr.height, world)
        self._packed = torch.zeros((world * b, intr.width, 4), dtype=torch.float64, device=self._dev)
        self._packed[..., 0] = float("inf")
        self._integrator = SplitIntegrator()
        self.exchange = "none" if world == 1 else exchange
        self._peer = None
        if exchange == "auto" and world > 1:
            self.exchange = "p2p" if peer_exchange_supported(world, group) else "collective"
        if self.exchange == "p2p":
            self._peer = _connect_peers(intr, rank, world, group, required=exchange == "p2p")
            if self._peer is None:
                self.exchange = "collective"
            else:
                self.partial, self.model = self._peer.partial, self._peer.model
        self.frames = 0
        self.migrations = 0
        self._last_costs: list[float] | None = None

    # ---- ownership -------------------------------------------------------------
    def _new_tile(self, u: int, voxels: torch.Tensor | None = None) -> TsdfSubvolume:
        side = self.unit_n * self.voxel_size
        t = (TsdfSubvolume.empty(self.units[u], self.unit_n, side) if voxels is None
             else TsdfSubvolume(self.units[u], self.unit_n, side, voxels=voxels))
        if self.color and t.color is None:
            t.enable_color()
        t.counters = self._counters[u]
        return t

    def _refresh(self) -> None:
        self.keys = [self.units[u] for u in sorted(self._tiles)]
        self.tiles = [self._tiles[u] for u in sorted(self._tiles)]

    def unit_costs(self) -> list[float]:
        """Work per unit since the last rebalance, summed over ranks (collective)."""
        c = self._counters.to(torch.float64)
        cost = c[:, 0] * WORK_GENERAL_BRICK + c[:, 1]
        if self.world > 1:
            dist.all_reduce(cost, op=dist.ReduceOp.SUM, group=self.group)
        return cost.cpu().tolist()

    def rebalance(self) -> int:
        """Recompute the owners from the measured work and migrate; returns
        the number of units that moved.  Collective: every rank calls it."""
        costs = self.unit_costs()
        self._last_costs = costs
        new = balanced_owners(costs, self.world, self.owner)
        moved = self.migrate(new)
        self._counters.zero_()
        return moved

    def migrate(self, new_owner: Sequence[int]) -> int:
        """Move every unit whose owner changes (move_units: NCCL send / recv
        of its voxels, and colours); collective."""
        moves = [(u, self.owner[u], new_owner[u]) for u in range(len(self.units))
                 if self.owner[u] != new_owner[u]]
        if not moves:
            return 0
        payloads = {}
        for u, a, _ in moves:
            if a == self.rank:
                t = self._tiles.pop(u)
                t._device_read()
                payloads[u] = [t.voxels] + ([t.color] if self.color else [])
        n = self.unit_n

        def alloc(u):
            bufs = [torch.empty((n, n, n, 2), dtype=torch.float32, device=self._dev)]
            if self.color:
                bufs.append(torch.empty((n, n, n, 4), dtype=torch.uint8, device=self._dev))
            return bufs

        got = move_units(moves, self.rank, payloads, alloc, self.group)
        for u, bufs in got.items():
            t = self._new_tile(u, bufs[0])
            if self.color:
                t.color = bufs[1]
            self._tiles[u] = t
        self.owner = list(new_owner)
        self._refresh()
        self.migrations += len(moves)
        return len(moves)

    # ---- dynamic placement (whole tiles, retile 1) --------------------------------
    def add_unit(self, key) -> None:
        """Allocate a tile (replicated decision, every rank calls it): owned by
        the rank with the fewest units (ties: lowest rank)."""
        if self.retile_k != 1:
            raise ValueError("dynamic tiles are not re-tiled")
        key = tuple(int(x) for x in key)
        counts = [self.owner.count(r) for r in range(self.world)]
        r = self.rank if self.replicated else min(range(self.world), key=lambda q: (counts[q], q))
        self.units.append(key)
        self.owner.append(r)
        c = torch.zeros((len(self.units), 2), dtype=torch.int64, device=self._dev)
        c[:-1] = self._counters
        self._counters = c
        for u, t in self._tiles.items():
            t.counters = self._counters[u]
        if r == self.rank:
            self._tiles[len(self.units) - 1] = self._new_tile(len(self.units) - 1)
        self._refresh()

    def remove_unit(self, key) -> TsdfSubvolume | None:
        """Retire a tile (every rank calls it); returns it on its owner."""
        key = tuple(int(x) for x in key)
        u = self.units.index(key)
        tile = self._tiles.pop(u, None)
        keep = [i for i in range(len(self.units)) if i != u]
        self.units = [self.units[i] for i in keep]
        self.owner = [self.owner[i] for i in keep]
        self._counters = self._counters[keep].clone()
        self._tiles = {keep.index(i): t for i, t in self._tiles.items()}
        for i, t in self._tiles.items():
            t.counters = self._counters[i]
        if tile is not None:
            tile.counters = None
        self._refresh()
        return tile

    def balance_report(self) -> dict:
        """Per-rank share of the last measured work (collective)."""
        if self.replicated:
            return {"mode": "replicated", "tiles": len(self.units),
                    "rows": f"block rows b with b % {self.world} == rank (8-pixel rows)"}
        costs = self._last_costs if self._last_costs is not None else self.unit_costs()
        load = [0.0] * self.world
        for u, c in enumerate(costs):
            load[self.owner[u]] += c
        mean = sum(load) / self.world if self.world else 0.0
        return {"units": len(self.units), "unit_voxels_per_side": self.unit_n,
                "retile": self.retile_k, "rebalance_every": self.rebalance_every,
                "load_per_rank": load, "imbalance_max_over_mean": (max(load) / mean) if mean else None,
                "units_per_rank": [self.owner.count(r) for r in range(self.world)],
                "migrations": self.migrations,
                "work_measure": f"bricks swept per unit (general x {WORK_GENERAL_BRICK:g} + free-space)"}

    def check_exchange(self) -> None:
        if self._peer is not None and self._peer.error():
            raise RuntimeError("peer-memory ray-map reduction: a flag wait timed out")

    # ---- one frame ---------------------------------------------------------------
    def step(self, depth: torch.Tensor, pose: Pose, color=None, depth_ready=None) -> RayMap:
        """One frame.  ``depth_ready`` (see SplitIntegrator): an event after
        which ``depth`` is valid, True for a frame with no pending producer,
        or None (the integration's first half then waits for the stream)."""
        if self.rebalance_every and self.frames and self.frames % self.rebalance_every == 0:
            self.rebalance()
        self.frames += 1
        self._integrator(self.tiles, depth, pose, self.intr, self.params, self.stats, color=color,
                         depth_ready=depth_ready)
        raycast_volumes(self.tiles, pose, self.intr, self.partial, self.params, self.stats,
                        rows=(self.rank, self.world) if self.replicated else None, fresh=True)
        if self.world == 1:
            self.model, self.partial = self.partial, self.model
            return self.model
        return self.reduce(pose)

    def reduce(self, pose: Pose) -> RayMap:
        """Merge every rank's partial into ``model`` on every rank (collective)."""
        if self._peer is not None:
            return self._peer.reduce()
        h, w = self.intr.height, self.intr.width
        packed = self._packed
        packed[:h, :, 0] = self.partial.distance_dev
        packed[:h, :, 1:] = self.partial.normals_dev
        blocks = rowblock_exchange(packed, self.world, self.group)
        merged = gather_blocks(merge_blocks(blocks, merge_packed_cuda), self.world, self.group)
        self.model.distance_dev.copy_(merged[:h, :, 0])
        self.model.normals_dev.copy_(merged[:h, :, 1:])
        nat.check(nat.lib().tf_raymap_vertices(
            nat.ptr(self.model.distance_dev), 1, nat.ptr(self.model.vertices_dev), nat.camera(self.intr),
            nat.mat9(pose.rotation), nat.vec3(pose.translation), 0, h, nat.stream_handle()),
            "tf_raymap_vertices")
        self.model._device_written()
        return self.model
