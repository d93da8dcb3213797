"""Multi-GPU host schedule on CPU: world size 2 over gloo (127.0.0.1).

Covers the parts of distributed.py that are backend-agnostic: volume
ownership, the rank-0 frame broadcast, the all-gather of partial ray maps
and their rank-order _hit_wins merge.  The merge operator here is a numpy
restatement of _hit_wins (_kernels.py:246-263); on GPUs the same schedule
calls tf_raymap_merge.  The merged map must equal a single-process merge of
all partials in any order (the reference's order-free invariant).
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1511_07106_b200.distributed import (broadcast_frame, gather_blocks, gather_partials,
                                               merge_blocks, merge_in_rank_order, owned_keys,
                                               owner_of, row_block, rowblock_exchange)


def hit_wins_merge(acc, other):
    """_hit_wins applied per pixel: acc = (dist, vert, norm) tensors, in place."""
    d0, v0, n0 = acc
    d1, v1, n1 = other
    better = d1 < d0
    tie = d1 == d0
    for a in range(3):
        neq = n1[..., a] != n0[..., a]
        better = better | (tie & neq & (n1[..., a] > n0[..., a]))
        tie = tie & ~neq
    d0[better] = d1[better]
    v0[better] = v1[better]
    n0[better] = n1[better]


def partial_map(seed, h=12, w=16):
    """A physically consistent partial map: the hit vertex is distance x the
    pixel's ray; distances are coarse so exact ties (broken by normals) occur."""
    g = torch.Generator().manual_seed(seed)
    d = torch.where(torch.rand(h, w, generator=g) < 0.5, torch.full((h, w), float("inf")),
                    torch.round(torch.rand(h, w, generator=g) * 8) / 8 + 1.0).double()
    hit = torch.isfinite(d)
    ray = torch.stack(torch.meshgrid(torch.arange(h), torch.arange(w), indexing="ij") +
                      (torch.ones(h, w, dtype=torch.long),), -1).double()
    v = torch.where(hit[..., None], d[..., None] * ray, torch.zeros(()).double())
    n = torch.round(torch.rand(h, w, 3, generator=g) * 4).double() / 4  # ties happen
    n = torch.where(hit[..., None], n, torch.zeros(()).double())
    return [d, v, n]


def hit_wins_packed(acc, other):
    """_hit_wins on (t, nx, ny, nz) records, in place (tf_raymap_merge_packed)."""
    better = other[..., 0] < acc[..., 0]
    tie = other[..., 0] == acc[..., 0]
    for a in range(1, 4):
        neq = other[..., a] != acc[..., a]
        better = better | (tie & neq & (other[..., a] > acc[..., a]))
        tie = tie & ~neq
    acc[better] = other[better]


def packed_partial(seed, h, w, world):
    d, _, n = partial_map(seed, h, w)
    b = row_block(h, world)
    out = torch.zeros((world * b, w, 4), dtype=torch.float64)
    out[..., 0] = float("inf")
    out[:h, :, 0] = d
    out[:h, :, 1:] = n
    return out


def _rowblock_worker(rank, world, port, h, w, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blocks = rowblock_exchange(packed_partial(200 + rank, h, w, world), world)
        merged = gather_blocks(merge_blocks(blocks, hit_wins_packed), world)
        out[rank] = merged[:h].clone()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,h", [(2, 12), (3, 7)])
def test_gloo_rowblock_exchange_equals_single_merge(world, h):
    """All-to-all of row blocks, rank-order _hit_wins fold, all-gather: every
    rank ends with the single-process merge of all partials (ragged last block)."""
    w = 5
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rowblock_worker, args=(world, _free_port(), h, w, out), nprocs=world, join=True)
    want = packed_partial(200, h, w, world)[:h].clone()
    for r in range(1, world):
        hit_wins_packed(want, packed_partial(200 + r, h, w, world)[:h])
    for r in range(world):
        assert torch.equal(out[r], want)
    # order-free: folding in reverse rank order gives the same map
    rev = packed_partial(200 + world - 1, h, w, world)[:h].clone()
    for r in range(world - 2, -1, -1):
        hit_wins_packed(rev, packed_partial(200 + r, h, w, world)[:h])
    assert torch.equal(rev, want)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        depth = torch.full((4, 5), float(rank + 1), dtype=torch.float64)
        broadcast_frame(depth, src=0)
        parts = partial_map(100 + rank)
        gathered = gather_partials(parts)
        merged = merge_in_rank_order(gathered, hit_wins_merge)
        out[rank] = {"depth": depth.clone(), "merged": [t.clone() for t in merged],
                     "keys": owned_keys(list(range(8)), rank, world)}
    finally:
        dist.destroy_process_group()


def test_owner_partition_covers_every_volume_once():
    keys = [(i, 0, 0) for i in range(11)]
    grid = [(x, y, z) for x in (-511, -1) for y in (-511, -1) for z in (0, 510)]  # config 3
    for ks in (keys, grid):
        for world in (1, 2, 3, 4, 8):
            owned = [owned_keys(ks, r, world) for r in range(world)]
            flat = [k for o in owned for k in o]
            assert sorted(flat) == sorted(ks)
            assert max(map(len, owned)) - min(map(len, owned)) <= 1
            for o in owned:  # allocation order kept within a rank
                assert o == [k for k in ks if k in o]
    assert all(owner_of(i, 4) == i % 4 for i in range(11))
    # config 3 on 2 ranks: each rank gets one tile of every (y, z) row; on 4
    # ranks one tile per y layer and per z layer
    for world, axes in ((2, (1, 2)), (4, (1,))):
        for r in range(world):
            mine = owned_keys(grid, r, world)
            for a in axes:
                assert len({k[a] for k in mine}) == 2
    for r in range(4):
        assert len({k[2] for k in owned_keys(grid, r, 4)}) == 2


def test_gloo_world2_broadcast_gather_merge():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    # every rank received rank 0's frame
    for r in range(world):
        assert torch.equal(out[r]["depth"], torch.full((4, 5), 1.0, dtype=torch.float64))
    # every rank holds the same merged map ...
    assert all(torch.equal(a, b) for a, b in zip(out[0]["merged"], out[1]["merged"]))
    # ... equal to a single-process merge of all partials, in either order
    for order in ([0, 1], [1, 0]):
        acc = [t.clone() for t in partial_map(100 + order[0])]
        for r in order[1:]:
            hit_wins_merge(acc, partial_map(100 + r))
        assert all(torch.equal(a, b) for a, b in zip(acc, out[0]["merged"]))
    # volume ownership is disjoint and complete
    assert sorted(out[0]["keys"] + out[1]["keys"]) == list(range(8))


def _handles_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1511_07106_b200.distributed import exchange_handles, peer_exchange_supported
        out[rank] = (exchange_handles(bytes([rank + 1]) * 64, world),
                     peer_exchange_supported(world))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_peer_handle_exchange(world):
    """PeerExchange.connect's host plumbing: every rank gets every rank's IPC
    handle in rank order; without distinct CUDA devices the peer-memory path
    is not selected (the NCCL/gloo row-block exchange runs instead)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_handles_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    want = [bytes([r + 1]) * 64 for r in range(world)]
    for r in range(world):
        assert out[r][0] == want
        assert out[r][1] is False


def _connect_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1511_07106_b200.distributed import _connect_peers
        from paper_1511_07106_b200.geometry import CameraIntrinsics
        intr = CameraIntrinsics(100.0, 100.0, 31.5, 23.5, 64, 48)
        got = _connect_peers(intr, rank, world, None, required=False)
        try:
            _connect_peers(intr, rank, world, None, required=True)
            raised = False
        except RuntimeError:
            raised = True
        out[rank] = (got is None, raised)
    finally:
        dist.destroy_process_group()


def test_gloo_peer_connect_agreement():
    """No rank can map peer memory here (no GPU): every rank agrees to fall
    back (None) or, when the peer path was required, every rank raises —
    none is left waiting in a collective."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_connect_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] == (True, True) and out[1] == (True, True)


# ---------------------------------------------------------------------------
# re-tiling, balanced ownership and unit migration
# ---------------------------------------------------------------------------

from paper_1511_07106_b200.distributed import (balanced_owners, default_retile, initial_owners,  # noqa: E402
                                               move_units, retile, valid_retile)


@pytest.mark.parametrize("n,k", [(512, 2), (512, 3), (256, 2), (64, 2)])
def test_retile_partitions_each_tile_with_two_voxel_overlap(n, k):
    import numpy as np
    keys = [(-511, -511, 0), (-1, -511, 0)] if n == 512 else [(0, 0, 0)]
    units, m = retile(keys, n, 0.004, k)
    assert len(units) == len(keys) * k ** 3 and m == (n - 2) // k + 2
    for i, key in enumerate(keys):
        cover = np.zeros((n, n, n), np.int32)
        mine = units[i * k ** 3:(i + 1) * k ** 3]  # sub-tiles come in tile order
        assert len(mine) == k ** 3
        for u in mine:
            lo = [u[a] - key[a] for a in range(3)]
            assert all(lo[a] + m <= n for a in range(3))  # inside the tile
            cover[lo[2]:lo[2] + m, lo[1]:lo[1] + m, lo[0]:lo[0] + m] += 1
        assert cover.min() >= 1  # the union is the tile
        # neighbours along an axis share exactly two voxel layers
        s = (n - 2) // k
        assert m - s == 2


def test_retile_validity_and_defaults():
    assert valid_retile(512, 2) and valid_retile(512, 3) and not valid_retile(512, 4)
    assert valid_retile(256, 2) and not valid_retile(256, 3)
    assert default_retile(1) == 1 and default_retile(2) == 2 and default_retile(8) == 3
    assert default_retile(8, 256) == 2
    with pytest.raises(ValueError):
        retile([(0, 0, 0)], 256, 0.01, 3)


def test_balanced_owners_deterministic_balanced_and_sticky():
    import random
    rng = random.Random(3)
    for world in (2, 3, 8):
        costs = [rng.expovariate(1.0) for _ in range(64)]
        a = balanced_owners(costs, world)
        assert a == balanced_owners(list(costs), world)
        load = [sum(c for c, o in zip(costs, a) if o == r) for r in range(world)]
        mean = sum(costs) / world
        assert max(load) <= mean + max(costs) + 1e-12  # LPT bound
        # a balanced current assignment survives a rebalance on the same costs
        assert balanced_owners(costs, world, a) == a
        # a small change of the costs moves few units
        costs2 = [c * (1.0 + 0.02 * rng.random()) for c in costs]
        b = balanced_owners(costs2, world, a)
        assert sum(x != y for x, y in zip(a, b)) <= len(costs) // 4
    assert balanced_owners([1.0, 2.0], 1) == [0, 0]
    keys = [(x, y, z) for x in (0, 1) for y in (0, 1) for z in (0, 1)]
    own = initial_owners(keys, 4)
    assert sorted(own) == [0, 0, 1, 1, 2, 2, 3, 3]


def _move_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        moves = [(0, 0, 1), (1, 2, 0), (2, 1, 2), (3, 0, 2), (4, 1, 1)]
        payloads = {u: [torch.full((3, 4), float(10 * u + a)), torch.arange(5, dtype=torch.int64) + u]
                    for u, a, b in moves if a == rank}
        got = move_units(moves, rank, payloads,
                         lambda u: [torch.empty(3, 4), torch.empty(5, dtype=torch.int64)])
        out[rank] = {u: [t.clone() for t in ts] for u, ts in got.items()}
    finally:
        dist.destroy_process_group()


def test_gloo_move_units_world3():
    world = 3
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_move_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    want = {1: {0: 0.0}, 0: {1: 12.0}, 2: {2: 21.0, 3: 30.0}}
    for r in range(world):
        assert set(out[r]) == set(want[r])
        for u, v in want[r].items():
            assert torch.equal(out[r][u][0], torch.full((3, 4), v))
            assert torch.equal(out[r][u][1], torch.arange(5, dtype=torch.int64) + u)
