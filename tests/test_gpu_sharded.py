"""ShardedFusion's world > 1 step with the real CUDA kernels: two ranks on the
one visible GPU, collectives over gloo (host-staged, so no rank's kernel
waits on another's).  Functional check of the row-block exchange, the packed
merge and the vertex rebuild: the merged model equals the single-process
fused raycast over all volumes bit for bit.  (Timing is never taken here.)"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup():
    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200.synth import demo_scene
    intr = tf.CameraIntrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 24)
    frames = [torch.from_numpy(demo_scene().render_depth(p, intr).data.astype(np.float64)).cuda()
              for p in poses[:4]]
    return tf, intr, spec, params, poses, frames


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1511_07106_b200.distributed import ShardedFusion
        tf, intr, spec, params, poses, frames = _setup()
        shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params,
                              intr, rank, world)
        for f, p in zip(frames, poses):
            model = shard.step(f, p)
        torch.cuda.synchronize()
        out[rank] = [model.distance_dev.cpu(), model.vertices_dev.cpu(), model.normals_dev.cpu(),
                     len(shard.keys)]
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one_process():
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from paper_1511_07106_b200.distributed import ShardedFusion
    tf, intr, spec, params, poses, frames = _setup()
    single = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params,
                           intr, 0, 1)
    for f, p in zip(frames, poses):
        model = single.step(f, p)
    want = [model.distance_dev.cpu(), model.vertices_dev.cpu(), model.normals_dev.cpu()]
    assert torch.isfinite(want[0]).sum().item() > 3000
    assert out[0][3] + out[1][3] == len(spec.keys)
    for r in range(world):
        for got, ref in zip(out[r][:3], want):
            assert torch.equal(got, ref)


@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_emulated_ranks_equal_one_process(world):
    """The peer-memory reduction (csrc/comm.cu) with `world` emulated ranks in
    this process on the one GPU: each rank integrates and raycasts only the
    volumes it owns into its region's partial, then each rank's reduce kernel
    runs in turn without flag waits (TF_COMM_NOWAIT; ranks that wait on one
    another never share a GPU).  Every rank's model equals the single-process
    raycast over all volumes bit for bit, frame after frame."""
    from paper_1511_07106_b200.distributed import PeerExchange, ShardedFusion, owned_keys
    tf, intr, spec, params, poses, frames = _setup()
    single = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params,
                           intr, 0, 1)
    peers = [PeerExchange(intr, r, world) for r in range(world)]
    PeerExchange.link_local(peers)
    tiles = [[tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length)
              for k in owned_keys(spec.keys, r, world)] for r in range(world)]
    assert sum(len(t) for t in tiles) == len(spec.keys)
    for f, p in zip(frames, poses):
        want = single.step(f, p)
        for r in range(world):
            tf.integrate_volumes(tiles[r], f, p, intr, params)
            peers[r].partial.reset()
            tf.raycast_volumes(tiles[r], p, intr, peers[r].partial, params)
        for r in range(world):
            peers[r].reduce(nowait=True)
        torch.cuda.synchronize()
        assert torch.isfinite(want.distance_dev).sum().item() > 3000
        for r in range(world):
            m = peers[r].model
            assert torch.equal(m.distance_dev, want.distance_dev)
            assert torch.equal(m.vertices_dev, want.vertices_dev)
            assert torch.equal(m.normals_dev, want.normals_dev)
    assert all(pe.error() == 0 for pe in peers)


def test_peer_exchange_region_and_handle():
    """A fresh region reads as the empty ray map; the IPC handle exports."""
    from paper_1511_07106_b200.distributed import PeerExchange
    tf, intr, *_ = _setup()
    pe = PeerExchange(intr, 1, 2)
    for m in (pe.partial, pe.model):
        assert torch.equal(m.distance_dev, torch.full((intr.height, intr.width), float("inf"),
                                                      dtype=torch.float64, device="cuda"))
        assert not m.vertices_dev.any() and not m.normals_dev.any()
    h = pe.export()
    assert len(h) == 64 and any(h)
    with pytest.raises(RuntimeError):
        pe.reduce()  # rank 0's region is not mapped
