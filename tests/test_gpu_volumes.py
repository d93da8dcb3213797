"""VolumeSet residency semantics and bin_endpoints known answers on the GPU
package: the reference's test_volumes.py cases (volumes.py:156-331), run for
both spill tiers — the reference's files ("disk") and pinned host memory
("host", same LRU order and whole-image counters; files only on persist())."""

import numpy as np
import torch
import pytest

import paper_1511_07106_b200 as tf
from paper_1511_07106_b200.geometry import DepthFrame, Pose

pytestmark = pytest.mark.gpu

PARAMS = tf.FusionParams(truncation=0.2)
TIERS = ["disk", "host"]


def make_set(tmp_path, max_resident, tier, n=4):
    return tf.VolumeSet(PARAMS, voxels_per_side=n, voxel_size=0.1, max_resident=max_resident,
                        spill_dir=tmp_path, spill_tier=tier)


@pytest.mark.parametrize("tier", TIERS)
def test_volume_set_lifecycle(tmp_path, tier):
    vs = make_set(tmp_path, 2, tier)
    vs.add((0, 0, 0))
    assert (0, 0, 0) in vs and len(vs) == 1
    vol = vs.acquire((0, 0, 0))
    vol.tsdf[0, 0, 0] = 0.25
    with pytest.raises(RuntimeError):
        vs.acquire((0, 0, 0))
    vs.release((0, 0, 0))
    with pytest.raises(RuntimeError):
        vs.release((0, 0, 0))
    with pytest.raises(KeyError):
        vs.acquire((9, 9, 9))
    assert vs.acquire((0, 0, 0)).tsdf[0, 0, 0] == np.float32(0.25)


@pytest.mark.parametrize("tier", TIERS)
def test_eviction_is_least_recently_used(tmp_path, tier):
    vs = make_set(tmp_path, 2, tier)
    a, b, c = (0, 0, 0), (4, 0, 0), (8, 0, 0)
    for key in (a, b, c):
        vs.add(key)
    for key in (a, b, c):  # a is least recently used when c arrives: a is spilled
        vs.acquire(key)
        vs.release(key)
    assert vs.files_written == 1
    assert [k for k, _ in vs.resident_volumes()] == [b, c]
    if tier == "disk":
        assert vs.spill_path(a).exists() and not vs.spill_path(b).exists()
    vs.acquire(a)
    vs.release(a)
    assert vs.files_read == 1 and vs.bytes_read == tf.spill_file_size(4)


@pytest.mark.parametrize("tier", TIERS)
def test_live_tiles_survive_pressure(tmp_path, tier):
    vs = make_set(tmp_path, 1, tier)
    vs.add((0, 0, 0))
    vs.add((4, 0, 0))
    vs.acquire((0, 0, 0))
    vs.acquire((4, 0, 0))  # the budget is full of live tiles: overflow, not eviction
    assert vs.resident_count == 2 and vs.files_written == 0
    vs.release((0, 0, 0))
    vs.release((4, 0, 0))


@pytest.mark.parametrize("tier", TIERS)
def test_round_robin_transfer_counts(tmp_path, tier):
    vs = make_set(tmp_path, 1, tier)
    keys = [(0, 0, 0), (4, 0, 0), (8, 0, 0)]
    for key in keys:
        vs.add(key)

    def sweep():
        for key in keys:
            vs.acquire(key)
            vs.release(key)

    sweep()
    assert (vs.files_read, vs.files_written) == (0, 2)
    sweep()
    assert (vs.files_read, vs.files_written) == (3, 5)
    sweep()
    assert (vs.files_read, vs.files_written) == (6, 8)
    assert vs.bytes_written == 8 * tf.spill_file_size(4)


@pytest.mark.parametrize("tier", TIERS)
def test_remove_returns_archived_state(tmp_path, tier):
    vs = make_set(tmp_path, 1, tier)
    vs.add((0, 0, 0))
    vs.add((4, 0, 0))
    vol = vs.acquire((0, 0, 0))
    vol.tsdf[1, 2, 3] = 0.125  # a host-mirror edit must survive the spill
    vs.release((0, 0, 0))
    vs.acquire((4, 0, 0))
    vs.release((4, 0, 0))
    archived = vs.remove((0, 0, 0))
    assert archived.tsdf[1, 2, 3] == np.float32(0.125)
    assert (0, 0, 0) not in vs and not vs.spill_path((0, 0, 0)).exists()


@pytest.mark.parametrize("tier", TIERS)
def test_flush_persists_without_evicting(tmp_path, tier):
    vs = make_set(tmp_path, 4, tier)
    for key in [(0, 0, 0), (4, 0, 0)]:
        vs.add(key)
        vs.acquire(key)
        vs.release(key)
    vs.flush()
    assert vs.resident_count == 2 and vs.files_written == 2
    if tier == "disk":
        assert vs.spill_path((0, 0, 0)).exists() and vs.spill_path((4, 0, 0)).exists()
    else:
        assert vs.persist() == 2 * tf.spill_file_size(4)
        back, _ = tf.load_subvolume(vs.spill_path((4, 0, 0)))
        assert np.array_equal(back.tsdf, vs.acquire((4, 0, 0)).tsdf)


@pytest.mark.parametrize("tier", TIERS)
def test_volume_set_validation(tmp_path, tier):
    with pytest.raises(ValueError):
        make_set(tmp_path, 0, tier)
    vs = make_set(tmp_path, 1, tier)
    vs.add((0, 0, 0))
    with pytest.raises(ValueError):
        vs.add((0, 0, 0))


# ---- bin_endpoints known answers (reference test_volumes.py:238-266) ----------------

def test_bin_endpoints_single_pixel(small_intr):
    depth = np.zeros((60, 80))
    depth[30, 40] = 2.0  # optical axis: endpoint (0, 0, 2) in block (0, 0, 1) of 1.5 m
    assert tf.bin_endpoints(DepthFrame(depth), small_intr, Pose.identity(), 30, 0.05) == {(0, 0, 30): 1}


def test_bin_endpoints_uses_ray_length_along_unit_ray(small_intr):
    depth = np.zeros((60, 80))
    depth[30, 60] = 2.0  # 2 m along the unit ray (0.2, 0, 1) / |.|: x 0.392, z 1.961
    assert tf.bin_endpoints(DepthFrame(depth), small_intr, Pose.identity(), 30, 0.05) == {(0, 0, 30): 1}


def test_bin_endpoints_negative_cells(small_intr):
    depth = np.zeros((60, 80))
    depth[30, 40] = 2.0
    behind = Pose(np.eye(3), np.array([-2.0, 0.0, 0.0]))
    assert tf.bin_endpoints(DepthFrame(depth), small_intr, behind, 30, 0.05) == {(-60, 0, 30): 1}


def test_bin_endpoints_empty_frame(small_intr):
    assert tf.bin_endpoints(DepthFrame(np.zeros((60, 80))), small_intr, Pose.identity(), 30, 0.05) == {}


def test_device_endpoint_histogram_equals_sorted_unique():
    """tf_bin_endpoints (hash-table histogram, one read-back) == the per-pixel
    cells + sort-based unique, on corridor frames, on a frame with more cells
    than the table holds (host fallback) and with cells beyond the packed key
    range (fallback)."""
    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200 import volumes as vm
    from paper_1511_07106_b200.synth import corridor_depth, corridor_scene
    intr = tf.RunConfig().intrinsics()
    scene = corridor_scene()
    poses = tf.corridor_trajectory(20.0, 2000)
    for i in (0, 333, 1000, 1999):
        f = torch.as_tensor(corridor_depth(scene, poses[i], intr).data, device="cuda")
        for spacing, vs in ((256, 0.004), (30, 0.004), (8, 0.004), (4, 0.0001)):
            got = vm.bin_endpoints(f, intr, poses[i], spacing, vs)
            want = vm._bin_endpoints_sorted(f, intr, poses[i], spacing, vs)
            assert got == want and list(got) == list(want), (i, spacing)
    far = tf.Pose(np.eye(3), np.array([5.0e3, 0.0, 0.0]))  # cells beyond +-2^20 blocks
    f = torch.full((intr.height, intr.width), 2.0, dtype=torch.float64, device="cuda")
    assert vm.bin_endpoints(f, intr, far, 1, 0.001) == vm._bin_endpoints_sorted(f, intr, far, 1, 0.001)
    empty = torch.zeros((intr.height, intr.width), dtype=torch.float64, device="cuda")
    assert vm.bin_endpoints(empty, intr, poses[0], 256, 0.004) == {}


def test_packed_spill_images_round_trip_bounds():
    """tf_pack_voxels / tf_unpack_voxels (the host_packed capacity mode):
    tsdf within half rounding (<= 2^-11 |tsdf|), integral weights <= 255 exact,
    larger weights saturate at 255."""
    from paper_1511_07106_b200 import _native as nat
    g = torch.Generator(device="cpu").manual_seed(5)
    n = 1 << 20
    t = (torch.rand(n, generator=g) * 2 - 1) * 0.05
    w = torch.randint(0, 300, (n,), generator=g).float()
    vox = torch.stack([t, w], -1).cuda()
    ht = torch.empty(n, dtype=torch.float16, device="cuda")
    hw = torch.empty(n, dtype=torch.uint8, device="cuda")
    back = torch.empty_like(vox)
    L = nat.lib()
    nat.check(L.tf_pack_voxels(nat.ptr(vox), n, nat.ptr(ht), nat.ptr(hw), nat.stream_handle()), "pack")
    nat.check(L.tf_unpack_voxels(nat.ptr(ht), nat.ptr(hw), n, nat.ptr(back), nat.stream_handle()), "unpack")
    back = back.cpu()
    err = (back[:, 0] - t).abs()
    assert bool((err <= t.abs() * 2.0 ** -11 + 6e-8).all())
    assert torch.equal(back[:, 1], torch.clamp(w, max=255.0))


def test_host_packed_tier_keeps_placement_and_bounds_the_error(tmp_path):
    """The dynamic corridor run (tests/golden/dynamic_small.npz) with the lossy
    packed spill tier: allocation, residency and spill counters equal the
    reference's; weights equal the exact host tier's; tsdf within the half
    rounding of every spill the tile went through."""
    import paper_1511_07106_b200 as tf
    from conftest import load_golden
    g = load_golden("dynamic_small.npz")
    fx, fy, cx, cy, w, h = g["intr"]
    runs = {}
    for tier in ("host", "host_packed"):
        cfg = tf.RunConfig(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h), dynamic=True,
                           block_voxels=34, block_side_length=0.64, max_volumes=4, max_resident=3,
                           use_groundtruth=True, spill_tier=tier)
        pipe = tf.FusionPipeline(cfg, tmp_path / tier)
        recs = []
        for i, (f, m) in enumerate(zip(g["frames"], g["poses"])):
            r = pipe.step(tf.DepthFrame(f), Pose(m[:3, :3], m[:3, 3]))
            recs.append([r.volumes, r.resident, r.files_read, r.files_written, r.bytes_read, r.bytes_written])
        assert recs == g["counters"].tolist()
        vols = {}
        for k in pipe.volumes.keys():
            v = pipe.volumes.acquire(k)
            vols[k] = v.voxels.cpu()
            pipe.volumes.release(k)
        runs[tier] = (vols, pipe.volumes.link_bytes_written, pipe.volumes.files_written)
    exact, packed = runs["host"][0], runs["host_packed"][0]
    assert exact.keys() == packed.keys()
    tau = tf.FusionParams.for_voxel_size(0.64 / 32).truncation
    spills = runs["host"][2]
    for k in exact:
        assert torch.equal(exact[k][..., 1], packed[k][..., 1])
        assert float((exact[k][..., 0] - packed[k][..., 0]).abs().max()) <= spills * 4.9e-4 * tau
    assert runs["host_packed"][1] * 8 == runs["host"][1] * 3  # 3 B per voxel instead of 8


@pytest.mark.parametrize("tier", ["host", "host_packed"])
def test_dropped_tiles_free_their_memory_without_the_gc(tmp_path, tier):
    """Volumes and ray maps hold no reference cycle: a tile evicted to the host
    tier, or dropped, releases its device memory at once (with the cyclic
    garbage collector off), so a long spill sequence does not pile up."""
    import gc
    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200.volumes import VolumeSet
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    try:
        base = torch.cuda.memory_allocated()
        params = tf.FusionParams.for_voxel_size(0.004)
        vset = VolumeSet(params, voxels_per_side=128, voxel_size=0.004, max_resident=2,
                         spill_dir=tmp_path, spill_tier=tier)
        for k in range(4):
            vset.add((k * 126, 0, 0))
        tile_bytes = 128 ** 3 * 8
        for _ in range(3):
            for k in vset.keys():
                vset.acquire(k)
                tf.raycast_volumes([vset._resident[k]], tf.Pose.identity(),
                                   tf.CameraIntrinsics(50.0, 50.0, 31.5, 23.5, 64, 48),
                                   tf.RayMap.empty(tf.CameraIntrinsics(50.0, 50.0, 31.5, 23.5, 64, 48)),
                                   params)
                vset.release(k)
                torch.cuda.synchronize()
                assert torch.cuda.memory_allocated() - base < 3.5 * tile_bytes
        del vset
        torch.cuda.synchronize()
        assert torch.cuda.memory_allocated() - base < 0.5 * tile_bytes
    finally:
        gc.enable()
