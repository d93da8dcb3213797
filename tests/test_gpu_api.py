"""The reference's own API-level tests, run against the B200 package.

Mirrors tilefusion's test_tsdf.py (hand-computed oracles), test_pipeline.py
(end-to-end behaviour), test_volumes.py (spill format and residency
counters) and the tracking tests, with the operators running in libtfb200.
"""

import dataclasses
import tempfile

import numpy as np
import pytest
import torch

import paper_1511_07106_b200 as tf
from paper_1511_07106_b200.geometry import rotation_angle, rotation_from_axis_angle
from paper_1511_07106_b200.synth import demo_scene

pytestmark = pytest.mark.gpu


def flat_frame(depth, width=80, height=60):
    return tf.DepthFrame(np.full((height, width), float(depth)))


@pytest.fixture
def wall_volume(small_intr):
    vol = tf.TsdfSubvolume.empty(np.array([-5, -5, 16]), 10, 1.0)
    params = tf.FusionParams.for_voxel_size(vol.voxel_size)
    tf.integrate(vol, flat_frame(2.05), tf.Pose.identity(), small_intr, params)
    return vol, params


# ---- tsdf hand oracles (reference test_tsdf.py:65-200) --------------------------------

def test_integrate_center_column_oracle(small_intr):
    vol = tf.TsdfSubvolume.empty(np.array([-4, -4, 16]), 10, 1.0)
    params = tf.FusionParams.for_voxel_size(0.1)
    tf.integrate(vol, flat_frame(2.0), tf.Pose.identity(), small_intr, params)
    assert vol.tsdf[0, 4, 4] == pytest.approx(0.4)
    assert vol.tsdf[2, 4, 4] == pytest.approx(0.2)
    assert vol.tsdf[7, 4, 4] == pytest.approx(-0.3)
    assert vol.weight[2, 4, 4] == 1.0
    assert vol.tsdf[9, 4, 4] == 0.0 and vol.weight[9, 4, 4] == 0.0


def test_integrate_ray_correction_running_mean_cap(small_intr):
    vol = tf.TsdfSubvolume.empty(np.array([-4, -4, 16]), 10, 1.0)
    params = tf.FusionParams.for_voxel_size(0.1)
    tf.integrate(vol, flat_frame(2.0), tf.Pose.identity(), small_intr, params)
    assert vol.tsdf[3, 4, 5] == pytest.approx(0.09974408, abs=1e-6)
    tf.integrate(vol, flat_frame(2.2), tf.Pose.identity(), small_intr, params)
    assert vol.tsdf[2, 4, 4] == pytest.approx(0.3, abs=1e-7)
    assert vol.weight[2, 4, 4] == 2.0
    capped = tf.TsdfSubvolume.empty(np.array([-4, -4, 16]), 10, 1.0)
    p3 = tf.FusionParams(truncation=0.4, max_weight=3.0)
    for _ in range(5):
        tf.integrate(capped, flat_frame(2.0), tf.Pose.identity(), small_intr, p3)
    assert capped.weight[2, 4, 4] == 3.0


def test_integrate_invalid_pixels_and_size_mismatch(small_intr):
    vol = tf.TsdfSubvolume.empty(np.array([-4, -4, 16]), 10, 1.0)
    params = tf.FusionParams.for_voxel_size(0.1)
    tf.integrate(vol, flat_frame(0.0), tf.Pose.identity(), small_intr, params)
    assert vol.observed_count() == 0
    with pytest.raises(ValueError):
        tf.integrate(vol, flat_frame(2.0, width=81), tf.Pose.identity(), small_intr, params)


def test_trilinear_sample(wall_volume):
    vol, _ = wall_volume
    assert tf.trilinear_sample(vol, np.array([0.0, 0.0, 1.95])) == pytest.approx(0.1, abs=1e-6)
    assert tf.trilinear_sample(vol, np.array([0.0, 0.0, 0.5])) is None
    assert tf.trilinear_sample(vol, np.array([0.0, 0.0, 2.46])) is None


def test_raycast_oracles(wall_volume, small_intr):
    vol, params = wall_volume
    rm = tf.RayMap.empty(small_intr)
    tf.raycast(vol, tf.Pose.identity(), small_intr, rm, params)
    assert rm.distance[30, 40] == pytest.approx(2.05, abs=1e-6)
    assert np.allclose(rm.vertices[30, 40], [0.0, 0.0, 2.05], atol=1e-6)
    assert np.allclose(rm.normals[30, 40], [0.0, 0.0, -1.0], atol=5e-3)
    assert rm.distance[30, 50] == pytest.approx(2.0602245, abs=5e-3)
    away = tf.RayMap.empty(small_intr)
    tf.raycast(vol, tf.Pose(np.eye(3), np.array([0.0, 0.0, 3.5])), small_intr, away, params)
    assert not away.valid.any()


def test_raycast_merges_by_distance(small_intr):
    params = tf.FusionParams.for_voxel_size(0.1)
    near = tf.TsdfSubvolume.empty(np.array([-5, -5, 16]), 10, 1.0)
    far = tf.TsdfSubvolume.empty(np.array([-5, -5, 26]), 10, 1.0)
    tf.integrate(near, flat_frame(2.05), tf.Pose.identity(), small_intr, params)
    tf.integrate(far, flat_frame(3.05), tf.Pose.identity(), small_intr, params)
    merged = tf.RayMap.empty(small_intr)
    tf.raycast(far, tf.Pose.identity(), small_intr, merged, params)
    assert merged.distance[30, 40] == pytest.approx(3.05, abs=1e-6)
    tf.raycast(near, tf.Pose.identity(), small_intr, merged, params)
    assert merged.distance[30, 40] == pytest.approx(2.05, abs=1e-6)
    half = merged.downsampled()
    assert half.distance.shape == (30, 40)


def test_extract_wall_points_and_empty(wall_volume):
    vol, _ = wall_volume
    cloud = tf.extract_points(vol)
    assert len(cloud) == 100
    assert np.abs(cloud.vertices[:, 2] - 2.05).max() < 5e-3
    assert cloud.normals[:, 2].max() < -0.99
    assert len(tf.extract_points(tf.TsdfSubvolume.empty(np.zeros(3), 8, 0.8))) == 0


def test_host_mirror_edits_reach_the_device(small_intr):
    vol = tf.TsdfSubvolume.empty(np.array([-4, -4, 16]), 10, 1.0)
    params = tf.FusionParams.for_voxel_size(0.1)
    w = vol.weight            # held mirror
    w[2, 4, 4] = 5.0          # edited on the host ...
    tf.integrate(vol, flat_frame(2.0), tf.Pose.identity(), small_intr, params)
    assert w[2, 4, 4] == 6.0  # ... uploaded before the kernel, refreshed after it
    assert vol.voxels[2, 4, 4, 1].item() == 6.0


# ---- spill format and residency (reference test_volumes.py) -----------------------------

def test_spill_round_trip_and_corruption(tmp_path, small_intr):
    vol = tf.TsdfSubvolume.empty(np.array([-4, -4, 16]), 10, 1.0)
    params = tf.FusionParams.for_voxel_size(0.1)
    tf.integrate(vol, flat_frame(2.0), tf.Pose.identity(), small_intr, params)
    n = tf.save_subvolume(tmp_path / "a.tsdv", vol, params)
    assert n == 52 + 10 ** 3 * 8 == (tmp_path / "a.tsdv").stat().st_size
    back, p2 = tf.load_subvolume(tmp_path / "a.tsdv")
    assert torch.equal(back.voxels, vol.voxels)
    assert np.array_equal(back.origin_voxel, vol.origin_voxel)
    assert p2.truncation == pytest.approx(params.truncation)
    blob = bytearray((tmp_path / "a.tsdv").read_bytes())
    blob[0] = ord("X")
    (tmp_path / "b.tsdv").write_bytes(bytes(blob))
    with pytest.raises(ValueError, match="magic"):
        tf.load_subvolume(tmp_path / "b.tsdv")
    (tmp_path / "c.tsdv").write_bytes(bytes(blob[:100]))
    with pytest.raises(ValueError):
        tf.load_subvolume(tmp_path / "c.tsdv")


@pytest.mark.parametrize("tier", ["disk", "host"])
def test_spill_traffic_matches_the_schedule(tmp_path, small_intr, tier):
    """Acceptance 7 (test_acceptance.py:271-320): cold (0, 2) then (3, 3), for
    both the reference's file tier and the pinned-host tier."""
    params = tf.FusionParams.for_voxel_size(0.05)
    vs = tf.VolumeSet(params, voxels_per_side=16, voxel_size=0.05, max_resident=1, spill_dir=tmp_path,
                      spill_tier=tier)
    keys = [(-24, -8, 20), (-8, -8, 20), (8, -8, 20)]
    for k in keys:
        vs.add(k)
    snaps, per_frame = {}, []
    for depth in (1.5, 1.52, 1.48, 1.5):
        frame = tf.DepthFrame(np.full((60, 80), depth, np.float32))
        r0, w0 = vs.files_read, vs.files_written
        for k in keys:
            vol = vs.acquire(k)
            assert vs.resident_count <= 1
            if k in snaps:
                assert np.array_equal(vol.tsdf, snaps[k][0]) and np.array_equal(vol.weight, snaps[k][1])
            tf.integrate(vol, frame, tf.Pose.identity(), small_intr, params)
            snaps[k] = (vol.tsdf.copy(), vol.weight.copy())
            vs.release(k)
        per_frame.append((vs.files_read - r0, vs.files_written - w0))
    assert per_frame[0] == (0, 2) and all(c == (3, 3) for c in per_frame[1:])


def test_host_tier_lru_persist_and_remove(tmp_path, small_intr):
    """Pinned-host tier: reference LRU/counter semantics (test_volumes.py:140-226),
    summaries survive a round trip, persist() writes loadable .tsdv files."""
    params = tf.FusionParams.for_voxel_size(0.1)
    disk = tf.VolumeSet(params, 10, 0.1, max_resident=2, spill_dir=tmp_path / "d")
    host = tf.VolumeSet(params, 10, 0.1, max_resident=2, spill_dir=tmp_path / "h", spill_tier="host")
    keys = [(-4, -4, 16), (4, -4, 16), (-4, 4, 16)]
    pose = tf.Pose.identity()
    for vs in (disk, host):
        for k in keys:
            vs.add(k)
        for depth in (2.0, 2.1, 1.9):
            for k in keys:
                vol = vs.acquire(k)
                tf.integrate(vol, flat_frame(depth), pose, small_intr, params)
                rm = tf.RayMap.empty(small_intr)
                tf.raycast(vol, pose, small_intr, rm, params)  # builds the brick summary
                vs.release(k)
    assert (host.files_read, host.files_written, host.bytes_read, host.bytes_written) == (
        disk.files_read, disk.files_written, disk.bytes_read, disk.bytes_written)
    assert [k for k, _ in host.resident_volumes()] == [k for k, _ in disk.resident_volumes()]
    assert not any(host.spill_path(k).exists() for k in keys)
    for k in keys:  # same voxels through either tier; a host-loaded summary is exact
        a, b = disk.acquire(k), host.acquire(k)
        assert torch.equal(a.voxels, b.voxels)
        if b.brick_bad is not None:
            bad, flags = b.brick_bad.clone(), b.brick_flags.clone()
            b.invalidate_summary()
            b._summary_for(params.truncation)
            assert torch.equal(bad, b.brick_bad) and torch.equal(flags, b.brick_flags)
        disk.release(k)
        host.release(k)
    written = host.persist()
    assert written == 3 * tf.spill_file_size(10)
    for k in keys:
        back, _ = tf.load_subvolume(host.spill_path(k))
        vol = host.acquire(k)
        assert torch.equal(back.voxels, vol.voxels)
        host.release(k)
    gone = host.remove(keys[0])
    assert not host.spill_path(keys[0]).exists() and keys[0] not in host
    assert torch.equal(gone.voxels, disk.remove(keys[0]).voxels)
    with pytest.raises(ValueError):
        tf.VolumeSet(params, 10, 0.1, max_resident=1, spill_dir=tmp_path, spill_tier="tape")


# ---- pipeline (reference test_pipeline.py) ---------------------------------------------------

def small_config(**kw):
    base = dict(fx=131.25, fy=131.25, cx=80.0, cy=60.0, width=160, height=120, side_length=3.0,
                resolution=124, resident_resolution=62, use_groundtruth=True)
    base.update(kw)
    return tf.RunConfig(**base)


def render_orbit(intr, frames, step_deg=None):
    scene = demo_scene()
    if step_deg is None:
        poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, frames)
    else:
        poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, round(360.0 / step_deg))[:frames]
    return [scene.render_depth(p, intr) for p in poses], poses


def surface_mean_distance(points):
    return float(np.abs(demo_scene().signed_distance(points)).mean())


def test_groundtruth_fusion_accuracy(tmp_path):
    cfg = small_config()
    frames, poses = render_orbit(cfg.intrinsics(), 6)
    res = tf.run_fusion(frames, cfg, tmp_path, gt_poses=poses)
    assert res.lost_frames == 0 and len(res.cloud) > 1000
    assert surface_mean_distance(res.cloud.vertices) < 3e-3


def test_records_reflect_memory_pressure(tmp_path):
    cfg = small_config(max_resident=2)
    frames, poses = render_orbit(cfg.intrinsics(), 3)
    res = tf.run_fusion(frames, cfg, tmp_path / "disk", gt_poses=poses)
    assert all(r.volumes == 8 and r.resident <= 2 for r in res.records)
    assert res.records[0].files_read == 0
    assert all(r.files_read > 0 and r.bytes_read > 0 for r in res.records[1:])
    # the pinned-host tier: same schedule, same records, same cloud
    host = tf.run_fusion(frames, small_config(max_resident=2, spill_tier="host"), tmp_path / "host",
                         gt_poses=poses)
    strip = lambda recs: [dataclasses.replace(r, residual_rms=0.0) for r in recs]  # NaN in GT mode
    assert strip(host.records) == strip(res.records)
    assert np.array_equal(host.cloud.vertices, res.cloud.vertices)


def test_tracking_mode_follows_orbit(tmp_path):
    cfg = small_config(use_groundtruth=False, min_correspondences=500)
    frames, poses = render_orbit(cfg.intrinsics(), 6, step_deg=1.5)
    res = tf.run_fusion(frames, cfg, tmp_path)
    assert res.lost_frames == 0 and all(r.tracked for r in res.records)
    for est, gt in zip(res.poses, poses):
        delta = est.invert().compose(gt)
        assert rotation_angle(delta.rotation) < np.deg2rad(1.0)
        assert np.linalg.norm(delta.translation) < 0.02


def test_lost_frame_keeps_previous_pose(tmp_path):
    cfg = small_config(use_groundtruth=False)
    intr = cfg.intrinsics()
    frames, _ = render_orbit(intr, 1)
    pipe = tf.FusionPipeline(cfg, tmp_path)
    pipe.step(frames[0])
    rec = pipe.step(tf.DepthFrame(np.zeros((intr.height, intr.width))))
    assert not rec.tracked and pipe.lost_frames == 1 and pipe.poses[1] is pipe.poses[0]


def test_dynamic_corridor_respects_budget(tmp_path):
    scene = tf.Scene((tf.Plane((0.9, 0.0, 0.0), (-1.0, 0.0, 0.0)),
                      tf.Plane((-0.9, 0.0, 0.0), (1.0, 0.0, 0.0))))
    cfg = small_config(dynamic=True, block_voxels=32, block_side_length=0.6, max_volumes=4,
                       max_resident=4)
    intr = cfg.intrinsics()
    pipe = tf.FusionPipeline(cfg, tmp_path)
    mean_z = []
    for pose in tf.corridor_trajectory(2.0, 8):
        d = scene.render_depth(pose, intr).data.copy()
        d[d > 4.0] = 0.0
        rec = pipe.step(tf.DepthFrame(d), gt_pose=pose)
        keys = pipe.volumes.keys()
        assert rec.volumes <= 4 and len(keys) == len(set(keys))
        mean_z.append(float(np.mean([k[2] for k in keys])))
    assert mean_z[-1] > mean_z[0]
    assert len(pipe.finish().cloud) > 0


def test_run_fusion_is_deterministic(tmp_path):
    cfg = small_config()
    frames, poses = render_orbit(cfg.intrinsics(), 3)
    a = tf.run_fusion(frames, cfg, tmp_path / "a", gt_poses=poses)
    b = tf.run_fusion(frames, cfg, tmp_path / "b", gt_poses=poses)
    assert np.array_equal(a.cloud.vertices, b.cloud.vertices)
    assert np.array_equal(a.cloud.normals, b.cloud.normals)


# ---- tracking (reference test_tracking.py) ---------------------------------------------------

def test_track_self_model_fixed_point_and_recovery(small_intr):
    scene = demo_scene()
    pose = tf.Pose.identity()
    frame = scene.render_depth(pose, small_intr)
    vm = tf.VertexNormalMap.from_depth(small_intr, frame).transformed(pose)
    dist = np.where(vm.valid, np.linalg.norm(vm.vertices - pose.translation, axis=-1), np.inf)
    model = tf.RayMap(vm.vertices, vm.normals, dist)
    params = tf.TrackingParams(min_correspondences=200)
    res = tf.track(frame, small_intr, model, pose, params)
    assert not res.lost and res.residual_rms < 1e-9
    assert np.abs(res.pose.matrix - np.eye(4)).max() < 1e-8
    bump = tf.Pose(rotation_from_axis_angle(np.array([0.0, 1.0, 0.0]), np.radians(1.0)),
                   np.array([0.01, 0.0, 0.0]))
    res = tf.track(frame, small_intr, model, pose, params, init=pose.compose(bump))
    delta = pose.invert().compose(res.pose)
    assert np.degrees(rotation_angle(delta.rotation)) < 0.01 and np.linalg.norm(delta.translation) < 1e-4


def test_params_volume_layout_and_validation():
    """test_tsdf.py:38-63: params, empty layout, counters, validation."""
    with pytest.raises(ValueError):
        tf.FusionParams(truncation=0.0)
    with pytest.raises(ValueError):
        tf.FusionParams(truncation=0.1, max_weight=0.5, sample_weight=1.0)
    assert tf.FusionParams.for_voxel_size(0.1).truncation == pytest.approx(0.4)
    vol = tf.TsdfSubvolume.empty(np.array([-4, -4, 16]), 8, 0.8)
    assert vol.voxel_size == pytest.approx(0.1)
    assert np.allclose(vol.world_min, [-0.4, -0.4, 1.6]) and np.allclose(vol.world_max, [0.3, 0.3, 2.3])
    assert vol.payload_bytes() == 8 * 8 ** 3 and vol.observed_count() == 0
    with pytest.raises(ValueError):
        tf.TsdfSubvolume.empty(np.array([0, 0]), 8, 0.8)
    with pytest.raises(ValueError):
        tf.TsdfSubvolume.empty(np.zeros(3), 1, 0.8)


def test_raymap_downsampled_and_point_clouds(small_intr):
    """test_tsdf.py:181-186, :201-210."""
    rm = tf.RayMap.empty(small_intr)
    rm.distance[0, 0] = 1.0  # a host-mirror edit reaches the device copy
    half = rm.downsampled()
    assert half.distance.shape == (30, 40) and half.valid[0, 0]
    with pytest.raises(ValueError):
        tf.PointCloud(np.zeros((3, 3)), np.zeros((2, 3)))
    merged = tf.PointCloud.concatenate([tf.PointCloud(np.zeros((2, 3)), np.ones((2, 3))),
                                        tf.PointCloud.empty()])
    assert len(merged) == 2 and len(tf.PointCloud.concatenate([])) == 0


def test_trilinear_outside_and_raycast_miss(wall_volume, small_intr):
    """test_tsdf.py:129-134 (outside -> None) and :160-165 (a miss leaves +inf)."""
    vol, params = wall_volume
    assert tf.trilinear_sample(vol, np.array([10.0, 10.0, 10.0])) is None
    rm = tf.RayMap.empty(small_intr)
    away = tf.Pose(np.diag([1.0, -1.0, -1.0]), np.zeros(3))  # looking away from the wall
    tf.raycast(vol, away, small_intr, rm, params)
    assert np.isinf(rm.distance).all() and not rm.valid.any()


def test_device_track_matches_host_loop():
    """tf_icp_track (whole pyramid on the device) vs the host-loop track_host
    (numpy 6x6 gate / solve / pose update): same lost flags and counts, poses
    equal to rounding, over an orbit with real motion between frames."""
    from paper_1511_07106_b200.tracking import track_host
    cfg = small_config(use_groundtruth=True)
    intr = cfg.intrinsics()
    frames, poses = render_orbit(intr, 8, step_deg=1.5)
    pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp())
    params = tf.TrackingParams(min_correspondences=300)
    checked = 0
    for i, (f, p) in enumerate(zip(frames, poses)):
        if i > 0:
            model, model_pose = pipe._model, pipe._model_pose
            for init in (None, poses[i - 1].compose(tf.Pose(rotation_from_axis_angle(
                    np.array([0.3, 1.0, 0.0]), np.radians(0.7)), np.array([0.004, -0.002, 0.003])))):
                a = tf.track(f, intr, model, model_pose, params, init=init)
                b = track_host(f, intr, model, model_pose, params, init=init)
                assert a.lost == b.lost and a.correspondences == b.correspondences
                assert abs(a.residual_rms - b.residual_rms) <= 1e-12 + 1e-9 * b.residual_rms
                # (acos of the trace amplifies 1e-16 to 1e-8 near identity: compare entries)
                assert np.abs(a.pose.rotation - b.pose.rotation).max() < 1e-12
                assert np.abs(a.pose.translation - b.pose.translation).max() < 1e-12
                checked += 1
        pipe.step(f, p)
    assert checked == 14
    # a lost case agrees too: far too few pairs required
    strict = tf.TrackingParams(min_correspondences=10 ** 7)
    a = tf.track(frames[1], intr, pipe._model, pipe._model_pose, strict)
    b = track_host(frames[1], intr, pipe._model, pipe._model_pose, strict)
    assert a.lost and b.lost and a.pose == b.pose


def test_lone_sphere_is_degenerate_on_the_device(small_intr):
    """test_tracking.py:132-152: exact sphere geometry leaves rotations about the
    centre unobservable; the conditioning gate (now evaluated on the device)
    must report lost, as the numpy host loop does."""
    from paper_1511_07106_b200.synth import Scene, Sphere
    from paper_1511_07106_b200.tracking import track_host
    scene = Scene((Sphere(np.array([0.0, 0.0, 1.5]), 0.45),))
    pose = tf.Pose.identity()
    frame = scene.render_depth(pose, small_intr)
    rays = small_intr.pixel_rays()
    unit = rays / np.linalg.norm(rays, axis=-1, keepdims=True)
    t = scene.primitives[0].intersect(np.zeros(3), unit.reshape(-1, 3)).reshape(unit.shape[:2])
    hit = np.isfinite(t)
    vertices = unit * np.where(hit, t, 0.0)[..., None]
    normals = np.where(hit[..., None], (vertices - np.array([0.0, 0.0, 1.5])) / 0.45, 0.0)
    model = tf.RayMap(vertices=vertices, normals=normals, distance=np.where(hit, t, np.inf))
    params = tf.TrackingParams(min_correspondences=200)
    assert tf.track(frame, small_intr, model, pose, params).lost
    assert track_host(frame, small_intr, model, pose, params).lost


def test_track_lost_cases(small_intr):
    scene = demo_scene()
    pose = tf.Pose.identity()
    vol = tf.TsdfSubvolume.empty(np.array([-50, -50, 24]), 100, 2.5)
    params = tf.FusionParams.for_voxel_size(0.025)
    tf.integrate(vol, scene.render_depth(pose, small_intr), pose, small_intr, params)
    model = tf.RayMap.empty(small_intr)
    tf.raycast(vol, pose, small_intr, model, params)
    tp = tf.TrackingParams(min_correspondences=200)
    empty = scene.render_depth(pose, small_intr)
    empty.data[:] = 0.0
    res = tf.track(empty, small_intr, model, pose, tp)
    assert res.lost and np.array_equal(res.pose.rotation, pose.rotation)
    seed = tf.Pose(np.eye(3), np.array([5.0, 5.0, 5.0]))
    res = tf.track(scene.render_depth(pose, small_intr), small_intr, model, pose, tp, init=seed)
    assert res.lost and np.array_equal(res.pose.translation, seed.translation)
    good = tf.track(scene.render_depth(pose, small_intr), small_intr, model, pose, tp)
    assert not good.lost and good.correspondences > 1000
