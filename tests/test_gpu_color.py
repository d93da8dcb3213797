"""Colour channel (north_star; absent from the reference, so parity is
unpinned against it): the device rule is checked against a numpy restatement
of the same rule, bit for bit, and for consistency between the float32-screened
and the reference-order integration paths."""

import numpy as np
import pytest
import torch

import paper_1511_07106_b200 as tf
from paper_1511_07106_b200 import _native as nat
from paper_1511_07106_b200.geometry import CameraIntrinsics
from paper_1511_07106_b200.synth import demo_scene, render_rgb

pytestmark = pytest.mark.gpu

INTR = CameraIntrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)


def numpy_color_fusion(origin, n, vs, tau, frames):
    """The colour rule of tf_integrate_rgb (include/tfb200.h) in numpy: the
    reference's integration gates and float64 orders (_kernels.py:99-128)
    pick each voxel's pixel; voxels with sdf < tau take the running mean."""
    color = np.zeros((n, n, n, 4), dtype=np.uint8)
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    gx = (x + float(origin[0])) * vs
    gy = (y + float(origin[1])) * vs
    gz = (z + float(origin[2])) * vs
    for depth, rgb, pose in frames:
        inv = pose.invert()
        R, t, c = inv.rotation, inv.translation, pose.translation
        pcx = ((R[0, 0] * gx + R[0, 1] * gy) + R[0, 2] * gz) + t[0]
        pcy = ((R[1, 0] * gx + R[1, 1] * gy) + R[1, 2] * gz) + t[1]
        pcz = ((R[2, 0] * gx + R[2, 1] * gy) + R[2, 2] * gz) + t[2]
        ok = pcz > 0
        with np.errstate(divide="ignore", invalid="ignore"):
            u = (INTR.fx * pcx) / pcz + INTR.cx
            v = (INTR.fy * pcy) / pcz + INTR.cy
        ui, vi = np.floor(u + 0.5), np.floor(v + 0.5)
        ok &= (ui >= 0) & (ui < INTR.width) & (vi >= 0) & (vi < INTR.height)
        uu, vv = np.where(ok, ui, 0).astype(np.int64), np.where(ok, vi, 0).astype(np.int64)
        d = depth[vv, uu]
        ok &= d > 0
        rx, ry = (uu - INTR.cx) / INTR.fx, (vv - INTR.cy) / INTR.fy
        rs = np.sqrt((rx * rx + ry * ry) + 1.0)
        ddx, ddy, ddz = gx - c[0], gy - c[1], gz - c[2]
        dist = np.sqrt((ddx * ddx + ddy * ddy) + ddz * ddz)
        sdf = d - dist / rs
        band = ok & (sdf >= -tau) & (sdf < tau)
        obs = rgb[vv, uu].astype(np.float32)
        w = color[..., 3].astype(np.float32)
        for ch in range(3):
            new = np.rint((w * color[..., ch].astype(np.float32) + obs[..., ch]) / (w + np.float32(1)))
            color[..., ch] = np.where(band, new.astype(np.uint8), color[..., ch])
        color[..., 3] = np.where(band, np.minimum(color[..., 3].astype(np.int32) + 1, 255), color[..., 3])
    return color


def test_color_rule_matches_numpy_restatement():
    scene = demo_scene()
    vol = tf.TsdfSubvolume.empty(np.array([-30, -10, 20]), 48, 48 * 0.025).enable_color()
    params = tf.FusionParams.for_voxel_size(vol.voxel_size)
    frames = []
    for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 24)[:3]:
        depth = scene.render_depth(pose, INTR)
        rgb = render_rgb(scene, pose, INTR)
        tf.integrate(vol, depth, pose, INTR, params, color=rgb)
        frames.append((depth.data, rgb, pose))
    want = numpy_color_fusion(vol.origin_voxel, 48, vol.voxel_size, params.truncation, frames)
    got = vol.color.cpu().numpy()
    assert (want[..., 3] > 0).sum() > 1000
    assert np.array_equal(got, want)


def test_color_fast_path_equals_exact_path():
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    a = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length).enable_color()
         for k in spec.keys]
    b = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length).enable_color()
         for k in spec.keys]
    scene = demo_scene()
    lib = nat.load_library()
    try:
        for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 24)[:5]:
            depth, rgb = scene.render_depth(pose, INTR), render_rgb(scene, pose, INTR)
            lib.tf_set_debug_flags(0)
            tf.integrate_volumes(a, depth, pose, INTR, params, color=rgb)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.integrate_volumes(b, depth, pose, INTR, params, color=rgb)
    finally:
        lib.tf_set_debug_flags(0)
    for x, y in zip(a, b):
        assert torch.equal(x.voxels, y.voxels) and torch.equal(x.color, y.color)
    assert sum(int((x.color[..., 3] > 0).sum()) for x in a) > 10000


def test_raycast_colors_reproduce_the_scene():
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length).enable_color()
             for k in spec.keys]
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 48)
    for pose in poses[:6]:
        tf.integrate_volumes(tiles, scene.render_depth(pose, INTR), pose, INTR, params,
                             color=render_rgb(scene, pose, INTR, square=0.5))
    rm = tf.RayMap.empty(INTR)
    tf.raycast_volumes(tiles, poses[3], INTR, rm, params)
    col = tf.raycast_colors(tiles, rm, poses[3], INTR).cpu().numpy()
    ref = render_rgb(scene, poses[3], INTR, square=0.5).astype(np.float32)
    hit = np.isfinite(rm.distance)
    coloured = hit & (col.sum(-1) > 0)
    assert coloured.sum() > 0.8 * hit.sum() > 3000
    err = np.abs(col[coloured] - ref[coloured]).max(axis=-1)
    # (colours bleed across primitive boundaries within the +-tau band)
    assert np.median(err) < 2.0 and np.mean(err < 25.0) > 0.8
    assert not col[~hit].any()


def test_host_tier_keeps_color(tmp_path):
    params = tf.FusionParams.for_voxel_size(0.1)
    vs = tf.VolumeSet(params, 10, 0.1, max_resident=1, spill_dir=tmp_path, spill_tier="host")
    vs.add((-4, -4, 16))
    vs.add((4, -4, 16))
    vol = vs.acquire((-4, -4, 16)).enable_color()
    vol.color[1, 2, 3] = torch.tensor([10, 20, 30, 4], dtype=torch.uint8)
    vs.release((-4, -4, 16))
    vs.acquire((4, -4, 16))  # spills the first tile to pinned host memory
    vs.release((4, -4, 16))
    back = vs.acquire((-4, -4, 16))
    assert back.color is not None and back.color[1, 2, 3].tolist() == [10, 20, 30, 4]


def test_pipeline_with_color(tmp_path):
    cfg = tf.RunConfig(fx=131.25, fy=131.25, cx=79.5, cy=59.5, width=160, height=120, side_length=3.0,
                       resolution=124, resident_resolution=62, use_groundtruth=True, color=True)
    pipe = tf.FusionPipeline(cfg, tmp_path)
    scene = demo_scene()
    for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 48)[:4]:
        pipe.step(scene.render_depth(pose, INTR), pose, color=render_rgb(scene, pose, INTR))
    assert pipe.model_colors is not None and pipe.model_colors.shape == (120, 160, 3)
    assert float(pipe.model_colors.sum()) > 0
    assert all(v.color is not None for _, v in pipe.volumes.resident_volumes())
