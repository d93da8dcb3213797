"""Randomised stress of the exact-by-construction fast paths:
random camera poses (including cameras inside a volume and near its faces),
random intrinsics, image sizes, voxel sizes, truncation scales and weight
caps.  Per case the float32-screened / culled integration must equal the
exact integration (TF_DEBUG_EXACT_ONLY) bit for bit, and the certified
raycast (per-lane and the cooperative pass) the exact march bit for bit, with
no certification failure.  Seeds are fixed: a failure names its case."""

import os

import numpy as np
import pytest
import torch

import paper_1511_07106_b200 as tf
from paper_1511_07106_b200 import _native as nat
from paper_1511_07106_b200.geometry import CameraIntrinsics, Pose, rotation_from_axis_angle
from paper_1511_07106_b200.synth import demo_scene

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(seed)
    w = int(rng.choice([64, 96, 160, 200]))
    h = int(rng.choice([48, 72, 120, 150]))
    f = float(rng.uniform(0.6, 1.4) * w)
    intr = CameraIntrinsics(f, f * float(rng.uniform(0.9, 1.1)), (w - 1) / 2 + float(rng.uniform(-5, 5)),
                            (h - 1) / 2 + float(rng.uniform(-5, 5)), w, h)
    n = int(rng.choice([40, 64, 96]))
    vs = float(rng.uniform(0.006, 0.03))
    origin = tuple(int(x) for x in rng.integers(-n, 0, size=3))
    origin = (origin[0], origin[1], int(rng.integers(0, n // 2)))
    scale = float(rng.choice([3.0, 4.0, 6.0]))
    params = tf.FusionParams(truncation=scale * vs, max_weight=float(rng.choice([3.0, 16.0, 128.0])),
                             sample_weight=float(rng.choice([1.0, 1.0, 0.5, 2.0])))
    # cameras around the scene centre; some inside the volume / near a face
    centre = np.array([0.1, 0.05, 1.5])
    poses = []
    for k in range(4):
        if rng.random() < 0.3:  # inside / at the boundary of the volume
            lo = np.array(origin) * vs
            cam = lo + rng.uniform(-0.05, 0.3, size=3) * n * vs
        else:
            cam = centre + rng.normal(0, 1, size=3) * np.array([0.8, 0.3, 0.8])
            cam[2] = min(cam[2], 0.9)
        fwd = centre - cam
        fwd /= np.linalg.norm(fwd)
        axis = np.cross([0.0, 0.0, 1.0], fwd)
        ang = float(np.arccos(np.clip(fwd[2], -1, 1)))
        rot = rotation_from_axis_angle(axis, ang) if np.linalg.norm(axis) > 1e-9 else np.eye(3)
        rot = rot @ rotation_from_axis_angle(np.array([0.0, 0.0, 1.0]), float(rng.uniform(-0.3, 0.3)))
        poses.append(Pose(rot, cam))
    return intr, n, vs, origin, params, poses


# TFB200_STRESS_CASES widens the sweep (DESIGN.md §3 records a 20 000-case run)
@pytest.mark.parametrize("seed", range(int(os.environ.get("TFB200_STRESS_CASES", "24"))))
def test_fast_paths_equal_exact_random_cases(seed):
    intr, n, vs, origin, params, poses = _case(seed)
    scene = demo_scene()
    lib = nat.load_library()
    a = tf.TsdfSubvolume.empty(origin, n, n * vs)
    b = tf.TsdfSubvolume.empty(origin, n, n * vs)
    stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    try:
        for k, pose in enumerate(poses):
            frame = scene.render_depth(pose, intr)
            lib.tf_set_debug_flags(0)
            tf.integrate_volumes([a], frame, pose, intr, params)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.integrate_volumes([b], frame, pose, intr, params)
            lib.tf_set_debug_flags(0)
            assert torch.equal(a.voxels, b.voxels), f"seed {seed}: integration, pose {k}"
            exact = tf.RayMap.empty(intr)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.raycast_volumes([b], pose, intr, exact, params)
            for flag in (0, nat.DEBUG_COOP_ALL):
                got = tf.RayMap.empty(intr)
                lib.tf_set_debug_flags(flag)
                tf.raycast_volumes([a], pose, intr, got, params, stats)
                assert torch.equal(got.distance_dev, exact.distance_dev), f"seed {seed} pose {k} flag {flag}"
                assert torch.equal(got.vertices_dev, exact.vertices_dev)
                assert torch.equal(got.normals_dev, exact.normals_dev)
    finally:
        lib.tf_set_debug_flags(0)
    assert stats[nat.STAT_CERT_FAILURES].item() == 0
