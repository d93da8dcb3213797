"""Host-side logic on CPU: placement policy, grid layout, config, pose algebra,
the synthetic renderer and the spill format — against known answers from the
reference's own tests and (in the build container) the live reference."""

import numpy as np
import pytest

from paper_1511_07106_b200 import config as cfg
from paper_1511_07106_b200.geometry import (CameraIntrinsics, DepthFrame, Pose, rotation_angle,
                                           rotation_from_axis_angle)
from paper_1511_07106_b200.synth import (Box, Plane, Scene, Sphere, corridor_trajectory,
                                        demo_scene, orbit_trajectory, parse_scene, format_scene)
from paper_1511_07106_b200.volumes import (AllocationPolicy, init_grid, spill_file_size,
                                          update_allocation)

from conftest import load_golden, reference_module


# ---- update_allocation known answers (reference test_volumes.py:269-304) ----------

def test_allocation_fills_free_slots_by_count():
    added, removed = update_allocation([], {(0, 0, 0): 5, (30, 0, 0): 9, (60, 0, 0): 1},
                                       AllocationPolicy(max_volumes=2))
    assert (added, removed) == ([(30, 0, 0), (0, 0, 0)], [])


def test_allocation_hysteresis():
    pol = AllocationPolicy(max_volumes=1, hysteresis=1.5)
    assert update_allocation([(0, 0, 0)], {(0, 0, 0): 10, (30, 0, 0): 14}, pol) == ([], [])
    assert update_allocation([(0, 0, 0)], {(0, 0, 0): 10, (30, 0, 0): 16}, pol) == (
        [(30, 0, 0)], [(0, 0, 0)])


def test_allocation_zero_counts_and_lexicographic_ties():
    added, removed = update_allocation([], {(30, 0, 0): 4, (0, 30, 0): 4, (60, 0, 0): 0},
                                       AllocationPolicy(max_volumes=2))
    assert (added, removed) == ([(0, 30, 0), (30, 0, 0)], [])


def test_allocation_unseen_incumbent_counts_zero():
    pol = AllocationPolicy(max_volumes=1, hysteresis=1.5)
    assert update_allocation([(0, 0, 0)], {(30, 0, 0): 1}, pol) == ([(30, 0, 0)], [(0, 0, 0)])


def test_allocation_policy_validation():
    with pytest.raises(ValueError):
        AllocationPolicy(max_volumes=0)
    with pytest.raises(ValueError):
        AllocationPolicy(max_volumes=1, hysteresis=0.5)


def test_allocation_matches_reference_randomized():
    ref = reference_module()
    from tilefusion.volumes import AllocationPolicy as RP, update_allocation as rua
    rng = np.random.default_rng(5)
    for _ in range(300):
        keys = [tuple(int(v) * 30 for v in rng.integers(-3, 4, 3)) for _ in range(rng.integers(0, 14))]
        counts = {k: int(rng.integers(0, 60)) for k in keys}
        cur = list(dict.fromkeys(keys[: rng.integers(0, 6)]))
        mv, hy = int(rng.integers(1, 7)), float(rng.choice([1.0, 1.5, 2.0]))
        assert update_allocation(cur, counts, AllocationPolicy(mv, hy)) == rua(cur, counts, RP(mv, hy))


# ---- grid layout (reference test_volumes.py:81-114) ----------------------------------

def test_init_grid_layout():
    g = init_grid(3.0, 124, 62)
    assert g.voxels_per_side == 64 and g.spacing == 62 and len(g.keys) == 8
    assert g.keys[0] == (-63, -63, 0) and g.keys[-1] == (-1, -1, 62)
    assert g.voxel_size == pytest.approx(3.0 / 124)
    c3 = init_grid(4.08, 1020, 510)
    assert c3.voxels_per_side == 512 and len(c3.keys) == 8 and c3.voxel_size == pytest.approx(0.004)
    with pytest.warns(UserWarning):
        assert len(init_grid(3.0, 100, 30).keys) == 64
    with pytest.raises(ValueError):
        init_grid(3.0, 10, 20)


def test_init_grid_matches_reference():
    ref = reference_module()
    for args in [(3.0, 124, 62), (4.08, 1020, 510), (1.8, 28, 14), (3.0, 254, 254)]:
        a, b = init_grid(*args), ref.init_grid(*args)
        assert (a.voxels_per_side, a.voxel_size, a.spacing, a.keys) == (
            b.voxels_per_side, b.voxel_size, b.spacing, b.keys)


def test_spill_file_size():
    assert spill_file_size(16) == 52 + 16 ** 3 * 8


# ---- config (reference test_config.py) ---------------------------------------------------

def test_config_defaults_and_validation(tmp_path):
    c = cfg.RunConfig()
    assert (c.cx, c.cy, c.width, c.height) == (319.5, 239.5, 640, 480)
    assert c.validate() == []
    bad = cfg.RunConfig(fx=-1, max_resident=0, iterations=(), spill_tier="tape")
    errs = bad.validate()
    assert any("focal" in e for e in errs) and any("max_resident" in e for e in errs)
    assert any("spill_tier" in e for e in errs)
    cfg.save_config(tmp_path / "a.ini", cfg.RunConfig(resolution=200, iterations=(3, 2),
                                                        spill_tier="host"))
    back = cfg.load_config(tmp_path / "a.ini")
    assert back.resolution == 200 and back.iterations == (3, 2) and back.spill_tier == "host"
    (tmp_path / "b.ini").write_text("[camera]\nfx = 1\nbogus = 2\n[nope]\nx = 1\n")
    with pytest.raises(ValueError, match="unknown"):
        cfg.load_config(tmp_path / "b.ini")


# ---- pose algebra & renderer -----------------------------------------------------------------

def test_pose_algebra():
    rng = np.random.default_rng(1)
    for _ in range(20):
        r = rotation_from_axis_angle(rng.normal(size=3), rng.uniform(0, np.pi))
        p = Pose(r, rng.normal(size=3))
        ident = p.compose(p.invert())
        assert np.allclose(ident.matrix, np.eye(4), atol=1e-12)
        q = Pose.from_quaternion(*p.translation, *p.quaternion())
        assert np.allclose(q.matrix, p.matrix, atol=1e-12)
        assert rotation_angle(p.orthonormalized().rotation @ p.rotation.T) < 1e-7
    with pytest.raises(ValueError):
        Pose(np.diag([1.0, 1.0, -1.0]), np.zeros(3))
    with pytest.raises(ValueError):
        DepthFrame(np.array([[1.0, -1.0]]))


def test_pose_math_bit_identical_to_reference():
    ref = reference_module()
    rng = np.random.default_rng(2)
    for _ in range(50):
        r = rotation_from_axis_angle(rng.normal(size=3), rng.uniform(0, np.pi))
        t = rng.normal(size=3)
        a, b = Pose(r, t), ref.Pose(r, t)
        assert np.array_equal(a.invert().rotation, b.invert().rotation)
        assert np.array_equal(a.invert().translation, b.invert().translation)
        d = rng.normal(size=6) * 0.01
        from paper_1511_07106_b200.tracking import apply_delta
        from tilefusion.geometry import rotation_from_axis_angle as rr
        rot = rr(d[:3], float(np.linalg.norm(d[:3])))
        want = ref.Pose(rot @ b.rotation, rot @ b.translation + d[3:]).orthonormalized()
        got = apply_delta(a, d)
        assert np.array_equal(got.matrix, want.matrix)


def test_renderer_reproduces_golden_frames():
    g = load_golden("fusion_small.npz")
    a = g["intr"]
    intr = CameraIntrinsics(a[0], a[1], a[2], a[3], int(a[4]), int(a[5]))
    for frame, m in zip(g["frames"], g["poses"]):
        got = demo_scene().render_depth(Pose(m[:3, :3], m[:3, 3]), intr).data
        assert np.array_equal(got, frame)


def test_scene_text_format_round_trip():
    s = Scene((Sphere(np.array([0.0, 0.0, 1.5]), 0.5), Plane((0, 0.5, 0), (0, -1, 0)),
               Box((-1, -1, 1), (0, 0, 2))))
    back = parse_scene(format_scene(s))
    assert len(back.primitives) == 3
    with pytest.raises(ValueError):
        parse_scene("cone 1 2 3\n")


def test_trajectories():
    orbit = orbit_trajectory((0, 0, 1.5), 1.5, 8)
    assert np.allclose(orbit[0].matrix, np.eye(4))
    assert np.allclose(orbit[2].translation, [-1.5, 0.0, 1.5])
    walk = corridor_trajectory(4.0, 5)
    assert np.allclose(walk[-1].translation, [0, 0, 4.0])
