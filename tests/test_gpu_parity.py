"""CUDA path (libtfb200 through the package API) vs the golden vectors and the
oracle.  Bit-exact for integration (tsdf AND weights), raycast maps,
extraction, vertex/normal maps and endpoint cells; ICP inlier counts exact,
pose increments within 1e-5 m / 1e-6 rad."""

import numpy as np
import pytest
import torch

import oracle
import paper_1511_07106_b200 as tf
from paper_1511_07106_b200 import _native as nat
from paper_1511_07106_b200 import tracking as trk
from paper_1511_07106_b200.geometry import CameraIntrinsics, Pose
from paper_1511_07106_b200.synth import demo_scene

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _intr(a) -> CameraIntrinsics:
    return CameraIntrinsics(float(a[0]), float(a[1]), float(a[2]), float(a[3]), int(a[4]), int(a[5]))


def _pose(m) -> Pose:
    return Pose(m[:3, :3], m[:3, 3])


def test_native_library_is_the_one_loaded():
    lib = nat.load_library()
    assert lib.tf_abi_version() == nat.ABI_VERSION
    assert torch.cuda.is_available()


def test_fusion_fixture_bit_exact():
    g = load_golden("fusion_small.npz")
    intr = _intr(g["intr"])
    n = int(g["n"])
    vol = tf.TsdfSubvolume.empty(g["origin"], n, float(g["side"]))
    params = tf.FusionParams(float(g["tau"]), float(g["max_weight"]), float(g["sample_weight"]))
    for k, (frame, m) in enumerate(zip(g["frames"], g["poses"])):
        tf.integrate(vol, tf.DepthFrame(frame), _pose(m), intr, params)
        pair = vol.voxels.cpu().numpy()
        assert np.array_equal(pair[..., 0], g["tsdf_after"][k]), f"tsdf after frame {k}"
        assert np.array_equal(pair[..., 1], g["weight_after"][k]), f"weight after frame {k}"
    for i, pi in enumerate(g["ray_pose_index"]):
        rm = tf.RayMap.empty(intr)
        tf.raycast(vol, _pose(g["poses"][pi]), intr, rm, params)
        assert np.array_equal(rm.distance, g["ray_dist"][i])
        assert np.array_equal(rm.vertices, g["ray_vert"][i])
        assert np.array_equal(rm.normals, g["ray_norm"][i])
    cloud = tf.extract_points(vol)
    assert np.array_equal(cloud.vertices, g["cloud_verts"])
    assert np.array_equal(cloud.normals, g["cloud_norms"])


def test_tiled_fixture_fused_launch_bit_exact():
    g = load_golden("tiled_small.npz")
    intr = _intr(g["intr"])
    n = int(g["n"])
    params = tf.FusionParams.for_voxel_size(float(g["side"]) / n)
    assert params.truncation == float(g["tau"])
    tiles = [tf.TsdfSubvolume.empty(k, n, float(g["side"])) for k in g["keys"]]
    for f, (frame, m) in enumerate(zip(g["frames"], g["poses"])):
        pose = _pose(m)
        tf.integrate_volumes(tiles, tf.DepthFrame(frame), pose, intr, params)
        rm = tf.RayMap.empty(intr)
        tf.raycast_volumes(tiles, pose, intr, rm, params)
        assert np.array_equal(rm.distance, g["ray_dist"][f])
        assert np.array_equal(rm.vertices, g["ray_vert"][f])
        assert np.array_equal(rm.normals, g["ray_norm"][f])
    for i, t in enumerate(tiles):
        assert np.array_equal(t.tsdf, g["tsdf"][i])
        assert np.array_equal(t.weight, g["weight"][i])


def test_vertex_normal_maps_bit_exact():
    g = load_golden("icp_small.npz")
    intr = _intr(g["intr"])
    depth = torch.as_tensor(g["frame"], device="cuda")
    for level in range(3):
        lv = trk.source_level(depth, intr, level)
        assert np.array_equal(lv.verts.cpu().numpy(), g[f"vn{level}_verts"])
        assert np.array_equal(lv.norms.cpu().numpy(), g[f"vn{level}_norms"])
        assert np.array_equal(lv.valid.cpu().numpy().astype(bool), g[f"vn{level}_valid"])
        intr = intr.scaled(0.5)


def test_icp_steps_match_reference():
    g = load_golden("icp_small.npz")
    intr0 = _intr(g["intr"])
    model = tf.RayMap(g["model_vert"], g["model_norm"], g["model_dist"])
    depth = torch.as_tensor(g["frame"], device="cuda")
    params = tf.TrackingParams(max_distance=float(g["max_distance"]),
                               max_angle_deg=float(g["max_angle_deg"]),
                               iterations=tuple(int(i) for i in g["iterations"]),
                               min_correspondences=int(g["min_correspondences"]))
    levels = {}
    intr = intr0
    for level in range(3):
        levels[intr.width] = trk.source_level(depth, intr, level)
        intr = intr.scaled(0.5)
    ref_inv = _pose(g["ref_pose"]).invert()
    for k in range(len(g["step_count"])):
        src = levels[int(g["step_level_w"][k])]
        step = trk.solve_step(src, model, _pose(g["step_estimate"][k]), ref_inv, params,
                              int(g["step_min_pairs"][k]))
        if g["step_count"][k] < 0:
            assert step is None
            continue
        delta, count, rms = step
        assert count == g["step_count"][k], f"step {k}"
        assert np.abs(delta[:3] - g["step_delta"][k][:3]).max() <= 1e-6
        assert np.abs(delta[3:] - g["step_delta"][k][3:]).max() <= 1e-5
    res = tf.track(tf.DepthFrame(g["frame"]), intr0, model, _pose(g["ref_pose"]), params,
                   init=_pose(g["seed_pose"]))
    assert res.lost == bool(g["result_lost"])
    assert res.correspondences == int(g["result_count"])
    assert np.abs(res.pose.matrix - g["result_pose"]).max() < 1e-9


def test_bin_endpoints_match_reference():
    g = load_golden("endpoints_small.npz")
    intr = _intr(g["intr"])
    for f in range(len(g["frames"])):
        got = tf.bin_endpoints(tf.DepthFrame(g["frames"][f]), intr, _pose(g["poses"][f]),
                               int(g["spacing"]), float(g["voxel_size"]))
        lo, hi = g["offsets"][f], g["offsets"][f + 1]
        want = {tuple(int(x) for x in g["keys"][i]): int(g["counts"][i]) for i in range(lo, hi)}
        assert got == want


# ---------------------------------------------------------------------------
# the CUDA path vs the oracle at the benchmark camera and volume sizes
# ---------------------------------------------------------------------------

def _oracle_integrate(tsdf, weight, vol, frame, pose, intr, params, threads=8):
    inv = pose.invert()
    return oracle.integrate(tsdf, weight, vol.origin_voxel, vol.voxel_size, frame, inv.rotation,
                            inv.translation, pose.translation, intr.fx, intr.fy, intr.cx,
                            intr.cy, params.truncation, params.max_weight, params.sample_weight,
                            threads=threads)


def test_config1_volume_256_bit_exact_vs_oracle():
    """Config 1 geometry (one 256^3 tile, 640x480, demo orbit), 4 frames."""
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(3.0, 254, 254)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    vol = tf.TsdfSubvolume.empty(spec.keys[0], spec.voxels_per_side, spec.subvolume_side_length)
    n = spec.voxels_per_side
    t = np.zeros((n, n, n), np.float32)
    w = np.zeros((n, n, n), np.float32)
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)[:4]
    stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    for pose in poses:
        frame = scene.render_depth(pose, intr)
        stats.zero_()
        tf.integrate_volumes([vol], frame, pose, intr, params, stats)
        want = _oracle_integrate(t, w, vol, frame.data, pose, intr, params)
        got = int(stats[nat.STAT_VOXEL_UPDATES].item())
        assert got == want
        pair = vol.voxels.cpu().numpy()
        assert np.array_equal(pair[..., 0], t)
        assert np.array_equal(pair[..., 1], w)
    rm = tf.RayMap.empty(intr)
    tf.raycast(vol, poses[-1], intr, rm, params)
    d = np.full((intr.height, intr.width), np.inf)
    v = np.zeros((intr.height, intr.width, 3))
    nn = np.zeros_like(v)
    oracle.raycast(t, w, vol.origin_voxel, vol.voxel_size, params.truncation,
                   tf.tsdf.coarse_step(params, vol.voxel_size), poses[-1].rotation,
                   poses[-1].translation, intr.fx, intr.fy, intr.cx, intr.cy, d, v, nn, threads=8)
    assert np.isfinite(d).sum() > 100000
    assert np.array_equal(rm.distance, d)
    assert np.array_equal(rm.vertices, v)
    assert np.array_equal(rm.normals, nn)


def test_culling_never_drops_an_update():
    """Full-size property: culled and unculled sweeps are bitwise identical."""
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)  # config 3: 8 x 512^3 at 4 mm
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    keys = spec.keys[:2]
    a = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in keys]
    b = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in keys]
    scene = demo_scene()
    lib = nat.load_library()
    sa = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    sb = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    try:
        for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)[:3]:
            frame = scene.render_depth(pose, intr)
            lib.tf_set_debug_flags(0)
            tf.integrate_volumes(a, frame, pose, intr, params, sa)
            lib.tf_set_debug_flags(nat.DEBUG_NO_CULL)
            tf.integrate_volumes(b, frame, pose, intr, params, sb)
    finally:
        lib.tf_set_debug_flags(0)
    assert sa[nat.STAT_VOXEL_UPDATES].item() == sb[nat.STAT_VOXEL_UPDATES].item() > 0
    assert sa[nat.STAT_SWEPT_VOXELS].item() < sb[nat.STAT_SWEPT_VOXELS].item()
    for x, y in zip(a, b):
        assert torch.equal(x.voxels, y.voxels)


def test_fused_raycast_equals_per_volume_any_order():
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length)
             for k in spec.keys]
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 16)
    for pose in poses[:4]:
        tf.integrate_volumes(tiles, scene.render_depth(pose, intr), pose, intr, params)
    fused = tf.RayMap.empty(intr)
    tf.raycast_volumes(tiles, poses[1], intr, fused, params)
    order = np.random.default_rng(7).permutation(len(tiles))
    single = tf.RayMap.empty(intr)
    for i in order:
        tf.raycast(tiles[i], poses[1], intr, single, params)
    assert np.isfinite(fused.distance).sum() > 50000
    assert torch.equal(fused.distance_dev, single.distance_dev)
    assert torch.equal(fused.vertices_dev, single.vertices_dev)
    assert torch.equal(fused.normals_dev, single.normals_dev)


def test_table_division_is_ieee():
    """The running-mean division by integral weights (table reciprocal + FMA
    correction) equals IEEE division on 400 M random pairs."""
    lib = nat.load_library()
    for seed in (1, 2, 3, 4):
        assert lib.tf_debug_weight_division_check(100_000_000, seed) == 0


def test_certified_voxel_size_division_is_ieee():
    """The raycast's exact path divides by the voxel size with a reciprocal, one
    Newton correction and an exact remainder test that falls back to the IEEE
    division whenever it cannot prove the quotient correctly rounded: equal to
    __ddiv_rn bit for bit on 400 M random and adversarial pairs (multiples and
    half-multiples of b and their neighbours, perturbed reciprocals)."""
    lib = nat.load_library()
    for seed in (1, 2, 3, 4):
        assert lib.tf_debug_div_check(100_000_000, seed) == 0


def test_division_free_ray_interval_is_exact():
    """The raycast's ray/box interval from products with 1/d and 1/vs (with its
    certified margins and exact fallback) equals the reference's divisions
    (_kernels.py:299-348) on 400 M random and adversarial (volume, ray) pairs:
    origins on box faces, zero and 1e-16 direction components, entry t an
    integer multiple of the voxel size."""
    lib = nat.load_library()
    for seed in (1, 2, 3, 4):
        assert lib.tf_debug_ray_interval_check(100_000_000, seed) == 0


@pytest.mark.parametrize("sw,max_w", [(0.75, 128.0), (1.0, 5.0), (2.5, 10.0)])
def test_fractional_and_capped_weights(sw, max_w):
    """Non-integral running-mean denominators (the division falls back from
    the reciprocal table), low caps (the fixed point and the weight cap):
    float32-screened integration == exact integration, bit for bit."""
    intr = CameraIntrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams(truncation=4 * spec.voxel_size, max_weight=max_w, sample_weight=sw)
    a = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    b = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    scene = demo_scene()
    lib = nat.load_library()
    try:
        for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 24)[:8]:
            frame = scene.render_depth(pose, intr)
            lib.tf_set_debug_flags(0)
            tf.integrate_volumes(a, frame, pose, intr, params)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.integrate_volumes(b, frame, pose, intr, params)
    finally:
        lib.tf_set_debug_flags(0)
    for x, y in zip(a, b):
        assert torch.equal(x.voxels, y.voxels)
    assert float(a[0].voxels[..., 1].max()) > 0


@pytest.mark.parametrize("scale", [6.0, 8.0, 13.0])
def test_coarse_strides_above_two(scale):
    """Wider truncation -> coarse stride round(0.5 tau / vs) of 3, 4, 6: the
    certified per-lane march and the cooperative march equal the exact
    reference march (their coarse == 2 fast paths are not taken)."""
    intr = CameraIntrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size, truncation_scale=scale)
    assert tf.tsdf.coarse_step(params, spec.voxel_size) == round(0.5 * scale)
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 24)
    for pose in poses[:5]:
        tf.integrate_volumes(tiles, scene.render_depth(pose, intr), pose, intr, params)
    lib = nat.load_library()
    stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    try:
        for pose in (poses[2], poses[7]):
            exact = tf.RayMap.empty(intr)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.raycast_volumes(tiles, pose, intr, exact, params)
            assert torch.isfinite(exact.distance_dev).sum().item() > 2000
            for flag in (0, nat.DEBUG_COOP_ALL):
                got = tf.RayMap.empty(intr)
                lib.tf_set_debug_flags(flag)
                tf.raycast_volumes(tiles, pose, intr, got, params, stats)
                assert torch.equal(got.distance_dev, exact.distance_dev)
                assert torch.equal(got.vertices_dev, exact.vertices_dev)
                assert torch.equal(got.normals_dev, exact.normals_dev)
    finally:
        lib.tf_set_debug_flags(0)
    assert stats[nat.STAT_CERT_FAILURES].item() == 0


def test_more_volumes_than_one_launch_holds():
    """125 tiles (> TFB200_MAX_VOLUMES_PER_LAUNCH = 64): the chunked fused
    integrate / raycast equal per-tile calls bit for bit."""
    intr = CameraIntrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    spec = tf.init_grid(3.0, 100, 20)
    assert len(spec.keys) == 125
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    fused = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    single = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 16)
    for pose in poses[:3]:
        frame = scene.render_depth(pose, intr)
        tf.integrate_volumes(fused, frame, pose, intr, params)
        for v in single:
            tf.integrate(v, frame, pose, intr, params)
    for x, y in zip(fused, single):
        assert torch.equal(x.voxels, y.voxels)
    a = tf.RayMap.empty(intr)
    tf.raycast_volumes(fused, poses[1], intr, a, params)
    b = tf.RayMap.empty(intr)
    for v in single[::-1]:
        tf.raycast(v, poses[1], intr, b, params)
    assert np.isfinite(a.distance).sum() > 3000
    assert torch.equal(a.distance_dev, b.distance_dev)
    assert torch.equal(a.vertices_dev, b.vertices_dev)
    assert torch.equal(a.normals_dev, b.normals_dev)


def test_trilinear_sample_and_merge():
    g = load_golden("fusion_small.npz")
    n = int(g["n"])
    vol = tf.TsdfSubvolume(g["origin"], n, float(g["side"]), g["tsdf_after"][-1],
                           g["weight_after"][-1])
    rng = np.random.default_rng(0)
    lo = vol.world_min
    hi = vol.world_max
    t = g["tsdf_after"][-1]
    w = g["weight_after"][-1]
    for p in rng.uniform(lo, hi, size=(200, 3)):
        got = tf.trilinear_sample(vol, p)
        q = p / vol.voxel_size - vol.origin_voxel
        ok, val = oracle.sample(t, w, q[0], q[1], q[2])
        assert (got is not None) == ok
        if ok:
            assert got == val


def test_rowblock_merge_kernels():
    """tf_raymap_merge_packed == _hit_wins on packed records; tf_raymap_vertices
    rebuilds exactly the vertices tf_raycast wrote (the cross-GPU exchange)."""
    lib = nat.load_library()
    rng = torch.Generator().manual_seed(3)
    n = 4096
    a = torch.zeros(n, 4, dtype=torch.float64)
    b = torch.zeros(n, 4, dtype=torch.float64)
    for x in (a, b):
        x[:, 0] = torch.where(torch.rand(n, generator=rng) < 0.3, torch.full((n,), float("inf")),
                              torch.round(torch.rand(n, generator=rng) * 4) / 4)
        x[:, 1:] = torch.round(torch.rand(n, 3, generator=rng) * 2) / 2  # ties reach the normals
    want = a.clone()
    better = b[:, 0] < want[:, 0]
    tie = b[:, 0] == want[:, 0]
    for c in range(1, 4):
        neq = b[:, c] != want[:, c]
        better |= tie & neq & (b[:, c] > want[:, c])
        tie &= ~neq
    want[better] = b[better]
    got, src = a.cuda(), b.cuda()
    nat.check(lib.tf_raymap_merge_packed(nat.ptr(got), nat.ptr(src), n, nat.stream_handle()), "merge")
    assert torch.equal(got.cpu(), want)

    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(3.0, 254, 127)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length)
             for k in spec.keys]
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 32)
    for pose in poses[:4]:
        tf.integrate_volumes(tiles, demo_scene().render_depth(pose, intr), pose, intr, params)
    rm = tf.RayMap.empty(intr)
    tf.raycast_volumes(tiles, poses[5], intr, rm, params)
    assert torch.isfinite(rm.distance_dev).sum().item() > 10000
    vert = torch.full_like(rm.vertices_dev, 7.0)
    h = intr.height
    nat.check(lib.tf_raymap_vertices(nat.ptr(rm.distance_dev), 1, nat.ptr(vert), nat.camera(intr),
                                     nat.mat9(poses[5].rotation), nat.vec3(poses[5].translation), 0, h,
                                     nat.stream_handle()), "vertices")
    assert torch.equal(vert, rm.vertices_dev)
    # a row block alone, from a strided (packed) distance view
    packed = torch.cat([rm.distance_dev[..., None], rm.normals_dev], -1).contiguous()
    blk = torch.zeros((100, intr.width, 3), dtype=torch.float64, device="cuda")
    nat.check(lib.tf_raymap_vertices(nat.ptr(packed[200]), 4, nat.ptr(blk), nat.camera(intr),
                                     nat.mat9(poses[5].rotation), nat.vec3(poses[5].translation), 200,
                                     100, nat.stream_handle()), "vertices block")
    assert torch.equal(blk, rm.vertices_dev[200:300])


def test_fast_screen_equals_exact_path_full_size():
    """Config-3 volumes: the float32-screened kernel == reference-order float64 kernel."""
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    keys = [spec.keys[0], spec.keys[5]]
    a = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in keys]
    b = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in keys]
    scene = demo_scene()
    lib = nat.load_library()
    sa = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    sb = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    try:
        for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)[::9]:
            frame = scene.render_depth(pose, intr)
            lib.tf_set_debug_flags(0)
            tf.integrate_volumes(a, frame, pose, intr, params, sa)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.integrate_volumes(b, frame, pose, intr, params, sb)
    finally:
        lib.tf_set_debug_flags(0)
    assert sa[nat.STAT_VOXEL_UPDATES].item() == sb[nat.STAT_VOXEL_UPDATES].item() > 0
    for x, y in zip(a, b):
        assert torch.equal(x.voxels, y.voxels)


def test_axis_aligned_rays_and_lattice_plane_cameras():
    """Degenerate geometry: integer principal point (rays with exactly zero
    components), axis-aligned camera rotations and camera centres on voxel
    lattice planes.  Certified raycast == exact march and float32-screened
    integration == exact integration, bit for bit."""
    intr = CameraIntrinsics(100.0, 100.0, 80.0, 60.0, 160, 120)
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    vs = spec.voxel_size
    rot_y = lambda deg: tf.Pose(np.array([[np.cos(np.radians(deg)), 0, np.sin(np.radians(deg))],
                                          [0, 1, 0],
                                          [-np.sin(np.radians(deg)), 0, np.cos(np.radians(deg))]]),
                                np.zeros(3)).rotation
    poses = []
    for deg, t in ((0, (0.0, 0.0, 0.0)), (90, (-1.5, 0.0, 1.5)), (180, (0.0, 0.0, 3.0)),
                   (270, (1.5, 0.0, 1.5)), (0, (10 * vs, -5 * vs, 20 * vs))):
        r = np.round(rot_y(deg), 12)  # exact 0 / +-1 entries
        poses.append(tf.Pose(r, np.array(t)))
    scene = demo_scene()
    a = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    b = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    lib = nat.load_library()
    stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    try:
        for pose in poses:
            frame = scene.render_depth(pose, intr)
            lib.tf_set_debug_flags(0)
            tf.integrate_volumes(a, frame, pose, intr, params)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.integrate_volumes(b, frame, pose, intr, params)
        for x, y in zip(a, b):
            assert torch.equal(x.voxels, y.voxels)
        hits = 0
        for pose in poses:
            for flag in (0, nat.DEBUG_COOP_ALL):
                fast = tf.RayMap.empty(intr)
                lib.tf_set_debug_flags(flag)
                tf.raycast_volumes(a, pose, intr, fast, params, stats)
                exact = tf.RayMap.empty(intr)
                lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
                tf.raycast_volumes(a, pose, intr, exact, params)
                assert torch.equal(fast.distance_dev, exact.distance_dev)
                assert torch.equal(fast.vertices_dev, exact.vertices_dev)
                assert torch.equal(fast.normals_dev, exact.normals_dev)
                hits += torch.isfinite(exact.distance_dev).sum().item()
    finally:
        lib.tf_set_debug_flags(0)
    assert hits > 5000
    assert stats[nat.STAT_CERT_FAILURES].item() == 0


@pytest.mark.parametrize("n", [49, 50])
def test_odd_and_even_sizes_vs_oracle(n):
    """Partial bricks and the unpaired (odd n) voxel path against the oracle."""
    g = load_golden("fusion_small.npz")
    intr = _intr(g["intr"])
    vs = 0.03
    vol = tf.TsdfSubvolume.empty([-25, -23, 7], n, n * vs)
    params = tf.FusionParams(float(g["tau"]))
    t = np.zeros((n, n, n), np.float32)
    w = np.zeros((n, n, n), np.float32)
    stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    for frame, m in zip(g["frames"], g["poses"]):
        pose = _pose(m)
        stats.zero_()
        tf.integrate_volumes([vol], tf.DepthFrame(frame), pose, intr, params, stats)
        want = _oracle_integrate(t, w, vol, frame, pose, intr, params, threads=2)
        assert stats[nat.STAT_VOXEL_UPDATES].item() == want
    pair = vol.voxels.cpu().numpy()
    assert np.array_equal(pair[..., 0], t)
    assert np.array_equal(pair[..., 1], w)


def test_saturated_fixed_point_shortcut_is_exact():
    """max_weight = 3 saturates quickly; skipped no-op stores must equal real ones."""
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(3.0, 254, 254)
    params = tf.FusionParams(truncation=4 * spec.voxel_size, max_weight=3.0)
    vols = [tf.TsdfSubvolume.empty(spec.keys[0], spec.voxels_per_side, spec.subvolume_side_length)
            for _ in range(3)]
    scene = demo_scene()
    lib = nat.load_library()
    stats = [torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda") for _ in range(3)]
    flags = [0, nat.DEBUG_NO_FIXEDPOINT, nat.DEBUG_EXACT_ONLY]
    try:
        for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)[:6]:
            frame = scene.render_depth(pose, intr)
            for v, s, fl in zip(vols, stats, flags):
                lib.tf_set_debug_flags(fl)
                tf.integrate_volumes([v], frame, pose, intr, params, s)
    finally:
        lib.tf_set_debug_flags(0)
    assert stats[0][nat.STAT_NOOP_UPDATES].item() > 0
    assert stats[1][nat.STAT_NOOP_UPDATES].item() == 0
    assert (stats[0][nat.STAT_VOXEL_UPDATES].item() == stats[1][nat.STAT_VOXEL_UPDATES].item()
            == stats[2][nat.STAT_VOXEL_UPDATES].item())
    assert torch.equal(vols[0].voxels, vols[2].voxels)
    assert torch.equal(vols[1].voxels, vols[2].voxels)


def test_certified_raycast_equals_exact_march_full_size():
    """Config-3 volumes, several views: certified fast march == exact reference march."""
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length)
             for k in spec.keys]
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
    for pose in poses[:8]:
        tf.integrate_volumes(tiles, scene.render_depth(pose, intr), pose, intr, params)
    lib = nat.load_library()
    stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    try:
        for pose in (poses[3], poses[7], poses[20]):
            fast = tf.RayMap.empty(intr)
            lib.tf_set_debug_flags(0)
            tf.raycast_volumes(tiles, pose, intr, fast, params, stats)
            exact = tf.RayMap.empty(intr)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.raycast_volumes(tiles, pose, intr, exact, params)
            assert torch.isfinite(exact.distance_dev).sum().item() > 30000
            assert torch.equal(fast.distance_dev, exact.distance_dev)
            assert torch.equal(fast.vertices_dev, exact.vertices_dev)
            assert torch.equal(fast.normals_dev, exact.normals_dev)
    finally:
        lib.tf_set_debug_flags(0)
    # the certified path must carry the bulk of the work
    assert stats[nat.STAT_EXACT_SAMPLES].item() < 0.02 * stats[nat.STAT_RAY_SAMPLES].item()
    assert stats[nat.STAT_CERT_FAILURES].item() == 0


def test_cooperative_raycast_equals_exact_march_full_size():
    """Every ray through the warp-cooperative march (TF_DEBUG_COOP_ALL) == exact march."""
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length)
             for k in spec.keys]
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
    for pose in poses[:10]:
        tf.integrate_volumes(tiles, scene.render_depth(pose, intr), pose, intr, params)
    lib = nat.load_library()
    stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    try:
        for pose in (poses[4], poses[11]):
            coop = tf.RayMap.empty(intr)
            lib.tf_set_debug_flags(nat.DEBUG_COOP_ALL)
            tf.raycast_volumes(tiles, pose, intr, coop, params, stats)
            exact = tf.RayMap.empty(intr)
            lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
            tf.raycast_volumes(tiles, pose, intr, exact, params)
            assert torch.isfinite(exact.distance_dev).sum().item() > 30000
            assert torch.equal(coop.distance_dev, exact.distance_dev)
            assert torch.equal(coop.vertices_dev, exact.vertices_dev)
            assert torch.equal(coop.normals_dev, exact.normals_dev)
    finally:
        lib.tf_set_debug_flags(0)
    assert stats[nat.STAT_CERT_FAILURES].item() == 0


def test_brick_summary_stays_exact_under_integration():
    """The incrementally maintained free-space summary equals a rebuild."""
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length)
             for k in spec.keys[:4]]
    scene = demo_scene()
    for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)[:6]:
        tf.integrate_volumes(tiles, scene.render_depth(pose, intr), pose, intr, params)
    lib = nat.load_library()
    for t in tiles:
        maintained = t.brick_bad.clone()
        flags = t.brick_flags.clone()
        t.invalidate_summary()
        t._summary_for(params.truncation)
        assert torch.equal(maintained, t.brick_bad)
        assert torch.equal(flags, t.brick_flags)
    good = sum(int(((t.brick_bad & 0xFFFF) == 0).sum().item()) for t in tiles)
    unseen = sum(int(((t.brick_bad >> 16) == 0).sum().item()) for t in tiles)
    assert good > 1000 and unseen > 1000  # both kinds of skippable bricks exist
    assert lib.tf_good_threshold(params.truncation) > 0.99 * params.truncation


def test_volume_offsets_beyond_32_bits():
    """n = 1640 (35 GB per volume): voxel offsets of slices z >= 1597 exceed
    2^32.  A plane 0.52 m in front of a camera at z = 6.0 m puts the surface
    at voxel z ~ 1630, so bricks there mix free-space and band voxels (the
    general kernel's free-space path writes past 2^32); the float32-screened
    integration equals the exact one, bit for bit, and so do the raycasts."""
    n, vs = 1640, 0.004
    intr = CameraIntrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    params = tf.FusionParams.for_voxel_size(vs)
    pose = Pose(np.eye(3), np.array([0.0, 0.0, 6.0]))
    depth = torch.full((120, 160), 0.52, dtype=torch.float64, device="cuda")
    lib = nat.load_library()
    a = tf.TsdfSubvolume.empty((-820, -820, 0), n, n * vs)
    b = tf.TsdfSubvolume.empty((-820, -820, 0), n, n * vs)
    try:
        tf.integrate_volumes([a], depth, pose, intr, params)
        lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
        tf.integrate_volumes([b], depth, pose, intr, params)
        lib.tf_set_debug_flags(0)
        assert (a.voxels[1620:, ..., 1] > 0).any()
        assert torch.equal(a.voxels[1500:], b.voxels[1500:])
        assert torch.equal(a.voxels, b.voxels)
        got, want = tf.RayMap.empty(intr), tf.RayMap.empty(intr)
        tf.raycast_volumes([a], pose, intr, got, params)
        lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
        tf.raycast_volumes([a], pose, intr, want, params)
        assert torch.isfinite(want.distance_dev).sum().item() > 10000
        assert torch.equal(got.distance_dev, want.distance_dev)
        assert torch.equal(got.normals_dev, want.normals_dev)
    finally:
        lib.tf_set_debug_flags(0)
        del a, b
        torch.cuda.empty_cache()


@pytest.mark.parametrize("pinned", [False, True])
def test_pipeline_with_tracking_matches_the_reference(tmp_path, pinned):
    """run_fusion with ICP tracking on, against the reference's own
    run_fusion (tests/golden/pipeline_small.npz, pipeline.py:117-197): the
    same frames tracked, identical inlier counts per frame, poses equal to
    1e-12 (the device ICP's float64 sums associate differently from numpy's;
    measured 3e-16), and the final extracted cloud bit-identical (8360
    points: the poses' last-bit differences reach no TSDF voxel here)."""
    g = load_golden("pipeline_small.npz")
    fx, fy, cx, cy, w, h = g["intr"]
    cfg = tf.RunConfig(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h), side_length=3.0,
                       resolution=126, resident_resolution=126, use_groundtruth=False)
    gt = [Pose(m[:3, :3], m[:3, 3]) for m in g["gt_poses"]]
    # pinned host frames take the double-buffered upload and the split
    # integration (its first half overlapping the previous raycast)
    frames = ([torch.from_numpy(np.ascontiguousarray(f)).pin_memory() for f in g["frames"]] if pinned
              else [tf.DepthFrame(f) for f in g["frames"]])
    res = tf.run_fusion(frames, cfg, tmp_path, gt_poses=gt)
    assert res.lost_frames == int(g["lost_frames"]) == 0
    assert [r.tracked for r in res.records] == g["tracked"].tolist()
    assert [r.correspondences for r in res.records] == g["correspondences"].tolist()
    got = np.stack([p.matrix for p in res.poses])
    assert np.abs(got - g["poses"]).max() < 1e-12
    rms = np.array([r.residual_rms for r in res.records])
    ok = np.isfinite(g["residual_rms"])
    assert np.array_equal(np.isfinite(rms), ok)
    assert np.allclose(rms[ok], g["residual_rms"][ok], rtol=1e-6, atol=1e-12)
    assert np.array_equal(res.cloud.vertices, g["cloud_vertices"])
    assert np.array_equal(res.cloud.normals, g["cloud_normals"])


@pytest.mark.parametrize("tier,pinned", [("disk", False), ("host", False), ("host", True)])
def test_dynamic_placement_and_spill_match_the_reference(tmp_path, tier, pinned):
    """Dynamic placement down a corridor with tiles spilling (at most 4 tiles,
    3 resident), against the reference's own pipeline
    (tests/golden/dynamic_small.npz, pipeline.py:117-197, volumes.py:249-331):
    every frame's allocated keys in allocation order, the residency and spill
    counters, and the final extracted cloud, bit for bit — with the reference's
    disk tier and with the pinned-host tier."""
    g = load_golden("dynamic_small.npz")
    fx, fy, cx, cy, w, h = g["intr"]
    cfg = tf.RunConfig(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h), dynamic=True,
                       block_voxels=34, block_side_length=0.64, max_volumes=4, max_resident=3,
                       use_groundtruth=True, spill_tier=tier)
    pipe = tf.FusionPipeline(cfg, tmp_path)
    for i, (f, m) in enumerate(zip(g["frames"], g["poses"])):
        frame = torch.from_numpy(np.ascontiguousarray(f)).pin_memory() if pinned else tf.DepthFrame(f)
        r = pipe.step(frame, Pose(m[:3, :3], m[:3, 3]))
        want = [tuple(k) for k in g["keys"][g["offsets"][i]:g["offsets"][i + 1]].tolist()]
        assert list(pipe.volumes.keys()) == want, f"frame {i}"
        got = [r.volumes, r.resident, r.files_read, r.files_written, r.bytes_read, r.bytes_written]
        assert got == g["counters"][i].tolist(), f"frame {i}"
    res = pipe.finish()
    assert np.array_equal(res.cloud.vertices, g["cloud_vertices"])
    assert np.array_equal(res.cloud.normals, g["cloud_normals"])


def test_split_integration_equals_one_call():
    """SplitIntegrator (tf_integrate_prepare on a side stream, then
    tf_integrate_finish) == integrate_volumes, bit for bit, voxels and brick
    summaries, frame after frame, with the frames' pipelining on."""
    intr = CameraIntrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    a = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    b = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 24)[:8]
    frames = [torch.from_numpy(scene.render_depth(p, intr).data).cuda() for p in poses]
    torch.cuda.synchronize()
    split = tf.tsdf.SplitIntegrator()
    for f, p in zip(frames, poses):
        tf.integrate_volumes(a, f, p, intr, params)
        split(b, f, p, intr, params, depth_ready=True)
        rm = tf.RayMap.empty(intr)
        tf.raycast_volumes(b, p, intr, rm, params)  # the raycast the next prepare overlaps
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x.voxels, y.voxels)
        if x.brick_bad is not None:
            assert torch.equal(x.brick_bad, y.brick_bad)
            assert torch.equal(x.brick_flags, y.brick_flags)
    assert float(b[0].voxels[..., 1].max()) > 0


_HANDOVER_SCRIPT = r"""
import torch, paper_1511_07106_b200 as tf
from paper_1511_07106_b200 import _native as nat
from paper_1511_07106_b200.synth import demo_scene
intr = tf.RunConfig().intrinsics()
spec = tf.init_grid(4.08, 1020, 510)
params = tf.FusionParams.for_voxel_size(spec.voxel_size)
tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
scene = demo_scene()
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
for pose in poses[:10]:
    tf.integrate_volumes(tiles, scene.render_depth(pose, intr), pose, intr, params)
lib = nat.load_library()
stats = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
for pose in (poses[4], poses[11], poses[30]):
    fast = tf.RayMap.empty(intr)
    tf.raycast_volumes(tiles, pose, intr, fast, params, stats)
    exact = tf.RayMap.empty(intr)
    lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
    tf.raycast_volumes(tiles, pose, intr, exact, params)
    lib.tf_set_debug_flags(0)
    assert torch.isfinite(exact.distance_dev).sum().item() > 30000
    assert torch.equal(fast.distance_dev, exact.distance_dev)
    assert torch.equal(fast.vertices_dev, exact.vertices_dev)
    assert torch.equal(fast.normals_dev, exact.normals_dev)
print("coop_rays", stats[nat.STAT_COOP_RAYS].item(), "cert_failures", stats[nat.STAT_CERT_FAILURES].item())
"""


@pytest.mark.parametrize("budget", [2000, 60000])
def test_mid_march_handover_equals_exact_march(budget):
    """Rays handed to the cooperative pass mid-march (tiny per-warp budgets) resume
    from the per-lane march's state and still equal the exact march bit for bit."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, TFB200_RAY_BUDGET=str(budget))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _HANDOVER_SCRIPT], env=env, cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    words = r.stdout.split()
    coop = int(words[words.index("coop_rays") + 1])
    assert coop > 5000, r.stdout          # the hand-over really happened, many times
    assert int(words[words.index("cert_failures") + 1]) == 0


_SCREEN_SCRIPT = r"""
import torch, paper_1511_07106_b200 as tf
from paper_1511_07106_b200 import _native as nat
from paper_1511_07106_b200.synth import demo_scene
intr = tf.RunConfig().intrinsics()
spec = tf.init_grid(4.08, 1020, 510)
params = tf.FusionParams.for_voxel_size(spec.voxel_size)
keys = [spec.keys[k] for k in (2, 5, 6)]          # the busiest tiles and a quiet one
fast = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in keys]
exact = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in keys]
scene = demo_scene()
lib = nat.load_library()
sf = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
se = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
for pose in tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)[0:24:6]:
    depth = scene.render_depth(pose, intr)
    tf.integrate_volumes(fast, depth, pose, intr, params, sf)
    lib.tf_set_debug_flags(nat.DEBUG_EXACT_ONLY)
    tf.integrate_volumes(exact, depth, pose, intr, params, se)
    lib.tf_set_debug_flags(0)
    for a, b in zip(fast, exact):
        assert torch.equal(a.voxels.view(torch.int32), b.voxels.view(torch.int32))
    assert sf[nat.STAT_VOXEL_UPDATES].item() == se[nat.STAT_VOXEL_UPDATES].item()
print("updates", sf[nat.STAT_VOXEL_UPDATES].item(), "exact_voxels", sf[nat.STAT_EXACT_VOXELS].item())
"""


@pytest.mark.parametrize("split,queue_cap,stream", [("1", None, "2"), ("0", None, "2"), ("1", "2000", "2"),
                                                    ("0", "2000", "2"), ("1", None, "0"), ("1", "2000", "1")])
def test_screen_modes_and_queue_overflow_equal_exact(split, queue_cap, stream):
    """The general bricks' screen in the prepare phase (masks + brick_apply_kernel,
    the default) and the one-kernel screen+update (TFB200_SPLIT_SCREEN=0) equal the
    reference-order exact kernel bit for bit on config 3's busiest tiles — also with
    the exact queue capped at 2000 entries, so the overflow paths (exact updates in
    place; in the split screen, marked in the masks) carry most undecided voxels.
    ``stream``: TFB200_FUSED_STREAM (2: free-space + masked updates in one kernel, the
    exact band beside it; 1: the exact band after it; 0: separate free-space kernel)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, TFB200_SPLIT_SCREEN=split, TFB200_FUSED_STREAM=stream)
    if queue_cap:
        env["TFB200_QUEUE_CAP"] = queue_cap
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _SCREEN_SCRIPT], env=env, cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    words = r.stdout.split()
    assert int(words[words.index("updates") + 1]) > 1_000_000
    if queue_cap:  # far more undecided voxels than queue entries
        assert int(words[words.index("exact_voxels") + 1]) > 10 * int(queue_cap)


def test_tma_staged_free_bricks_equal_exact():
    """The TMA-staged free-space kernel (TFB200_FREE_TMA=1: 8x8x8 tensor-map box loads
    into shared memory, mbarrier double buffering) gives the same voxels as the
    reference-order exact kernel on config 3's busiest tiles."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, TFB200_FREE_TMA="1", TFB200_FUSED_STREAM="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _SCREEN_SCRIPT], env=env, cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]


def test_fresh_raycast_ignores_previous_map():
    """raycast_volumes(fresh=True) on a map full of stale hits (TF_RAYCAST_FRESH: the
    map is never read, every pixel written) == reset() + raycast, bit for bit —
    including the pixels finished by the cooperative pass (tiny per-warp budget
    via DEBUG_COOP_ALL on a second frame)."""
    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length)
             for k in spec.keys]
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
    for pose in poses[:6]:
        tf.integrate_volumes(tiles, scene.render_depth(pose, intr), pose, intr, params)
    lib = nat.load_library()
    try:
        for flag in (0, nat.DEBUG_COOP_ALL):
            lib.tf_set_debug_flags(flag)
            want = tf.RayMap.empty(intr)
            tf.raycast_volumes(tiles, poses[5], intr, want, params)
            stale = tf.RayMap.empty(intr)
            tf.raycast_volumes(tiles, poses[30], intr, stale, params)   # another view's hits
            stale.distance_dev[::7] = 0.25                               # and some nonsense
            stale.normals_dev[::5] = 3.0
            tf.raycast_volumes(tiles, poses[5], intr, stale, params, fresh=True)
            assert torch.equal(stale.distance_dev, want.distance_dev)
            assert torch.equal(stale.vertices_dev, want.vertices_dev)
            assert torch.equal(stale.normals_dev, want.normals_dev)
    finally:
        lib.tf_set_debug_flags(0)
