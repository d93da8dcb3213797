"""Small workload for memory checking: every kernel family of libtfb200
once on small inputs (and, with --big, one config-3 frame: 8 x 512^3, voxel
offsets near 2^31 per volume).

    TFB200_LIB=paper_1511_07106_b200/libtfb200_checked.so python tools/sanitize_small.py --big

With the bounds-checked build (-DTF_BOUNDS_CHECK) it reports the guarded
index violations (tf_debug_bounds_violations) and exits 1 when any occurred;
compute-sanitizer is closed on the GPU pool, this build stands in for its
memcheck.  (Under compute-sanitizer the same script runs unchanged.)

Covers: integration (screened + exact queue, exact-only, no-cull, colour),
split integration, raycast (per-lane + cooperative pass, all-cooperative,
exact-only), ray-map merge / reset / vertices, trilinear sample, extraction,
endpoint cells + the device histogram, vertex/normal maps + device ICP, and
the peer-memory ray-map reduction with emulated ranks (no waits)."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200 import _native as nat  # noqa: E402
from paper_1511_07106_b200.distributed import PeerExchange, ShardedFusion, owned_keys  # noqa: E402
from paper_1511_07106_b200.synth import demo_scene, render_rgb  # noqa: E402


def main():
    torch.cuda.set_device(0)
    lib = nat.load_library()
    intr = tf.CameraIntrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    spec = tf.init_grid(3.0, 124, 62)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    scene = demo_scene()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 24)[:4]
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length).enable_color()
             for k in spec.keys]
    for flag in (0, nat.DEBUG_EXACT_ONLY, nat.DEBUG_NO_CULL):
        lib.tf_set_debug_flags(flag)
        for p in poses:
            tf.integrate_volumes(tiles, scene.render_depth(p, intr), p, intr, params,
                                 color=render_rgb(scene, p, intr))
    lib.tf_set_debug_flags(0)
    split = tf.tsdf.SplitIntegrator()
    for p in poses:
        d = torch.from_numpy(scene.render_depth(p, intr).data).cuda()
        split(tiles, d, p, intr, params, depth_ready=True)
    for flag in (0, nat.DEBUG_COOP_ALL, nat.DEBUG_EXACT_ONLY):
        lib.tf_set_debug_flags(flag)
        rm = tf.RayMap.empty(intr)
        tf.raycast_volumes(tiles, poses[1], intr, rm, params)
    lib.tf_set_debug_flags(0)
    tf.raycast_colors(tiles, rm, poses[1], intr)
    other = tf.RayMap.empty(intr)
    tf.raycast(tiles[0], poses[2], intr, other, params)
    nat.check(lib.tf_raymap_merge(nat.ptr(rm.distance_dev), nat.ptr(rm.vertices_dev), nat.ptr(rm.normals_dev),
                                  nat.ptr(other.distance_dev), nat.ptr(other.vertices_dev),
                                  nat.ptr(other.normals_dev), intr.width * intr.height, nat.stream_handle()),
              "tf_raymap_merge")
    tf.trilinear_sample(tiles[0], np.array([0.0, 0.0, 1.2]))
    for t in tiles[:2]:
        tf.extract_points(t)
    for sp in (256, 8):
        tf.bin_endpoints(scene.render_depth(poses[0], intr), intr, poses[0], sp, 0.004)
    frame = scene.render_depth(poses[1], intr)
    tf.track(frame, intr, rm, poses[0], tf.TrackingParams(min_correspondences=100))
    # peer-memory reduction, 2 emulated ranks on this device (no waits)
    world = 2
    peers = [PeerExchange(intr, r, world) for r in range(world)]
    PeerExchange.link_local(peers)
    mine = [[tiles[spec.keys.index(k)] for k in owned_keys(spec.keys, r, world)] for r in range(world)]
    for r in range(world):
        peers[r].partial.reset()
        tf.raycast_volumes(mine[r], poses[1], intr, peers[r].partial, params)
    for r in range(world):
        peers[r].reduce(nowait=True)
    shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params, intr)
    for p in poses[:2]:
        shard.step(torch.from_numpy(scene.render_depth(p, intr).data).cuda(), p)
    if "--big" in sys.argv:
        bspec = tf.init_grid(4.08, 1020, 510)
        bintr = tf.RunConfig().intrinsics()
        bparams = tf.FusionParams.for_voxel_size(bspec.voxel_size)
        big = [tf.TsdfSubvolume.empty(k, bspec.voxels_per_side, bspec.subvolume_side_length) for k in bspec.keys]
        orbit = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
        for p in (orbit[0], orbit[9]):
            tf.integrate_volumes(big, scene.render_depth(p, bintr), p, bintr, bparams)
            rmb = tf.RayMap.empty(bintr)
            tf.raycast_volumes(big, p, bintr, rmb, bparams)
        tf.extract_points(big[2])
        del big
    torch.cuda.synchronize()
    v = int(lib.tf_debug_bounds_violations())
    if v == 2 ** 64 - 1:
        print("sanitize workload done (plain build: no bounds counters)")
        return 0
    print(f"sanitize workload done: {v} bounds violations")
    return 1 if v else 0


if __name__ == "__main__":
    sys.exit(main())
