"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container (needs /root/reference and numba):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every array in the fixtures is produced by the reference tilefusion code
(its numba kernels, its numpy tracking, its renderer); nothing here calls
the oracle or the CUDA path.  The fixtures pin both of them:
tests/test_oracle_golden.py (CPU) and tests/test_gpu_parity.py (GPU).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("TILEFUSION_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

import tilefusion as tf  # noqa: E402
from tilefusion import tracking as tr  # noqa: E402
from tilefusion.geometry import rotation_from_axis_angle  # noqa: E402

OUT = Path(__file__).resolve().parent


def anchored_scene():
    # tests/conftest.py:13-23 (same as the CLI demo scene)
    return tf.Scene((
        tf.Sphere(np.array([0.1, 0.05, 1.5]), 0.35),
        tf.Plane(np.array([0.0, 0.5, 0.0]), np.array([0.0, -1.0, 0.0])),
        tf.Box(np.array([-0.75, 0.1, 1.3]), np.array([-0.35, 0.5, 1.75])),
    ))


def intr_arr(intr):
    return np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height], np.float64)


def pose_arr(poses):
    return np.stack([p.matrix for p in poses])


def fusion_fixture():
    """Integrate + raycast + extract on one 48^3 volume (and a 2x1x1 tiling)."""
    intr = tf.CameraIntrinsics(fx=90.0, fy=90.0, cx=47.5, cy=35.5, width=96, height=72)
    scene = anchored_scene()
    poses = tf.orbit_trajectory(np.array([0.0, 0.0, 1.5]), 1.5, 40)[:5]
    frames = [scene.render_depth(p, intr) for p in poses]
    vol = tf.TsdfSubvolume.empty(np.array([-24, -24, 8]), 48, 48 * 0.03)
    params = tf.FusionParams.for_voxel_size(vol.voxel_size)
    snaps_t, snaps_w = [], []
    for f, p in zip(frames, poses):
        tf.integrate(vol, f, p, intr, params)
        snaps_t.append(vol.tsdf.copy())
        snaps_w.append(vol.weight.copy())
    raymaps = []
    for p in (poses[0], poses[4]):
        rm = tf.RayMap.empty(intr)
        tf.raycast(vol, p, intr, rm, params)
        raymaps.append(rm)
    cloud = tf.extract_points(vol)
    np.savez_compressed(
        OUT / "fusion_small.npz",
        intr=intr_arr(intr), poses=pose_arr(poses), frames=np.stack([f.data for f in frames]),
        origin=vol.origin_voxel, n=np.int64(48), side=np.float64(48 * 0.03),
        tau=np.float64(params.truncation), max_weight=np.float64(params.max_weight),
        sample_weight=np.float64(params.sample_weight),
        tsdf_after=np.stack(snaps_t), weight_after=np.stack(snaps_w),
        ray_pose_index=np.array([0, 4]),
        ray_dist=np.stack([r.distance for r in raymaps]),
        ray_vert=np.stack([r.vertices for r in raymaps]),
        ray_norm=np.stack([r.normals for r in raymaps]),
        cloud_verts=cloud.vertices, cloud_norms=cloud.normals,
    )
    print("fusion_small:", len(cloud), "points,", int(np.isfinite(raymaps[1].distance).sum()), "hits")


def tiled_fixture():
    """Tiled-vs-single (evaluation.equivalence_check, test_evaluation.py:59-67 sizes)."""
    intr = tf.CameraIntrinsics(fx=65.625, fy=65.625, cx=40.0, cy=30.0, width=80, height=60)
    scene = tf.Scene((tf.Sphere(np.array([0.0, 0.0, 0.9]), 0.5),))
    poses = tf.orbit_trajectory(np.array([0.0, 0.0, 0.9]), 0.9, 3)
    frames = [scene.render_depth(p, intr) for p in poses]
    spec_t = tf.init_grid(1.8, 28, 14)
    params = tf.FusionParams.for_voxel_size(spec_t.voxel_size)
    tiles = [tf.TsdfSubvolume.empty(np.array(k), spec_t.voxels_per_side, spec_t.subvolume_side_length)
             for k in spec_t.keys]
    dists, verts, norms = [], [], []
    for f, p in zip(frames, poses):
        for v in tiles:
            tf.integrate(v, f, p, intr, params)
        rm = tf.RayMap.empty(intr)
        for v in tiles:
            tf.raycast(v, p, intr, rm, params)
        dists.append(rm.distance)
        verts.append(rm.vertices)
        norms.append(rm.normals)
    np.savez_compressed(
        OUT / "tiled_small.npz",
        intr=intr_arr(intr), poses=pose_arr(poses), frames=np.stack([f.data for f in frames]),
        keys=np.array(spec_t.keys, np.int64), n=np.int64(spec_t.voxels_per_side),
        side=np.float64(spec_t.subvolume_side_length), tau=np.float64(params.truncation),
        tsdf=np.stack([v.tsdf for v in tiles]), weight=np.stack([v.weight for v in tiles]),
        ray_dist=np.stack(dists), ray_vert=np.stack(verts), ray_norm=np.stack(norms),
    )
    print("tiled_small:", len(tiles), "tiles")


def icp_fixture():
    """track() against a fused model with a perturbed seed; every _solve_step recorded."""
    intr = tf.CameraIntrinsics(fx=100.0, fy=100.0, cx=40.0, cy=30.0, width=80, height=60)
    scene = anchored_scene()
    pose = tf.Pose.identity()
    vol = tf.TsdfSubvolume.empty(np.array([-50, -50, 24]), 100, 2.5)
    params = tf.FusionParams.for_voxel_size(0.025)
    integ_frame = scene.render_depth(pose, intr)
    tf.integrate(vol, integ_frame, pose, intr, params)
    model = tf.RayMap.empty(intr)
    tf.raycast(vol, pose, intr, model, params)
    frame = scene.render_depth(pose, intr)
    bump = tf.Pose(rotation_from_axis_angle(np.array([1.0, 0.0, 0.0]), np.radians(1.0)),
                   np.array([0.0, 0.01, 0.0]))
    seed = pose.compose(bump)
    tparams = tf.TrackingParams(min_correspondences=200)

    steps = []
    real = tr._solve_step

    def spy(src_pts, src_nrm, src_valid, model_pts, model_nrm, model_valid, estimate,
            ref_inv, intr_l, params_l, min_pairs):
        out = real(src_pts, src_nrm, src_valid, model_pts, model_nrm, model_valid,
                   estimate, ref_inv, intr_l, params_l, min_pairs)
        rec = {"level_w": intr_l.width, "estimate": estimate.matrix.copy(),
               "min_pairs": min_pairs}
        if out is None:
            rec.update(count=-1, delta=np.full(6, np.nan), rms=np.nan)
        else:
            rec.update(count=out[1], delta=out[0].copy(), rms=out[2])
        steps.append(rec)
        return out

    tr._solve_step = spy
    try:
        result = tf.track(frame, intr, model, pose, tparams, init=seed)
    finally:
        tr._solve_step = real
    # vertex/normal maps of the three pyramid levels (geometry.py:313-317)
    levels = []
    f, i = frame, intr
    for _ in range(3):
        vm = tf.VertexNormalMap.from_depth(i, f)
        levels.append(vm)
        f, i = f.downsampled(), i.scaled(0.5)
    np.savez_compressed(
        OUT / "icp_small.npz",
        intr=intr_arr(intr), frame=frame.data, model_dist=model.distance,
        model_vert=model.vertices, model_norm=model.normals,
        ref_pose=pose.matrix, seed_pose=seed.matrix,
        max_distance=np.float64(tparams.max_distance), max_angle_deg=np.float64(tparams.max_angle_deg),
        iterations=np.array(tparams.iterations), min_correspondences=np.int64(tparams.min_correspondences),
        step_level_w=np.array([s["level_w"] for s in steps]),
        step_estimate=np.stack([s["estimate"] for s in steps]),
        step_min_pairs=np.array([s["min_pairs"] for s in steps]),
        step_count=np.array([s["count"] for s in steps]),
        step_delta=np.stack([s["delta"] for s in steps]),
        step_rms=np.array([s["rms"] for s in steps]),
        result_pose=result.pose.matrix, result_lost=np.bool_(result.lost),
        result_count=np.int64(result.correspondences), result_rms=np.float64(result.residual_rms),
        **{f"vn{l}_verts": levels[l].vertices for l in range(3)},
        **{f"vn{l}_norms": levels[l].normals for l in range(3)},
        **{f"vn{l}_valid": levels[l].valid for l in range(3)},
    )
    print("icp_small:", len(steps), "steps, lost", result.lost, "count", result.correspondences)


def endpoints_fixture():
    """bin_endpoints known answers on a corridor (volumes.py:305-331)."""
    intr = tf.CameraIntrinsics(fx=65.625, fy=65.625, cx=40.0, cy=30.0, width=80, height=60)
    scene = tf.Scene((
        tf.Plane(np.array([0.9, 0.0, 0.0]), np.array([-1.0, 0.0, 0.0])),
        tf.Plane(np.array([-0.9, 0.0, 0.0]), np.array([1.0, 0.0, 0.0])),
        tf.Plane(np.array([0.0, 0.5, 0.0]), np.array([0.0, -1.0, 0.0])),
    ))
    poses = tf.corridor_trajectory(4.0, 6)
    yaw = tf.Pose(rotation_from_axis_angle(np.array([0.0, 1.0, 0.0]), 0.3), np.zeros(3))
    poses = [p.compose(yaw) if k % 2 else p for k, p in enumerate(poses)]
    frames, keys, counts, offsets = [], [], [], [0]
    for p in poses:
        d = scene.render_depth(p, intr).data.copy()
        d[d > 4.0] = 0.0
        frames.append(d)
        c = tf.bin_endpoints(tf.DepthFrame(d), intr, p, 30, 0.02)
        for k in sorted(c):
            keys.append(k)
            counts.append(c[k])
        offsets.append(len(keys))
    np.savez_compressed(
        OUT / "endpoints_small.npz",
        intr=intr_arr(intr), poses=pose_arr(poses), frames=np.stack(frames),
        spacing=np.int64(30), voxel_size=np.float64(0.02),
        keys=np.array(keys, np.int64), counts=np.array(counts, np.int64),
        offsets=np.array(offsets, np.int64),
    )
    print("endpoints_small:", len(keys), "cells")


def pipeline_fixture():
    """run_fusion with ICP tracking on (pipeline.py:117-197, :208-230): one
    128^3 tile, 160x120 frames of the 1.5-degree orbit (config 2's motion),
    ground truth only for frame 0; per-frame poses and records, final cloud."""
    import tempfile
    cfg = tf.RunConfig(fx=131.25, fy=131.25, cx=79.5, cy=59.5, width=160, height=120,
                       side_length=3.0, resolution=126, resident_resolution=126,
                       use_groundtruth=False)
    intr = cfg.intrinsics()
    scene = anchored_scene()
    poses = tf.orbit_trajectory(np.array([0.0, 0.0, 1.5]), 1.5, 240)[:10]
    frames = [scene.render_depth(p, intr) for p in poses]
    with tempfile.TemporaryDirectory() as tmp:
        res = tf.run_fusion(frames, cfg, tmp, gt_poses=poses)
    rec = res.records
    np.savez_compressed(
        OUT / "pipeline_small.npz",
        intr=intr_arr(intr), gt_poses=pose_arr(poses), frames=np.stack([f.data for f in frames]),
        poses=pose_arr(res.poses), tracked=np.array([r.tracked for r in rec]),
        correspondences=np.array([r.correspondences for r in rec], np.int64),
        residual_rms=np.array([r.residual_rms for r in rec], np.float64),
        cloud_vertices=res.cloud.vertices, cloud_normals=res.cloud.normals,
        lost_frames=np.int64(res.lost_frames),
    )
    print("pipeline_small:", len(rec), "frames,", len(res.cloud.vertices), "cloud points, lost",
          res.lost_frames)


def dynamic_fixture():
    """Dynamic placement down a corridor (config 4's kind, pipeline.py:126-127,
    volumes.py:249-331): walls, floor and a box, depth beyond 4 m zeroed,
    ground-truth poses, at most 4 tiles of 34^3 voxels, 3 resident (so tiles
    spill to disk and come back); per frame the allocated keys in order and
    the record counters, then the final cloud."""
    import tempfile
    cfg = tf.RunConfig(fx=65.625, fy=65.625, cx=39.5, cy=29.5, width=80, height=60,
                       dynamic=True, block_voxels=34, block_side_length=0.64, max_volumes=4,
                       max_resident=3, use_groundtruth=True)
    intr = cfg.intrinsics()
    scene = tf.Scene((
        tf.Plane(np.array([0.9, 0.0, 0.0]), np.array([-1.0, 0.0, 0.0])),
        tf.Plane(np.array([-0.9, 0.0, 0.0]), np.array([1.0, 0.0, 0.0])),
        tf.Plane(np.array([0.0, 0.5, 0.0]), np.array([0.0, -1.0, 0.0])),
        tf.Box(np.array([-0.5, 0.2, 2.0]), np.array([-0.2, 0.5, 2.4])),
    ))
    poses = tf.corridor_trajectory(3.0, 12)
    frames = []
    for p in poses:
        d = scene.render_depth(p, intr).data.copy()
        d[d > 4.0] = 0.0
        frames.append(tf.DepthFrame(d))
    keys, offsets, counters = [], [0], []
    with tempfile.TemporaryDirectory() as tmp:
        pipe = tf.FusionPipeline(cfg, tmp)
        for f, p in zip(frames, poses):
            r = pipe.step(f, p)
            ks = pipe.volumes.keys()
            keys.extend(ks)
            offsets.append(len(keys))
            counters.append([r.volumes, r.resident, r.files_read, r.files_written, r.bytes_read,
                             r.bytes_written])
        res = pipe.finish()
    np.savez_compressed(
        OUT / "dynamic_small.npz",
        intr=intr_arr(intr), poses=pose_arr(poses), frames=np.stack([f.data for f in frames]),
        keys=np.array(keys, np.int64).reshape(-1, 3), offsets=np.array(offsets, np.int64),
        counters=np.array(counters, np.int64),
        cloud_vertices=res.cloud.vertices, cloud_normals=res.cloud.normals,
    )
    print("dynamic_small:", len(frames), "frames,", len(set(keys)), "distinct keys,",
          int(np.array(counters)[:, 3].sum()), "spill writes,", len(res.cloud.vertices), "cloud points")


def _sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def config3_fixture():
    """Config 3 at full size (BASELINE configs[2]): the 8 fixed 512^3 tiles of
    init_grid(4.08, 1020, 510), 640x480 frames of the demo orbit, ground-truth
    poses.  The reference's numba integrate_kernel runs frames 0, 9 and 18 into
    every tile (each tile sees the three frames in order); after each frame the
    SHA-256 of every tile's tsdf and weight bytes is recorded, and after frames 0
    and 18 the merged raycast of all 8 tiles (reference tile order).  Hashes
    only: the arrays are 8.6 GB.  Pins the GPU fused path (tests/test_gpu_parity.py)
    and the oracle (tests/test_oracle_golden.py, slow) on the busy tiles too."""
    cfg = tf.RunConfig()
    intr = cfg.intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    scene = anchored_scene()
    poses = tf.orbit_trajectory(np.array([0.0, 0.0, 1.5]), 1.5, 64)
    frames_idx = [0, 9, 18]
    tiles = [tf.TsdfSubvolume.empty(np.array(k), spec.voxels_per_side, spec.subvolume_side_length)
             for k in spec.keys]
    th, wh, upd = [], [], []
    ray = {}
    for f in frames_idx:
        frame = scene.render_depth(poses[f], intr)
        rt, rw, ru = [], [], []
        for v in tiles:
            w0 = v.weight.copy()
            tf.integrate(v, frame, poses[f], intr, params)
            ru.append(int(np.count_nonzero(v.weight != w0)))
            rt.append(_sha(v.tsdf))
            rw.append(_sha(v.weight))
        th.append(rt)
        wh.append(rw)
        upd.append(ru)
        if f in (0, 18):
            rm = tf.RayMap.empty(intr)
            for v in tiles:
                tf.raycast(v, poses[f], intr, rm, params)
            ray[f] = (_sha(rm.distance), _sha(rm.vertices), _sha(rm.normals),
                      int(np.isfinite(rm.distance).sum()))
        print("config3 frame", f, "updates", ru, flush=True)
    np.savez_compressed(
        OUT / "config3_hashes.npz",
        keys=np.array(spec.keys, np.int64), frames=np.array(frames_idx, np.int64),
        tsdf_sha=np.array(th), weight_sha=np.array(wh), changed=np.array(upd, np.int64),
        ray_frames=np.array(sorted(ray), np.int64),
        ray_sha=np.array([ray[f][:3] for f in sorted(ray)]),
        ray_hits=np.array([ray[f][3] for f in sorted(ray)], np.int64),
    )


def icp_full_fixture():
    """Config 2 at full resolution (BASELINE configs[1]): run_fusion's tracking
    on one 256^3 tile (init_grid(3.0, 254, 254)), 640x480, the 1.5-degree orbit,
    frames 0-5.  Every _solve_step of every track() call is recorded with its
    inputs (estimate, level) and outputs (count, delta, rms), plus the SHA-256
    of the model ray map each call tracks against and the reference's poses
    (exact bits), so a GPU pipeline driven by those poses rebuilds the identical
    model and replays every step (tests/test_gpu_parity.py)."""
    import tempfile
    cfg = tf.RunConfig(side_length=3.0, resolution=254, resident_resolution=254,
                       use_groundtruth=False)
    intr = cfg.intrinsics()
    scene = anchored_scene()
    poses = tf.orbit_trajectory(np.array([0.0, 0.0, 1.5]), 1.5, 240)[:6]
    steps = []
    models = []
    real = tr._solve_step
    frame_no = [0]

    def spy(src_pts, src_nrm, src_valid, model_pts, model_nrm, model_valid, estimate,
            ref_inv, intr_l, params_l, min_pairs):
        out = real(src_pts, src_nrm, src_valid, model_pts, model_nrm, model_valid,
                   estimate, ref_inv, intr_l, params_l, min_pairs)
        rec = {"frame": frame_no[0], "level_w": intr_l.width, "estimate": estimate.matrix.copy(),
               "min_pairs": min_pairs}
        if out is None:
            rec.update(count=-1, delta=np.full(6, np.nan), rms=np.nan)
        else:
            rec.update(count=out[1], delta=out[0].copy(), rms=out[2])
        steps.append(rec)
        return out

    tr._solve_step = spy
    import tilefusion.pipeline as tp
    tp_track = tp.track

    def track_spy(frame, intr_, model, ref_pose, params=tr.TrackingParams(), init=None):
        models.append((frame_no[0], _sha(model.distance), _sha(model.vertices),
                       _sha(model.normals), int(np.isfinite(model.distance).sum())))
        return tp_track(frame, intr_, model, ref_pose, params, init)

    tp.track = track_spy
    out_poses, recs = [], []
    try:
        with tempfile.TemporaryDirectory() as tmp:
            pipe = tf.FusionPipeline(cfg, tmp)
            for i, p in enumerate(poses):
                frame_no[0] = i
                r = pipe.step(scene.render_depth(p, intr), p)
                recs.append((r.tracked, r.correspondences, r.residual_rms))
                print("icp_full frame", i, r.tracked, r.correspondences, flush=True)
            out_poses = list(pipe.poses)
    finally:
        tr._solve_step = real
        tp.track = tp_track
    np.savez_compressed(
        OUT / "icp_full.npz",
        intr=intr_arr(intr), gt_poses=pose_arr(poses), poses=pose_arr(out_poses),
        tracked=np.array([r[0] for r in recs]), correspondences=np.array([r[1] for r in recs], np.int64),
        residual_rms=np.array([r[2] for r in recs], np.float64),
        model_frame=np.array([m[0] for m in models], np.int64),
        model_sha=np.array([m[1:4] for m in models]), model_hits=np.array([m[4] for m in models], np.int64),
        step_frame=np.array([s["frame"] for s in steps], np.int64),
        step_level_w=np.array([s["level_w"] for s in steps]),
        step_estimate=np.stack([s["estimate"] for s in steps]),
        step_min_pairs=np.array([s["min_pairs"] for s in steps]),
        step_count=np.array([s["count"] for s in steps]),
        step_delta=np.stack([s["delta"] for s in steps]),
        step_rms=np.array([s["rms"] for s in steps]),
    )
    print("icp_full:", len(steps), "steps over", len(models), "track calls")


CORRIDOR_BOXES = ((-0.85, 0.10, 3.0, -0.45, 0.50, 3.6),
                  (0.40, 0.20, 6.5, 0.85, 0.50, 7.2),
                  (-0.80, -0.30, 10.0, -0.50, 0.50, 10.4),
                  (0.30, 0.00, 13.5, 0.80, 0.50, 14.5),
                  (-0.70, 0.25, 17.0, -0.20, 0.50, 17.5))  # = synth.CORRIDOR_BOXES


def corridor_scene():
    prims = [tf.Plane(np.array([0.9, 0.0, 0.0]), np.array([-1.0, 0.0, 0.0])),
             tf.Plane(np.array([-0.9, 0.0, 0.0]), np.array([1.0, 0.0, 0.0])),
             tf.Plane(np.array([0.0, 0.5, 0.0]), np.array([0.0, -1.0, 0.0]))]
    prims += [tf.Box(np.array(b[:3]), np.array(b[3:])) for b in CORRIDOR_BOXES]
    return tf.Scene(tuple(prims))


CONFIG4 = dict(frames=2000, length=20.0, block_voxels=258, block_side_length=1.024,
               max_volumes=16, hysteresis=1.5)


def _config4_hist(i):
    cfg = tf.RunConfig(dynamic=True, block_voxels=CONFIG4["block_voxels"],
                       block_side_length=CONFIG4["block_side_length"])
    intr = cfg.intrinsics()
    pose = tf.corridor_trajectory(CONFIG4["length"], CONFIG4["frames"])[i]
    d = corridor_scene().render_depth(pose, intr).data.copy()
    d[d > 4.0] = 0.0  # test_acceptance.py:241
    spacing = CONFIG4["block_voxels"] - 2
    c = tf.bin_endpoints(tf.DepthFrame(d), intr, pose, spacing,
                         CONFIG4["block_side_length"] / spacing)
    return sorted(c.items())


def placement_fixture():
    """Config 4's placement over ALL 2000 corridor frames at 640x480
    (BASELINE configs[3]; pipeline.py:126-127, :175-184): per frame the
    reference's bin_endpoints histogram (volumes.py:305-331) and the
    update_allocation decision (volumes.py:358-389) given the allocation the
    previous frames left (ground-truth poses, so placement does not depend on
    the map).  Histograms are computed in a process pool (independent per
    frame); the decisions run in frame order."""
    import multiprocessing as mp
    n = CONFIG4["frames"]
    with mp.get_context("fork").Pool(min(8, os.cpu_count() or 1)) as pool:
        hists = pool.map(_config4_hist, range(n), chunksize=8)
    policy = tf.AllocationPolicy(max_volumes=CONFIG4["max_volumes"],
                                 hysteresis=CONFIG4["hysteresis"])
    current: list = []
    hk, hc, ho = [], [], [0]
    ak, ao, rk, ro = [], [0], [], [0]
    for h in hists:
        for k, c in h:
            hk.append(k)
            hc.append(c)
        ho.append(len(hk))
        added, removed = tf.update_allocation(tuple(current), dict(h), policy)
        for k in removed:
            current.remove(k)
        current.extend(added)
        ak.extend(added)
        ao.append(len(ak))
        rk.extend(removed)
        ro.append(len(rk))
    np.savez_compressed(
        OUT / "placement_config4.npz",
        frames=np.int64(n), length=np.float64(CONFIG4["length"]),
        block_voxels=np.int64(CONFIG4["block_voxels"]),
        block_side_length=np.float64(CONFIG4["block_side_length"]),
        max_volumes=np.int64(CONFIG4["max_volumes"]), hysteresis=np.float64(CONFIG4["hysteresis"]),
        hist_keys=np.array(hk, np.int64).reshape(-1, 3), hist_counts=np.array(hc, np.int64),
        hist_offsets=np.array(ho, np.int64),
        added=np.array(ak, np.int64).reshape(-1, 3), added_offsets=np.array(ao, np.int64),
        removed=np.array(rk, np.int64).reshape(-1, 3), removed_offsets=np.array(ro, np.int64),
        final_keys=np.array(current, np.int64).reshape(-1, 3),
    )
    print("placement_config4:", n, "frames,", len(hk), "cells,", len(ak), "adds,", len(rk), "removals")


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate only the named fixtures
        for name in sys.argv[1:]:
            globals()[name + "_fixture"]()
        sys.exit(0)
    fusion_fixture()
    tiled_fixture()
    icp_fixture()
    endpoints_fixture()
    pipeline_fixture()
    dynamic_fixture()
    config3_fixture()
    icp_full_fixture()
    placement_fixture()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size, "bytes")
