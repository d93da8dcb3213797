"""Debug: time the raycast of one config-3 frame per-lane vs. all-cooperative."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200 import _native as nat  # noqa: E402
from paper_1511_07106_b200.synth import demo_scene  # noqa: E402

intr = tf.RunConfig().intrinsics()
spec = tf.init_grid(4.08, 1020, 510)
params = tf.FusionParams.for_voxel_size(spec.voxel_size)
tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
scene = demo_scene()
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
for p in poses[:40]:
    tf.integrate_volumes(tiles, scene.render_depth(p, intr), p, intr, params)
lib = nat.load_library()
for flag, name in ((0, "per-lane"), (nat.DEBUG_COOP_ALL, "coop-all"), (0, "per-lane")):
    lib.tf_set_debug_flags(flag)
    st = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
    rm = tf.RayMap.empty(intr)
    tf.raycast_volumes(tiles, poses[41], intr, rm, params)
    rm = tf.RayMap.empty(intr)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    tf.raycast_volumes(tiles, poses[41], intr, rm, params, st)
    b.record()
    torch.cuda.synchronize()
    print("%-9s %.3f ms  coop rays %d  samples %d  exact %d" % (
        name, a.elapsed_time(b), st[nat.STAT_COOP_RAYS], st[nat.STAT_RAY_SAMPLES], st[nat.STAT_EXACT_SAMPLES]))
lib.tf_set_debug_flags(0)
